"""In-tree build of the CUDA library (``lib/libvc3_b200.so``) with nvcc.

sm_100a only.  Numerics flags are part of the contract with the reference's
IEEE arithmetic: no FMA contraction (``-fmad=false``; FMAs are written
explicitly where proven safe), no flush-to-zero, IEEE division and sqrt.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = Path(os.environ["VC3_BUILD_OUT"]) if os.environ.get("VC3_BUILD_OUT") else PKG / "lib"
LIB = LIB_DIR / "libvc3_b200.so"
SOURCES = ["vc3_kernels.cu", "vc3_fused.cu", "vc3_fused_as.cu", "vc3_host.cu", "vc3_variants.cu", "vc3_fr.cu"]
HEADERS = ["vc3_device.cuh", "vc3_fused.cuh", "vc3_kern_common.cuh", "vc3_rt.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NUMERICS = ["-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; set NVCC or install the CUDA toolkit")


def _stale() -> bool:
    if not LIB.exists():
        return True
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "vc3_b200.h", Path(__file__)]
    built = LIB.stat().st_mtime
    return any(d.stat().st_mtime > built for d in deps)


def _compile_cmd(src: Path, obj: Path, verbose: bool) -> list[str]:
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", *NUMERICS, "-Xcompiler", "-fPIC",
           "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
    cmd += [f"-D{d}" for d in os.environ.get("VC3_BUILD_DEFINES", "").split()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    return cmd


# headers each translation unit includes beyond the common ones
COMMON_DEPS = ["vc3_device.cuh", "vc3_rt.h"]
EXTRA_DEPS = {"vc3_fused_as.cu": ["vc3_fused.cuh", "vc3_kern_common.cuh"],
              "vc3_fused.cu": ["vc3_kern_common.cuh"],
              "vc3_kernels.cu": ["vc3_kern_common.cuh", "vc3_fused.cuh"]}


def _defines_stamp(obj_dir: Path) -> Path:
    return obj_dir / "defines.txt"


def _obj_stale(src: str, obj: Path) -> bool:
    if not obj.exists():
        return True
    stamp = _defines_stamp(obj.parent)
    if not stamp.exists() or stamp.read_text() != os.environ.get("VC3_BUILD_DEFINES", ""):
        return True
    deps = [CSRC / src] + [CSRC / h for h in COMMON_DEPS + EXTRA_DEPS.get(src, [])]
    deps += [ROOT / "include" / "vc3_b200.h", Path(__file__)]
    built = obj.stat().st_mtime
    return any(d.stat().st_mtime > built for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the shared library if any source is newer than it.

    Each translation unit compiles to its own object (only the stale ones, in
    parallel: the fused kernels' template instantiations dominate the build),
    then one link."""
    obj_dir = LIB_DIR / "obj"
    stamp = _defines_stamp(obj_dir)
    defines = os.environ.get("VC3_BUILD_DEFINES", "")
    if not force and not _stale() and stamp.exists() and stamp.read_text() == defines:
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    obj_dir.mkdir(exist_ok=True)
    objs = [obj_dir / (Path(s).stem + ".o") for s in SOURCES]
    procs = []
    for src, obj in zip(SOURCES, objs):
        if not force and not _obj_stale(src, obj):
            continue
        cmd = _compile_cmd(CSRC / src, obj, verbose)
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {' '.join(failed)}")
    stamp.write_text(defines)
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", *(str(o) for o in objs),
                    "-o", str(tmp)], check=True)
    os.replace(tmp, LIB)
    return LIB


TOOLS = ROOT / "tools"


def build_exhaustive(force: bool = False) -> Path:
    """The FMA-equivalence enumerator (test infrastructure, tools/exhaustive.cu)."""
    out = TOOLS / "exhaustive"
    src = TOOLS / "exhaustive.cu"
    deps = [src, CSRC / "vc3_device.cuh"]
    if force or not out.exists() or any(d.stat().st_mtime > out.stat().st_mtime for d in deps):
        subprocess.run([nvcc(), *ARCH, "-O3", "-std=c++17", *NUMERICS, "-I", str(ROOT / "include"),
                        str(src), "-o", str(out)], check=True)
    return out


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
