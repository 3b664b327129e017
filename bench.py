"""Benchmark of the compressed float3 vector add (BASELINE.json config C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One step = one fused ``add_compressed`` (c = compress(decompress(a) +
decompress(b)), all-single policy, layout <0,7,22>-17-18@80) over 2^28
synthetic cube vectors per GPU, inputs resident in HBM.  Weak scaling: every
rank owns its own contiguous 2^28-vector shard; there is no collective on the
data path (only the barrier and the max-over-ranks timing reduction).

Printed on rank 0, one JSON line: ``value`` = whole-job Gvec/s from CUDA
events (max over ranks); the same line carries the uncompressed float32 add on
the same GPU (the speed-up the paper reports), ``e2e`` (the same metric
through the public host-array API with host<->device copies in the timed
region), the roofline of the fused kernel against MEASURED_PEAKS.json, the
CPU baseline (the C restatement of the reference path on the host cores) and
SM clocks sampled during the timed region.

``--impl reference`` instead times the reference's CPU path (oracle/ port,
all host threads) on the same metric, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "compressed float3 vector-add Gvec/s & HBM GB/s vs fp32 add; speedup"
UNIT = "Gvec/s"
N_PER_GPU = 1 << 28
BYTES_COMPRESSED = 24   # read a, b words + write c word (bench.py:27)
BYTES_RAW = 36          # read two float3 + write one (bench.py:26)
CPU_SAMPLE = 1 << 22    # vectors per CPU-baseline step


def workload_config(n: int, world: int, scaling: str = "weak", global_n: int | None = None) -> dict:
    return {
        "workload": ("C2 compressed vector add c=a+b (fused decompress-add-recompress), "
                     "float3 cube vectors U[-1,1]^3, all-single policy, layout <0,7,22>-17-18@80"
                     if scaling == "weak" else
                     "C5 strong scaling: the C2 fused add on a fixed global array split into "
                     "contiguous shards"),
        "n_vectors_per_gpu": n,
        "global_vectors": global_n if global_n is not None else n * world,
        "bytes_per_vector": BYTES_COMPRESSED,
        "l2": "working set >= 6 GiB per GPU >> 126 MB L2; no flush needed",
        "parallelism": f"shard{world} (contiguous, no collective)",
    }


def measured_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text()) if p.exists() else {}
    except ValueError:
        return {}


def ncu_traffic() -> float | None:
    """DRAM bytes per fused-add launch from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_add_traffic.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["dram_bytes_per_launch"])
        except (KeyError, ValueError):
            return None
    return None


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during a region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = ("gloo" if args.impl == "reference" or os.environ.get("VC3_BENCH_SHARE_GPU") == "1"
                   else "nccl")
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path (C port of _kernels.py), all threads
# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    if rank != 0:
        return
    sample = args.cpu_sample
    sys.path.insert(0, str(ROOT / "oracle"))
    import vc3_oracle

    from paper_2003_02633_b200.layout import ALL_SINGLE_POLICY, DEFAULT_LAYOUT

    threads = vc3_oracle.default_threads()
    g = np.random.Generator(np.random.Philox(key=(0, 0)))
    va = g.uniform(-1.0, 1.0, (sample, 3)).astype(np.float32)
    vb = g.uniform(-1.0, 1.0, (sample, 3)).astype(np.float32)
    a = vc3_oracle.compress(va, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    b = vc3_oracle.compress(vb, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    for _ in range(args.warmup):
        vc3_oracle.add_compressed(a, b, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vc3_oracle.add_compressed(a, b, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    dt = (time.perf_counter() - t0) / args.steps
    value = sample / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(N_PER_GPU, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", **host_info(),
                         "sample": f"{sample} cube vectors per step (bounded sample of the "
                                   f"2^28-vector workload), oracle/vc3_oracle.c add_compressed "
                                   f"on {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def cpu_baseline_sample(sample: int = CPU_SAMPLE) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import vc3_oracle

    from paper_2003_02633_b200.layout import ALL_SINGLE_POLICY, DEFAULT_LAYOUT

    threads = vc3_oracle.default_threads()
    g = np.random.Generator(np.random.Philox(key=(0, 1)))
    va = g.uniform(-1.0, 1.0, (sample, 3)).astype(np.float32)
    vb = g.uniform(-1.0, 1.0, (sample, 3)).astype(np.float32)
    a = vc3_oracle.compress(va, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    b = vc3_oracle.compress(vb, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    vc3_oracle.add_compressed(a, b, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        vc3_oracle.add_compressed(a, b, DEFAULT_LAYOUT, ALL_SINGLE_POLICY, threads)
    dt = (time.perf_counter() - t0) / reps
    out = {"value": sample / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{reps} x {sample} cube vectors, oracle/vc3_oracle.c add_compressed, "
                     f"{threads} threads, after 1 warm-up pass"}
    out.update(host_info())
    shipped = numba_reference_sample(a, b)
    if shipped is not None:
        out["reference_as_shipped"] = shipped
    return out


def host_info() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "affinity_cores": len(os.sched_getaffinity(0))}


_NB_OPERANDS = None  # (a, b) inherited by the fork pool's workers (never pickled)


def _numba_shard(bounds):
    """Worker of the fork pool: the reference's own add_compressed on one
    contiguous shard (inputs inherited through fork, result discarded)."""
    import vc3.bench as rb

    lo, hi = bounds
    a, b = _NB_OPERANDS
    t0 = time.perf_counter()
    rb.add_compressed(a[lo:hi], b[lo:hi])
    return time.perf_counter() - t0


def numba_reference_sample(a: np.ndarray, b: np.ndarray) -> dict | None:
    """The reference's shipped CPU path (numba kernels through
    vc3.bench.add_compressed, bench.py:41-69), installed offline into
    baseline/_ref: one core as shipped, then sharded over all cores with a
    fork process pool.  None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "vc3").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vc3_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import vc3.bench as rb
    except Exception as exc:  # numba missing or broken: report, do not fail the bench
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    n = min(a.size, 1 << 21)
    rb.add_compressed(a[:1024], b[:1024])  # JIT compile (cached)
    t0 = time.perf_counter()
    rb.add_compressed(a[:n], b[:n])
    one = n / (time.perf_counter() - t0) / 1e9
    import multiprocessing as mp

    global _NB_OPERANDS
    procs = len(os.sched_getaffinity(0))
    nn = min(a.size, n * procs)
    _NB_OPERANDS = (a, b)
    bounds = [(nn * i // procs, nn * (i + 1) // procs) for i in range(procs)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_numba_shard, [(0, 1024)] * procs, chunksize=1)  # warm every worker's JIT
        t0 = time.perf_counter()
        pool.map(_numba_shard, bounds, chunksize=1)
        allc = nn / (time.perf_counter() - t0) / 1e9
    _NB_OPERANDS = None
    return {"one_core": {"value": one, "unit": UNIT, "cores": 1,
                         "sample": f"{n} cube vectors, vc3.bench.add_compressed (numba, as shipped)"},
            "all_cores": {"value": allc, "unit": UNIT, "cores": procs,
                          "sample": f"{nn} vectors in {procs} contiguous shards, fork pool"}}


def time_region(fn, steps, stream, torch):
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    end.synchronize()
    return start.elapsed_time(end) / steps  # ms


def run_secondary(args, vc3b, lib, dev, stream, n):
    """BASELINE configs C3 (variant codecs) and C4 (RK stage on an ICV field),
    each timed with CUDA events on the launching stream."""
    import torch

    from paper_2003_02633_b200 import _native, fields, variants

    lay = vc3b.DEFAULT_LAYOUT
    cl = _native.c_layout(lay)
    out = {}
    steps = max(3, min(args.steps, 10))

    # C3: companding + fractional splitting, round trip on n cube vectors
    gen = torch.Generator(device=dev).manual_seed(99)
    v = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    w = torch.empty(n, dtype=torch.uint64, device=dev)
    vh = torch.empty_like(v)
    c3 = {}
    for name, var in (("uniform", variants.Compander("uniform")),
                      ("cosine", variants.Compander("cosine")),
                      ("tanh_0.5", variants.Compander("tanh", 0.5)),
                      ("tanh_2.0", variants.Compander("tanh", 2.0)),
                      ("split_98304", variants.SplitConfig(35, 98303))):
        cv = variants.c_variant(var, lay)
        enc = lambda: lib.vc3_compress_variant(v.data_ptr(), w.data_ptr(), n, cl, cv, None,
                                              stream.cuda_stream)
        dec = lambda: lib.vc3_decompress_variant(w.data_ptr(), vh.data_ptr(), n, cl, cv,
                                                stream.cuda_stream)
        enc(); dec()
        torch.cuda.synchronize()
        te = time_region(enc, steps, stream, torch)
        td = time_region(dec, steps, stream, torch)
        c3[name] = {"compress_gvec_s": n / (te * 1e-3) / 1e9,
                    "decompress_gvec_s": n / (td * 1e-3) / 1e9}
    out["C3_variants"] = {"n_vectors": n, "unit": UNIT, "results": c3,
                          "note": "double-precision ORACLE-policy angles + CUDA libm "
                                  "transcendentals, as the reference's studies"}
    del v, w, vh

    # C4: low-storage RK stage on compressed momentum of an isentropic vortex
    n_elem = n // 125
    mom, vel = fields.icv_fields(n_elem, 30.0, device=dev)
    npts = mom.shape[0]
    pol = vc3b.ALL_SINGLE_POLICY
    q = vc3b.compress(mom, lay, pol)
    dq = vc3b.compress(vel * 1e-3, lay, pol)
    R = vc3b.compress(vel, lay, pol)
    qf, dqf, Rf = mom.reshape(-1).clone(), (vel * 1e-3).reshape(-1), vel.reshape(-1)
    del mom
    k = [0]

    def rk(flags=0):
        s_ = k[0] % 5
        k[0] += 1
        lib.vc3_rk_stage_ex(float(fields.LSRK_A[s_]), float(fields.LSRK_B[s_]), 1e-3, q.data_ptr(),
                            dq.data_ptr(), R.data_ptr(), npts, cl, pol.mask, flags, stream.cuda_stream)

    def rk_contract():
        rk(1)

    def rk32():
        s_ = k[0] % 5
        k[0] += 1
        lib.vc3_rk_stage_f32(float(fields.LSRK_A[s_]), float(fields.LSRK_B[s_]), 1e-3,
                             qf.data_ptr(), dqf.data_ptr(), Rf.data_ptr(), 3 * npts,
                             stream.cuda_stream)

    rk(); rk32()
    torch.cuda.synchronize()
    tc = time_region(rk, steps, stream, torch)
    rk_contract()
    tcc = time_region(rk_contract, steps, stream, torch)
    tf = time_region(rk32, steps, stream, torch)
    out["C4_rk_stage_icv"] = {
        "n_points": npts, "field": "ICV beta=5 gamma=1.4 psi=30deg, k=4 FR points, "
                                   "[n_upts][n_elem] rows", "unit": UNIT,
        "compressed_gvec_s": npts / (tc * 1e-3) / 1e9,
        "compressed_hbm_gb_s": 40 * npts / (tc * 1e-3) / 1e9,
        "compressed_contract_gvec_s": npts / (tcc * 1e-3) / 1e9,
        "fp32_gvec_s": npts / (tf * 1e-3) / 1e9,
        "fp32_hbm_gb_s": 60 * npts / (tf * 1e-3) / 1e9,
        "speedup_vs_fp32": tf / tc}
    del q, dq, R, qf, dqf, Rf, vel
    torch.cuda.empty_cache()

    # C4 at the paper's mesh size (800 elements x 125 points = 10^5 vectors):
    # one full LSRK step, five eager launches vs one CUDA-graph replay
    from paper_2003_02633_b200 import ops

    ms_, vs_ = fields.icv_fields(800, 30.0, device=dev)
    qs = vc3b.compress(ms_, lay, pol)
    dqs = vc3b.compress(vs_ * 1e-3, lay, pol)
    Rs = vc3b.compress(vs_, lay, pol)
    stp = ops.LSRKStep(qs, dqs, Rs, 1e-3, lay, pol).capture()
    reps = 200
    stp.step(); stp.step_eager()
    torch.cuda.synchronize()
    te_ = time_region(stp.step_eager, reps, stream, torch)
    tg_ = time_region(stp.step, reps, stream, torch)
    out["C4_rk_stage_icv"]["paper_mesh_lsrk_step_us"] = {
        "n_points": int(qs.numel()), "eager_5_launches": te_ * 1e3, "cuda_graph": tg_ * 1e3}
    del ms_, vs_, qs, dqs, Rs, stp

    # C6: FR flux divergence (Alg. 1) on the tcgen05 kernel,
    # degree-4 hexahedra, 5 equation rows per point, compressed vs float32 fluxes
    from paper_2003_02633_b200 import fr

    kdeg, n_vars, n_el = 4, 5, 1 << 18
    ns = (kdeg + 1) ** 3
    op = fr.Operator(fr.divergence_operator(kdeg))
    mom, vel = fields.icv_fields(n_el, 30.0, device=dev)
    F = torch.stack([mom.reshape(ns, n_el, 3) * (1.0 + 0.25 * c_) for c_ in range(n_vars - 1)]
                    + [vel.reshape(ns, n_el, 3)], dim=1).contiguous()
    del mom, vel
    words = vc3b.compress(F.reshape(-1, 3), lay, vc3b.ALL_SINGLE_POLICY).reshape(ns, n_vars, n_el)
    div = torch.empty((ns, n_vars, n_el), dtype=torch.float32, device=dev)
    fc = lambda: lib.vc3_fr_divergence(words.data_ptr(), op.staged.data_ptr(), div.data_ptr(), n_el,
                                       n_vars, n_el, ns, cl, stream.cuda_stream)
    ff = lambda: lib.vc3_fr_divergence_f32(F.data_ptr(), op.staged.data_ptr(), div.data_ptr(), n_el,
                                           n_vars, n_el, ns, stream.cuda_stream)
    m1 = np.ascontiguousarray(fr.lagrange_derivative_matrix(fr.gauss_legendre_nodes(kdeg)),
                              dtype=np.float32)
    hc = lambda: lib.vc3_fr_divergence_hex(words.data_ptr(), m1.ctypes.data, kdeg, div.data_ptr(),
                                           n_el, n_vars, n_el, cl, stream.cuda_stream)
    hf = lambda: lib.vc3_fr_divergence_hex_f32(F.data_ptr(), m1.ctypes.data, kdeg, div.data_ptr(),
                                               n_el, n_vars, n_el, stream.cuda_stream)
    fc(); ff(); hc(); hf()
    torch.cuda.synchronize()
    tcm = time_region(fc, steps, stream, torch)
    tf3 = time_region(ff, steps, stream, torch)
    thc = time_region(hc, steps, stream, torch)
    thf = time_region(hf, steps, stream, torch)
    rows = n_el * n_vars
    dense = 2.0 * 3 * ns * ns * rows  # flops of Alg. 1 per launch
    # dense TF32 peak: tools/umma_bench.cu (back-to-back tcgen05.mma kind::tf32
    # M128 N128 K8 from shared memory, one CTA per SM) measured 1058 TFLOP/s on
    # this pool's B200; B200_PROFILING.md states 1.1 PFLOP/s dense
    tf32_peak = 1058.0
    ach = 3 * dense / (tcm * 1e-3) / 1e12
    out["C6_fr_divergence"] = {
        "k": kdeg, "n_points": ns, "n_vars": n_vars, "n_elem": n_el, "unit": "G elem-eq/s",
        "field": "ICV momentum/velocity rows, [ns][n_vars][n_elem] words",
        "compressed": rows / (tcm * 1e-3) / 1e9, "fp32": rows / (tf3 * 1e-3) / 1e9,
        "speedup_vs_fp32": tf3 / tcm,
        "compressed_hbm_gb_s": rows * ns * 12 / (tcm * 1e-3) / 1e9,
        "fp32_hbm_gb_s": rows * ns * 16 / (tf3 * 1e-3) / 1e9,
        "dense_tflops": dense / (tcm * 1e-3) / 1e12,
        "sum_factorised": {"compressed": rows / (thc * 1e-3) / 1e9, "fp32": rows / (thf * 1e-3) / 1e9,
                           "compressed_hbm_gb_s": rows * ns * 12 / (thc * 1e-3) / 1e9,
                           "fp32_hbm_gb_s": rows * ns * 16 / (thf * 1e-3) / 1e9,
                           "note": "tensor-product hexahedron, 15 FMAs per output on CUDA cores"},
        "roofline": {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s",
                     "frac": ach / tf32_peak,
                     "note": "3xTF32: 3 tensor products per Alg.-1 product; peak = measured "
                             "tcgen05 tf32 issue rate (tools/umma_bench.cu)"}}
    del F, words, div, op
    torch.cuda.empty_cache()

    # sum-factorised kernels across degrees (same ~1.3 GB of words each):
    # where the compressed fluxes overtake the fp32 ones
    per_k = {}
    for kk in (1, 2, 3, 4):
        nsk = (kk + 1) ** 3
        ne = (n_el * 125) // nsk
        Fk = torch.rand((nsk, n_vars, ne, 3), device=dev, generator=gen).mul_(2).sub_(1)
        wk = vc3b.compress(Fk.reshape(-1, 3), lay, vc3b.ALL_SINGLE_POLICY).reshape(nsk, n_vars, ne)
        dk = torch.empty((nsk, n_vars, ne), dtype=torch.float32, device=dev)
        mk = np.ascontiguousarray(fr.lagrange_derivative_matrix(fr.gauss_legendre_nodes(kk)),
                                  dtype=np.float32)
        hck = lambda: lib.vc3_fr_divergence_hex(wk.data_ptr(), mk.ctypes.data, kk, dk.data_ptr(), ne,
                                                n_vars, ne, cl, stream.cuda_stream)
        hfk = lambda: lib.vc3_fr_divergence_hex_f32(Fk.data_ptr(), mk.ctypes.data, kk, dk.data_ptr(),
                                                    ne, n_vars, ne, stream.cuda_stream)
        hck(); hfk()
        torch.cuda.synchronize()
        tck, tfk = time_region(hck, steps, stream, torch), time_region(hfk, steps, stream, torch)
        rk_ = ne * n_vars
        per_k[str(kk)] = {"compressed": rk_ / (tck * 1e-3) / 1e9, "fp32": rk_ / (tfk * 1e-3) / 1e9,
                          "speedup": tfk / tck}
        del Fk, wk, dk
    out["C6_fr_divergence"]["sum_factorised"]["per_degree_g_elem_eq_s"] = per_k
    torch.cuda.empty_cache()
    return out


def run_gpu(args, world, rank, local):
    import torch

    import paper_2003_02633_b200 as vc3b
    from paper_2003_02633_b200 import _native

    # VC3_BENCH_SHARE_GPU=1: functional check of the multi-rank path on a
    # one-GPU box (ranks share cuda:0 over gloo; its timings are not results)
    share = os.environ.get("VC3_BENCH_SHARE_GPU") == "1"
    dev = torch.device("cuda", local % torch.cuda.device_count() if share else local)
    torch.cuda.set_device(dev)
    _native.load()
    lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
    if args.scaling == "strong":
        # C5: a fixed global problem split into contiguous shards
        from paper_2003_02633_b200.analysis import shard_range

        lo, hi = shard_range(args.total, rank, world)
        n = hi - lo
        global_n = args.total
    else:
        n = args.n
        global_n = n * world
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        on_gpu = dist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # synthetic shard: cube vectors generated on the device (counter-based
    # generator keyed by rank, so shards are independent), compressed once.
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    va = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    vb = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    a = vc3b.compress(va, lay, pol)
    b = vc3b.compress(vb, lay, pol)
    c = torch.empty_like(a)
    lib = _native.load()
    cl = _native.c_layout(lay)
    sptr = stream.cuda_stream

    def step_add(flags=0, out=None):
        lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), (out if out is not None else c).data_ptr(),
                                  n, cl, pol.mask, flags, sptr)

    rc = lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, cl, pol.mask, 0, sptr)
    _native.check(rc, "add_compressed")
    for _ in range(args.warmup):
        step_add()
    torch.cuda.synchronize()

    def timed(label_steps, fn=step_add):
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(dev.index) as clk:
            ms = time_region(fn, label_steps, stream, torch)
        torch.cuda.synchronize()
        barrier()
        return ms, clk.summary()

    ms, clocks = timed(args.steps)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    remeasured = False
    if bad & set(clocks["reasons"]):
        ms, clocks = timed(args.steps)
        remeasured = True
    ms_all = max_over_ranks(ms)
    value = global_n / (ms_all * 1e-3) / 1e9

    # the north-star tolerance mode (VC3_CONTRACT) on the same operands
    c_ct = torch.empty_like(a)
    step_ct = lambda: step_add(1, c_ct)
    for _ in range(args.warmup):
        step_ct()
    ms_ct, clocks_ct = timed(args.steps, step_ct)
    ms_ct_all = max_over_ranks(ms_ct)
    value_ct = global_n / (ms_ct_all * 1e-3) / 1e9
    step_add()  # c = the exact words again

    # uncompressed float32 baseline on the same GPU (same vectors, 36 B/vec)
    ra = va.reshape(-1)
    rb = vb.reshape(-1)
    rc_ = torch.empty_like(ra)

    def step_raw():
        lib.vc3_add_raw(ra.data_ptr(), rb.data_ptr(), rc_.data_ptr(), 3 * n, sptr)

    for _ in range(args.warmup):
        step_raw()
    torch.cuda.synchronize()
    barrier()
    raw_ms = max_over_ranks(time_region(step_raw, args.steps, stream, torch))
    raw_value = global_n / (raw_ms * 1e-3) / 1e9

    # secondary kernels: compress, decompress (both modes) and the fused axpy
    # y' = 0.75 x + y (24 B/vector, both modes), each with its roofline
    peak, peak_src = measured_peak()
    ns_ = min(n, N_PER_GPU)  # secondary kernels on (at most) one 2^28 shard
    out_v = torch.empty((ns_, 3), dtype=torch.float32, device=dev)
    y_out = torch.empty(ns_, dtype=torch.uint64, device=dev)

    def kline(t_ms, nbytes):
        gbs = nbytes * ns_ / (t_ms * 1e-3) / 1e9
        return {"gvec_s": ns_ / (t_ms * 1e-3) / 1e9, "gb_s": gbs, "frac_of_peak": gbs / peak, "ms": t_ms}

    sec = {"n_vectors": ns_}
    for name, fn, nbytes in (
            ("compress", lambda: lib.vc3_compress(va.data_ptr(), c.data_ptr(), ns_, cl, pol.mask, None, sptr), 20),
            ("decompress_exact", lambda: lib.vc3_decompress_ex(a.data_ptr(), out_v.data_ptr(), ns_, cl, 0, sptr), 20),
            ("decompress_contract", lambda: lib.vc3_decompress_ex(a.data_ptr(), out_v.data_ptr(), ns_, cl, 1, sptr), 20),
            ("axpy_exact", lambda: lib.vc3_axpy_ex(0.75, a.data_ptr(), b.data_ptr(), y_out.data_ptr(), ns_, cl,
                                                   pol.mask, 0, sptr), 24),
            ("axpy_contract", lambda: lib.vc3_axpy_ex(0.75, a.data_ptr(), b.data_ptr(), y_out.data_ptr(), ns_, cl,
                                                      pol.mask, 1, sptr), 24)):
        fn()
        torch.cuda.synchronize()
        sec[name] = kline(time_region(fn, max(3, args.steps // 5), stream, torch), nbytes)
    del out_v, y_out
    step_add()  # c was reused by the compress timing

    # parity at scale, in the measured run: the first 2^24 pairs of the timed
    # operands against the CPU oracle (C restatement of the reference path);
    # exact mode must match bit for bit, contract-mode differences are the ties
    parity = None
    if rank == 0:
        sys.path.insert(0, str(ROOT / "oracle"))
        import vc3_oracle

        ns = min(n, 1 << 24)
        ha_s, hb_s = a[:ns].cpu().numpy(), b[:ns].cpu().numpy()
        want = vc3_oracle.add_compressed(ha_s, hb_s, lay, pol, vc3_oracle.default_threads())
        got_ex, got_ct = c[:ns].cpu().numpy(), c_ct[:ns].cpu().numpy()
        parity = {"n_pairs": ns, "oracle": "oracle/vc3_oracle.c add_compressed (CPU)",
                  "exact_mismatches": int((got_ex != want).sum()),
                  "contract_ties": tie_stats(got_ct, want, lay)}
    del c_ct

    # e2e: public host-array API with the host<->device copies in the timed
    # region, from pinned buffers and from plain (pageable) numpy arrays; one
    # 2^28 shard at N = 1, a quarter of that per rank under torchrun
    e2e_n = min(n, N_PER_GPU if world == 1 else N_PER_GPU // 4)
    e2e_steps = max(1, min(args.steps, 5))
    pinned = [torch.empty(e2e_n, dtype=torch.uint64, pin_memory=True) for _ in range(3)]
    pinned[0].copy_(a[:e2e_n])
    pinned[1].copy_(b[:e2e_n])
    pin_np = [t.numpy() for t in pinned]
    page_np = [np.empty(e2e_n, dtype=np.uint64) for _ in range(3)]
    page_np[0][:] = pin_np[0]
    page_np[1][:] = pin_np[1]

    def e2e_time(bufs):
        def step():
            rc2 = lib.vc3_add_compressed_host(bufs[0].ctypes.data, bufs[1].ctypes.data, bufs[2].ctypes.data,
                                              e2e_n, cl, pol.mask, dev.index)
            _native.check(rc2, "add_compressed_host")
        step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            step()
        return max_over_ranks((time.perf_counter() - t0) / e2e_steps)

    e2e_s = e2e_time(pin_np)
    e2e_page_s = e2e_time(page_np)
    e2e_value = e2e_n * world / e2e_s / 1e9
    e2e_page_value = e2e_n * world / e2e_page_s / 1e9
    ref_c = c[:e2e_n].cpu().numpy()
    if not (np.array_equal(pin_np[2], ref_c) and np.array_equal(page_np[2], ref_c)):
        raise RuntimeError("host-API result differs from the device kernel result")
    del pinned, pin_np, page_np

    # secondary configs are single-GPU characterisations; scaling runs skip them
    secondary_configs = ({} if (args.no_secondary or world > 1)
                         else run_secondary(args, vc3b, lib, dev, stream, min(n, N_PER_GPU)))

    achieved = BYTES_COMPRESSED * n / (ms * 1e-3) / 1e9
    achieved_ct = BYTES_COMPRESSED * n / (ms_ct * 1e-3) / 1e9
    traffic = ncu_traffic()
    if rank != 0:
        return
    cpu = cpu_baseline_sample(args.cpu_sample) if world == 1 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_all, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(n, world, args.scaling, global_n),
        "mode": "exact (VC3_EXACT: output words bit-identical to the reference)",
        "hbm_gb_s": BYTES_COMPRESSED * global_n / (ms_all * 1e-3) / 1e9,
        "contract_mode": {
            "value": value_ct, "unit": UNIT, "ms_per_step": ms_ct_all,
            "hbm_gb_s": BYTES_COMPRESSED * global_n / (ms_ct_all * 1e-3) / 1e9,
            "roofline_frac": achieved_ct / peak,
            "speedup_vs_fp32_add": value_ct / raw_value,
            "ties": parity["contract_ties"] if parity else None,
            "clocks": {k: clocks_ct[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "definition": "VC3_CONTRACT: BASELINE.json north-star tolerance (decoded components "
                          "within 1 ulp of the reference decode, words bit-exact except one-bin ties)"},
        "parity_vs_oracle": parity,
        "fp32_add": {"value": raw_value, "unit": UNIT,
                     "hbm_gb_s": BYTES_RAW * global_n / (raw_ms * 1e-3) / 1e9,
                     "ms_per_step": raw_ms},
        "speedup_vs_fp32_add": value / raw_value,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "k_add_as<exact, default layout> (fused decompress-add-recompress)",
                     "algorithmic_bytes_per_launch": BYTES_COMPRESSED * n},
        "secondary_kernels": sec,
        "secondary_configs": secondary_configs,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * e2e_n,
                "d2h_bytes_per_step": 8 * e2e_n,
                "path": "vc3_add_compressed_host (C ABI; paper_2003_02633_b200.add_compressed "
                        "on numpy arrays), pinned host buffers, chunked H2D/kernel/D2H overlap",
                "pageable": {"value": e2e_page_value, "unit": UNIT,
                             "frac_of_pinned": e2e_page_value / e2e_value,
                             "path": "the same call on plain numpy (pageable) arrays"},
                "steps": e2e_steps},
        "gpu_launches": args.steps,
        "hbm_high_water_gib": torch.cuda.max_memory_allocated(dev) / 2 ** 30,
        "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "clock_samples": clocks["samples"],
        "remeasured": remeasured,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def tie_stats(got: np.ndarray, want: np.ndarray, lay) -> dict:
    """Words that differ from the oracle's: rate and the largest bucket /
    field deltas (theta wraps at +-pi)."""
    d = got != want
    t, p = lay.theta_bits, lay.phi_bits
    g, w = got[d].astype(np.int64), want[d].astype(np.int64)
    out = {"n": int(d.size), "n_diff": int(d.sum()), "rate": float(d.mean())}
    if d.any():
        tm, pm = (1 << t) - 1, (1 << p) - 1
        dt = np.abs((g & tm) - (w & tm))
        dt = np.minimum(dt, tm + 1 - dt)
        out.update(max_dn_theta=int(dt.max()),
                   max_dn_phi=int(np.abs(((g >> t) & pm) - ((w >> t) & pm)).max()),
                   max_dfield=int(np.abs((g >> (t + p)) - (w >> (t + p))).max()))
    else:
        out.update(max_dn_theta=0, max_dn_phi=0, max_dfield=0)
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", "--vectors", dest="n", type=int, default=N_PER_GPU,
                    help="vectors per GPU (--vectors under torchrun: its parser claims --n)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: --n vectors per GPU (C2); strong: --total split over GPUs (C5)")
    ap.add_argument("--total", type=int, default=1 << 31, help="global vectors for --scaling strong")
    ap.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE,
                    help="vectors per CPU-baseline / reference-arm step")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C3/C4 secondary configs (quick runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_gpu(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
