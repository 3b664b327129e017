"""ctypes binding of ``lib/libvc3_b200.so`` (the C ABI in include/vc3_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of any entry point raises ``ImportError`` with the build command.  The
signatures below are the single source of truth for the Python side and are
checked against the header by tests/test_boundary.py.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(os.environ.get("VC3_B200_LIB") or
                (Path(__file__).resolve().parent / "lib" / "libvc3_b200.so"))


class Layout(ctypes.Structure):
    """``vc3_layout`` (include/vc3_b200.h)."""

    _fields_ = [(name, ctypes.c_int32) for name in (
        "sign_bits", "exponent_bits", "mantissa_bits", "phi_bits", "theta_bits",
        "exponent_bias")]


class Variant(ctypes.Structure):
    """``vc3_variant`` (include/vc3_b200.h)."""

    _fields_ = [("kind", ctypes.c_int32), ("total_bits", ctypes.c_int32),
                ("n_phi_max", ctypes.c_int64), ("gamma", ctypes.c_double)]


VARIANT_UNIFORM, VARIANT_COSINE, VARIANT_TANH, VARIANT_SPLIT = 0, 1, 2, 3

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_f32 = ctypes.c_float

# name -> (argtypes, restype)
SIGNATURES = {
    "vc3_version": ([], ctypes.c_char_p),
    "vc3_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "vc3_last_cuda_error": ([], ctypes.c_int),
    "vc3_validate_layout": ([Layout], ctypes.c_int),
    "vc3_compress": ([_p, _p, _i64, Layout, _u32, _p, _p], ctypes.c_int),
    "vc3_decompress": ([_p, _p, _i64, Layout, _p], ctypes.c_int),
    "vc3_decompress_ex": ([_p, _p, _i64, Layout, _u32, _p], ctypes.c_int),
    "vc3_decode_tolerance": ([Layout, _p], ctypes.c_int),
    "vc3_prepare_layout": ([Layout, _u32], ctypes.c_int),
    "vc3_compress_events": ([_p, _p, _i64, Layout, _u32, _p, _p, _p], ctypes.c_int),
    "vc3_add_compressed": ([_p, _p, _p, _i64, Layout, _u32, _p], ctypes.c_int),
    "vc3_add_compressed_ex": ([_p, _p, _p, _i64, Layout, _u32, _u32, _p], ctypes.c_int),
    "vc3_add_raw": ([_p, _p, _p, _i64, _p], ctypes.c_int),
    "vc3_axpy": ([_f32, _p, _p, _p, _i64, Layout, _u32, _p], ctypes.c_int),
    "vc3_axpy_ex": ([_f32, _p, _p, _p, _i64, Layout, _u32, _u32, _p], ctypes.c_int),
    "vc3_rk_stage": ([_f32, _f32, _f32, _p, _p, _p, _i64, Layout, _u32, _p], ctypes.c_int),
    "vc3_rk_stage_ex": ([_f32, _f32, _f32, _p, _p, _p, _i64, Layout, _u32, _u32, _p], ctypes.c_int),
    "vc3_rk_stage_f32": ([_f32, _f32, _f32, _p, _p, _p, _i64, _p], ctypes.c_int),
    "vc3_to_spherical": ([_p, _p, _p, _p, _i64, _u32, _p, _p], ctypes.c_int),
    "vc3_quantize_angles": ([_p, _p, _p, _p, _i64, Layout, _u32, _p], ctypes.c_int),
    "vc3_dequantize_angles": ([_p, _p, _p, _p, _i64, Layout, _p], ctypes.c_int),
    "vc3_encode_magnitude": ([_p, _p, _i64, Layout, _p], ctypes.c_int),
    "vc3_decode_magnitude": ([_p, _p, _i64, Layout, _p], ctypes.c_int),
    "vc3_magnitude_events": ([_p, _i64, Layout, _p, _p], ctypes.c_int),
    "vc3_magnitude_events_checked": ([_p, _i64, Layout, _p, _p, _p], ctypes.c_int),
    "vc3_error_stats": ([_p, _p, _i64, _i32, _i64, _p, _p], ctypes.c_int),
    "vc3_error_stats_workspace": ([_i64, _i64, _p], ctypes.c_int),
    "vc3_error_stats_ws": ([_p, _p, _i64, _i32, _i64, _p, _p, ctypes.c_uint64, _p], ctypes.c_int),
    "vc3_compress_variant": ([_p, _p, _i64, Layout, Variant, _p, _p], ctypes.c_int),
    "vc3_decompress_variant": ([_p, _p, _i64, Layout, Variant, _p], ctypes.c_int),
    "vc3_variant_maxima": ([Layout, Variant, _p, _p], ctypes.c_int),
    "vc3_fr_operator_floats": ([ctypes.c_int], _i64),
    "vc3_fr_prepare_operator": ([_p, ctypes.c_int, _p, _p], ctypes.c_int),
    "vc3_fr_divergence": ([_p, _p, _p, _i64, ctypes.c_int, _i64, ctypes.c_int, Layout, _p], ctypes.c_int),
    "vc3_fr_divergence_f32": ([_p, _p, _p, _i64, ctypes.c_int, _i64, ctypes.c_int, _p], ctypes.c_int),
    "vc3_fr_divergence_hex": ([_p, _p, ctypes.c_int, _p, _i64, ctypes.c_int, _i64, Layout, _p], ctypes.c_int),
    "vc3_fr_divergence_hex_f32": ([_p, _p, ctypes.c_int, _p, _i64, ctypes.c_int, _i64, _p], ctypes.c_int),
    "vc3_add_compressed_host": ([_p, _p, _p, _i64, Layout, _u32, _i32], ctypes.c_int),
    "vc3_compress_host": ([_p, _p, _i64, Layout, _u32, _p, _i32], ctypes.c_int),
    "vc3_decompress_host": ([_p, _p, _i64, Layout, _i32], ctypes.c_int),
}

# numerics modes of the *_ex entry points (include/vc3_b200.h)
VC3_EXACT = 0
VC3_CONTRACT = 1
MODES = {"exact": VC3_EXACT, "contract": VC3_CONTRACT}


def mode_flag(mode: str) -> int:
    """``"exact"`` (bit-identical to the reference, the default) or
    ``"contract"`` (the north-star tolerance: one-ulp decodes, one-bin ties)."""
    try:
        return MODES[mode]
    except KeyError:
        raise ValueError(f"mode must be one of {sorted(MODES)}, got {mode!r}") from None

VC3_OK = 0
VC3_ERR_LAYOUT = -1
VC3_ERR_ARG = -2
VC3_ERR_CUDA = -3
VC3_ERR_NONFINITE = -4
VC3_ERR_LENGTH = -5

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) the CUDA library.  Raises ImportError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # VC3_B200_AUTOBUILD: unset -> build only when the library is missing;
    # "stale" -> also rebuild when a source is newer than it (development);
    # "0" -> never build
    autobuild = os.environ.get("VC3_B200_AUTOBUILD", "missing")
    if autobuild == "stale" and "VC3_B200_LIB" not in os.environ:
        from ._build import build

        build()
    if not LIB_PATH.exists():
        if autobuild != "0":
            from ._build import build

            build()
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (needs nvcc)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (argtypes, restype) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    _lib = lib
    return lib


def c_layout(layout) -> Layout:
    return Layout(*layout.as_c())


def check(status: int, what: str = "vc3") -> None:
    """Map a vc3_status onto the reference's exception classes."""
    if status == VC3_OK:
        return
    lib = load()
    text = lib.vc3_status_string(status).decode()
    if status == VC3_ERR_LAYOUT:
        raise errors.BadLayout(f"{what}: {text}")
    if status == VC3_ERR_NONFINITE:
        raise errors.NonFiniteInput(f"{what}: {text}")
    if status == VC3_ERR_LENGTH:
        raise errors.LengthMismatch(f"{what}: {text}")
    if status == VC3_ERR_CUDA:
        raise errors.DeviceError(f"{what}: {text} (cudaError {lib.vc3_last_cuda_error()})")
    raise ValueError(f"{what}: {text}")
