"""ctypes front end for the CPU restatement in ``vc3_oracle.c``.

TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  Callers
allowed to import this module: ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference``).  The product package
``paper_2003_02633_b200`` never imports it.

The functions mirror the reference's batch API (``vc3.codec.compress`` /
``decompress``, ``vc3.bench.add_compressed`` / ``add_raw``;
/root/reference/pkg/src/vc3/codec.py:189-228, bench.py:30-69) on numpy arrays.
Layouts are passed as any object with the reference's BitLayout attribute
names, policies as anything with ``theta_single``/``phi_single``/``quant_single``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libvc3_oracle.so"
_lib = None

_i64 = ctypes.c_int64
_int = ctypes.c_int
_p = ctypes.c_void_p


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = _HERE / "vc3_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE), "libvc3_oracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.vc3o_compress.argtypes = [_p, _p, _i64] + [_int] * 9
        L.vc3o_decompress.argtypes = [_p, _p, _i64] + [_int] * 6
        L.vc3o_add_compressed.argtypes = [_p, _p, _p, _i64] + [_int] * 9
        L.vc3o_add_raw.argtypes = [_p, _p, _p, _i64, _int]
        L.vc3o_axpy.argtypes = [ctypes.c_float, _p, _p, _p, _i64] + [_int] * 9
        L.vc3o_spherical.argtypes = [_p, _p, _p, _p, _i64, _int, _int]
        L.vc3o_quantize.argtypes = [_p, _p, _p, _p, _i64, _i64, _i64, _int]
        L.vc3o_encode_mag_batch.argtypes = [_p, _p, _i64, _int, _int, _int]
        L.vc3o_decode_mag_batch.argtypes = [_p, _p, _i64, _int, _int, _int]
        L.vc3o_angle_tables.argtypes = [_int, _int, _p, _p, _p, _p]
        L.vc3o_atan2_f32.argtypes = [ctypes.c_float, ctypes.c_float]
        L.vc3o_atan2_f32.restype = ctypes.c_float
        L.vc3o_acos_f32.argtypes = [ctypes.c_float]
        L.vc3o_acos_f32.restype = ctypes.c_float
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _lay(layout):
    return (layout.exponent_bits, layout.mantissa_bits, layout.phi_bits,
            layout.theta_bits, layout.exponent_bias)


def _pol(policy):
    return (int(policy.theta_single), int(policy.phi_single), int(policy.quant_single))


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def compress(vectors, layout, policy, nthreads: int = 1) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(vectors, dtype=np.float32).reshape(-1, 3))
    out = np.empty(v.shape[0], dtype=np.uint64)
    lib().vc3o_compress(_ptr(v), _ptr(out), v.shape[0], *_lay(layout), *_pol(policy), nthreads)
    return out


def decompress(words, layout, nthreads: int = 1) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).ravel())
    out = np.empty((w.size, 3), dtype=np.float32)
    lib().vc3o_decompress(_ptr(w), _ptr(out), w.size, *_lay(layout), nthreads)
    return out


def add_compressed(a, b, layout, policy, nthreads: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    assert a.shape == b.shape
    c = np.empty_like(a)
    lib().vc3o_add_compressed(_ptr(a), _ptr(b), _ptr(c), a.size, *_lay(layout), *_pol(policy),
                              nthreads)
    return c


def add_raw(a, b, nthreads: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    assert a.shape == b.shape
    c = np.empty_like(a)
    lib().vc3o_add_raw(_ptr(a), _ptr(b), _ptr(c), a.size, nthreads)
    return c


def axpy(alpha, x, y, layout, policy, nthreads: int = 1) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.ascontiguousarray(y, dtype=np.uint64)
    out = np.empty_like(y)
    lib().vc3o_axpy(float(np.float32(alpha)), _ptr(x), _ptr(y), _ptr(out), x.size,
                    *_lay(layout), *_pol(policy), nthreads)
    return out


def to_spherical(vectors, policy):
    v = np.ascontiguousarray(np.asarray(vectors, dtype=np.float32).reshape(-1, 3))
    n = v.shape[0]
    r, th, ph = np.empty(n), np.empty(n), np.empty(n)
    lib().vc3o_spherical(_ptr(v), _ptr(r), _ptr(th), _ptr(ph), n,
                         int(policy.theta_single), int(policy.phi_single))
    return r, th, ph


def quantize_angles(theta, phi, layout, policy):
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).ravel())
    ph = np.ascontiguousarray(np.asarray(phi, dtype=np.float64).ravel())
    nt = np.empty(th.size, dtype=np.int64)
    nph = np.empty(th.size, dtype=np.int64)
    lib().vc3o_quantize(_ptr(th), _ptr(ph), _ptr(nt), _ptr(nph), th.size,
                        (1 << layout.theta_bits) - 1, (1 << layout.phi_bits) - 1,
                        int(policy.quant_single))
    return nt, nph


def encode_magnitude(r, layout) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(r, dtype=np.float64).ravel())
    out = np.empty(a.size, dtype=np.int64)
    lib().vc3o_encode_mag_batch(_ptr(a), _ptr(out), a.size, layout.exponent_bits,
                                layout.mantissa_bits, layout.exponent_bias)
    return out


def decode_magnitude(field, layout) -> np.ndarray:
    f = np.ascontiguousarray(np.asarray(field).astype(np.int64).ravel())
    out = np.empty(f.size, dtype=np.float32)
    lib().vc3o_decode_mag_batch(_ptr(f), _ptr(out), f.size, layout.exponent_bits,
                                layout.mantissa_bits, layout.exponent_bias)
    return out


def angle_tables(t: int, p: int):
    """The reference's libm sin/cos tables (_kernels.py:252-273)."""
    st, ct = np.empty(1 << t), np.empty(1 << t)
    sp, cp = np.empty(1 << p), np.empty(1 << p)
    lib().vc3o_angle_tables(t, p, _ptr(st), _ptr(ct), _ptr(sp), _ptr(cp))
    return st, ct, sp, cp


def atan2_f32(y, x) -> np.float32:
    return np.float32(lib().vc3o_atan2_f32(float(np.float32(y)), float(np.float32(x))))


def acos_f32(w) -> np.float32:
    return np.float32(lib().vc3o_acos_f32(float(np.float32(w))))
