"""Drop-in codec API backed by the sm_100a kernels.

Same names, defaults, argument meaning, return shapes and exceptions as
/root/reference/pkg/src/vc3/codec.py (cited per function).  Operands may be
numpy-compatible host arrays (results are numpy, as in the reference) or CUDA
``torch.Tensor`` (results stay on the device, zero copy).

Word layout (normative, codec.py:1-8): MSB -> LSB the magnitude field
(sign bit if present, exponent, mantissa), then n_phi, then n_theta.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np

from . import _dev, _native
from ._dev import torch
from .errors import NonFiniteInput
from .layout import DEFAULT_LAYOUT, DEFAULT_POLICY, BitLayout, PrecisionPolicy, as_layout, as_policy  # noqa: F401

__all__ = [
    "SphericalTriple",
    "nint",
    "to_spherical",
    "to_spherical_one",
    "quantize_angles",
    "dequantize_angles",
    "encode_magnitude",
    "decode_magnitude",
    "compress",
    "decompress",
    "compress_one",
    "decompress_one",
    "magnitude_event_counts",
    "predict_error",
]


class SphericalTriple(NamedTuple):
    r: float
    theta: float
    phi: float


def _nonfinite_message(bad: int) -> str:
    return f"{bad} vector(s) contain NaN or infinity"


# ---------------------------------------------------------------------------
# operand normalisation (codec.py:70-83 shape rules)
# ---------------------------------------------------------------------------
def _host_vectors(vectors) -> np.ndarray:
    v = np.asarray(vectors, dtype=np.float32)
    if v.ndim == 1 and v.shape[0] == 3:
        v = v.reshape(1, 3)
    if v.ndim != 2 or v.shape[1] != 3:
        raise ValueError(f"expected shape (n, 3), got {v.shape}")
    return np.ascontiguousarray(v)


def _device_vectors(vectors):
    v = vectors if vectors.dtype == torch.float32 else vectors.to(torch.float32)
    if v.dim() == 1 and v.shape[0] == 3:
        v = v.reshape(1, 3)
    if v.dim() != 2 or v.shape[1] != 3:
        raise ValueError(f"expected shape (n, 3), got {tuple(v.shape)}")
    return v.contiguous()


def _device_words(words):
    w = words
    if w.dtype not in (torch.uint64, torch.int64):
        w = w.to(torch.int64)
    return w.reshape(-1).contiguous()


# ---------------------------------------------------------------------------
# hot path
# ---------------------------------------------------------------------------
def compress(vectors, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY):
    """Pack each float32 3-vector into one 64-bit word (codec.py:189-202).

    Raises NonFiniteInput if any component is NaN or infinite (checked inside
    the kernel; on the device path the check synchronises the stream)."""
    layout, policy = as_layout(layout), as_policy(policy)
    lib = _native.load()
    if _dev.is_device(vectors):
        v = _device_vectors(vectors)
        n = v.shape[0]
        out = torch.empty(n, dtype=torch.uint64, device=v.device)
        bad = torch.zeros(1, dtype=torch.int32, device=v.device)
        _native.check(lib.vc3_compress(v.data_ptr(), out.data_ptr(), n, _native.c_layout(layout),
                                       policy.mask, bad.data_ptr(), _dev.stream_of(v)),
                      "compress")
        nbad = int(bad.item())
        if nbad:
            raise NonFiniteInput(_nonfinite_message(nbad))
        return out
    v = _host_vectors(vectors)
    out = np.empty(v.shape[0], dtype=np.uint64)
    nbad = ctypes.c_int64(0)
    st = lib.vc3_compress_host(v.ctypes.data, out.ctypes.data, v.shape[0],
                               _native.c_layout(layout), policy.mask, ctypes.addressof(nbad),
                               _dev.device_ordinal())
    if st == _native.VC3_ERR_NONFINITE:
        raise NonFiniteInput(_nonfinite_message(nbad.value))
    _native.check(st, "compress")
    return out


def compress_with_events(vectors, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY):
    """``(compress(vectors), magnitude_event_counts(vectors))`` in one pass over
    the input (the event counters fused into the compress kernel).
    Host arrays are uploaded once; the words come back to the host."""
    layout, policy = as_layout(layout), as_policy(policy)
    lib = _native.load()
    host = not _dev.is_device(vectors)
    if host:
        hv = _host_vectors(vectors)
        if hv.shape[0] == 0:
            return np.empty(0, dtype=np.uint64), (0, 0)
        v = _dev.upload(hv)
    else:
        v = _device_vectors(vectors)
    n = v.shape[0]
    out = torch.empty(n, dtype=torch.uint64, device=v.device)
    bad = torch.zeros(1, dtype=torch.int32, device=v.device)
    ev = torch.zeros(2, dtype=torch.int64, device=v.device)
    _native.check(lib.vc3_compress_events(v.data_ptr(), out.data_ptr(), n, _native.c_layout(layout),
                                          policy.mask, bad.data_ptr(), ev.data_ptr(),
                                          _dev.stream_of(v)), "compress_events")
    nbad = int(bad.item())
    if nbad:
        raise NonFiniteInput(_nonfinite_message(nbad))
    counts = ev.cpu().tolist()
    return (_dev.download(out) if host else out), (int(counts[0]), int(counts[1]))


def decompress(words, layout=DEFAULT_LAYOUT, mode="exact"):
    """Reconstruct (n, 3) float32 vectors from packed words (codec.py:205-228).

    Every word decodes to a finite vector; a zero magnitude field decodes to
    (0, 0, 0) whatever the angle bits.  ``mode="exact"`` (default) is
    bit-identical to the reference's decode; ``mode="contract"`` skips the
    boundary re-evaluation (each component the reference's float32 or one ulp
    from it)."""
    layout = as_layout(layout)
    flags = _native.mode_flag(mode)
    lib = _native.load()
    if _dev.is_device(words):
        w = _device_words(words)
        n = w.shape[0]
        out = torch.empty((n, 3), dtype=torch.float32, device=w.device)
        with _dev.on_device(w):
            _native.check(lib.vc3_decompress_ex(w.data_ptr(), out.data_ptr(), n,
                                                _native.c_layout(layout), flags,
                                                _dev.stream_of(w)), "decompress")
        return out
    if flags:
        return _dev.download(decompress(_dev.upload(np.asarray(words, dtype=np.uint64).ravel()),
                                        layout, mode))
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).ravel())
    out = np.empty((w.size, 3), dtype=np.float32)
    _native.check(lib.vc3_decompress_host(w.ctypes.data, out.ctypes.data, w.size,
                                          _native.c_layout(layout), _dev.device_ordinal()),
                  "decompress")
    return out


def compress_one(v, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY) -> int:
    """codec.py:231-233"""
    return int(compress(np.asarray(v, dtype=np.float32).reshape(1, 3), layout, policy)[0])


def decompress_one(word: int, layout=DEFAULT_LAYOUT):
    """codec.py:236-238"""
    v = decompress(np.asarray([word], dtype=np.uint64), layout)[0]
    return float(v[0]), float(v[1]), float(v[2])


# ---------------------------------------------------------------------------
# pieces (codec.py:86-186): same kernels' building blocks, one launch each
# ---------------------------------------------------------------------------
def _scalar_in(x) -> bool:
    return np.isscalar(x) or np.asarray(x).ndim == 0


def nint(x):
    """Round to nearest, halves toward +inf: ceil(floor(2x)/2) (codec.py:86-96).
    A host helper, as in the reference (the kernels inline the same rule)."""
    a = np.asarray(x, dtype=np.float64)
    out = np.ceil(np.floor(2.0 * a) / 2.0)
    if np.isscalar(x) or a.ndim == 0:
        return int(out)
    return out.astype(np.int64)


def to_spherical(vectors, policy=DEFAULT_POLICY):
    """(r, theta, phi) in float64 under the policy's precisions
    (codec.py:99-114)."""
    policy = as_policy(policy)
    lib = _native.load()
    host = not _dev.is_device(vectors)
    v = _dev.upload(_host_vectors(vectors)) if host else _device_vectors(vectors)
    n = v.shape[0]
    r, th, ph = (torch.empty(n, dtype=torch.float64, device=v.device) for _ in range(3))
    bad = torch.zeros(1, dtype=torch.int32, device=v.device)
    _native.check(lib.vc3_to_spherical(v.data_ptr(), r.data_ptr(), th.data_ptr(), ph.data_ptr(),
                                       n, policy.mask, bad.data_ptr(), _dev.stream_of(v)),
                  "to_spherical")
    nbad = int(bad.item())
    if nbad:
        raise NonFiniteInput(_nonfinite_message(nbad))
    if host:
        return _dev.download(r), _dev.download(th), _dev.download(ph)
    return r, th, ph


def to_spherical_one(v, policy=DEFAULT_POLICY) -> SphericalTriple:
    r, th, ph = to_spherical(np.asarray(v, dtype=np.float32).reshape(1, 3), policy)
    return SphericalTriple(float(r[0]), float(th[0]), float(ph[0]))


def quantize_angles(theta, phi, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY):
    """Bucket indices (n_theta, n_phi), clamped to [0, n_max]
    (codec.py:122-140)."""
    layout, policy = as_layout(layout), as_policy(policy)
    lib = _native.load()
    if _dev.is_device(theta):
        th = theta.to(torch.float64).reshape(-1).contiguous()
        ph = phi.to(device=theta.device, dtype=torch.float64).reshape(-1).contiguous()
        if th.shape != ph.shape:
            raise ValueError("theta and phi must have the same shape")
        nt, nph = (torch.empty(th.shape[0], dtype=torch.int64, device=th.device) for _ in range(2))
        _native.check(lib.vc3_quantize_angles(th.data_ptr(), ph.data_ptr(), nt.data_ptr(),
                                              nph.data_ptr(), th.shape[0],
                                              _native.c_layout(layout), policy.mask,
                                              _dev.stream_of(th)), "quantize_angles")
        return nt.reshape(theta.shape), nph.reshape(theta.shape)
    th = np.atleast_1d(np.asarray(theta, dtype=np.float64))
    ph = np.atleast_1d(np.asarray(phi, dtype=np.float64))
    if th.shape != ph.shape:
        raise ValueError("theta and phi must have the same shape")
    dth, dph = _dev.upload(th.ravel()), _dev.upload(ph.ravel())
    nt, nph = (torch.empty(th.size, dtype=torch.int64, device=dth.device) for _ in range(2))
    _native.check(lib.vc3_quantize_angles(dth.data_ptr(), dph.data_ptr(), nt.data_ptr(),
                                          nph.data_ptr(), th.size, _native.c_layout(layout),
                                          policy.mask, _dev.stream_of(dth)), "quantize_angles")
    nt, nph = _dev.download(nt), _dev.download(nph)
    if _scalar_in(theta):
        return int(nt[0]), int(nph[0])
    return nt.reshape(th.shape), nph.reshape(ph.shape)


def dequantize_angles(n_theta, n_phi, layout=DEFAULT_LAYOUT):
    """theta_hat = pi*(2n/n_max - 1), phi_hat = pi*n/n_max (codec.py:143-153)."""
    layout = as_layout(layout)
    lib = _native.load()
    nt = np.atleast_1d(np.asarray(n_theta, dtype=np.int64))
    nph = np.atleast_1d(np.asarray(n_phi, dtype=np.int64))
    dnt, dnp = _dev.upload(nt.ravel()), _dev.upload(nph.ravel())
    th = torch.empty(nt.size, dtype=torch.float64, device=dnt.device)
    ph = torch.empty(nph.size, dtype=torch.float64, device=dnt.device)
    _native.check(lib.vc3_dequantize_angles(dnt.data_ptr(), dnp.data_ptr(), th.data_ptr(),
                                            ph.data_ptr(), nt.size, _native.c_layout(layout),
                                            _dev.stream_of(dnt)), "dequantize_angles")
    th, ph = _dev.download(th), _dev.download(ph)
    if _scalar_in(n_theta):
        return float(th[0]), float(ph[0])
    return th.reshape(nt.shape), ph.reshape(nph.shape)


def encode_magnitude(r, layout=DEFAULT_LAYOUT):
    """Magnitude field bits of non-negative radii (codec.py:156-175): narrow
    to float32 rounding up, truncate the mantissa, flush / saturate at the
    rails; zero encodes to the all-zeros field."""
    layout = as_layout(layout)
    lib = _native.load()
    a = np.atleast_1d(np.asarray(r, dtype=np.float64))
    if not np.isfinite(a).all():
        raise NonFiniteInput("magnitude must be finite")
    if (a < 0).any():
        raise ValueError("magnitude must be non-negative")
    da = _dev.upload(a.ravel())
    out = torch.empty(a.size, dtype=torch.uint64, device=da.device)
    _native.check(lib.vc3_encode_magnitude(da.data_ptr(), out.data_ptr(), a.size,
                                           _native.c_layout(layout), _dev.stream_of(da)),
                  "encode_magnitude")
    out = _dev.download(out)
    if _scalar_in(r):
        return int(out[0])
    return out.reshape(a.shape)


def decode_magnitude(field, layout=DEFAULT_LAYOUT):
    """float32 radius of a magnitude field; zero decodes to 0 (codec.py:178-186)."""
    layout = as_layout(layout)
    lib = _native.load()
    f = np.atleast_1d(np.asarray(field).astype(np.int64))
    df = _dev.upload(f.ravel())
    out = torch.empty(f.size, dtype=torch.float32, device=df.device)
    _native.check(lib.vc3_decode_magnitude(df.data_ptr(), out.data_ptr(), f.size,
                                           _native.c_layout(layout), _dev.stream_of(df)),
                  "decode_magnitude")
    out = _dev.download(out)
    if _scalar_in(field):
        return float(out[0])
    return out.reshape(f.shape)


def magnitude_event_counts(vectors, layout=DEFAULT_LAYOUT):
    """(flushed, saturated) vector counts (codec.py:241-262)."""
    layout = as_layout(layout)
    lib = _native.load()
    host = not _dev.is_device(vectors)
    if host:
        hv = _host_vectors(vectors)
        if not np.isfinite(hv).all():
            bad = int(np.count_nonzero(~np.isfinite(hv).all(axis=1)))
            raise NonFiniteInput(_nonfinite_message(bad))
        v = _dev.upload(hv)
    else:
        v = _device_vectors(vectors)
    counts = torch.zeros(2, dtype=torch.int64, device=v.device)
    nonfinite = torch.zeros(1, dtype=torch.int32, device=v.device)
    with _dev.on_device(v):
        _native.check(lib.vc3_magnitude_events_checked(v.data_ptr(), v.shape[0],
                                                       _native.c_layout(layout), counts.data_ptr(),
                                                       nonfinite.data_ptr(), _dev.stream_of(v)),
                      "magnitude_event_counts")
    bad = int(nonfinite.item())
    if bad:
        raise NonFiniteInput(_nonfinite_message(bad))
    c = counts.cpu().tolist()
    return int(c[0]), int(c[1])


def predict_error(r, theta, phi, layout=DEFAULT_LAYOUT):
    """First-order worst-case error-bound vector (codec.py:265-283).  A
    test-oracle envelope on the host, as in the reference, not a codec path."""
    layout = as_layout(layout)
    r = np.asarray(r, dtype=np.float64)
    th = np.asarray(theta, dtype=np.float64)
    ph = np.asarray(phi, dtype=np.float64)
    e_t = np.pi / layout.n_theta_max
    e_p = np.pi / (2.0 * layout.n_phi_max)
    st, ct = np.sin(th), np.cos(th)
    sp, cp = np.sin(ph), np.cos(ph)
    ex = r * (e_p * np.abs(ct * cp) + e_t * np.abs(st * sp))
    ey = r * (e_p * np.abs(st * cp) + e_t * np.abs(ct * sp))
    ez = r * e_p * np.abs(sp)
    return np.stack(np.broadcast_arrays(ex, ey, ez), axis=-1)
