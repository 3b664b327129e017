"""K7: companded and fractionally split angle coding on the GPU.

Mirrors /root/reference/pkg/src/vc3/analysis.py:259-417:

* ``SplitConfig``, ``joint_encode``, ``joint_decode``, ``_quantize_free``
  (analysis.py:259-306) and ``Compander``, ``compand``, ``compand_inverse``
  (analysis.py:342-393) keep the reference's names, validation and numpy
  semantics for the scalar / index helpers;
* ``compress_variant`` / ``decompress_variant`` run the whole variant round
  trip in CUDA (``vc3_compress_variant`` / ``vc3_decompress_variant``) with
  the word formats of include/vc3_b200.h;
* ``compand_study`` and ``split_sweep`` (analysis.py:309-337, 396-417) are
  the reference's studies on that device path plus the K6 statistics kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _native
from ._dev import torch
from .errors import EmptyDomain, InvalidSplit, NonFiniteInput
from .layout import DEFAULT_LAYOUT, as_layout

# ---------------------------------------------------------------------------
# fractional splitting (analysis.py:259-306)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SplitConfig:
    """Joint angle code J = n_phi*(n_theta_max+1) + n_theta in ``total_bits``."""

    total_bits: int
    n_phi_max: int
    n_theta_max: int = field(init=False)

    def __post_init__(self):
        if not 2 <= self.total_bits <= 62:
            raise InvalidSplit(f"total_bits {self.total_bits} out of range")
        if self.n_phi_max < 1:
            raise InvalidSplit("n_phi_max must be >= 1")
        capacity = 1 << self.total_bits
        theta_buckets = capacity // (self.n_phi_max + 1)
        if theta_buckets < 2:
            raise InvalidSplit(f"n_phi_max {self.n_phi_max} leaves no room for theta in "
                               f"{self.total_bits} bits")
        object.__setattr__(self, "n_theta_max", theta_buckets - 1)
        if (self.n_phi_max + 1) * (self.n_theta_max + 1) - 1 >= capacity:
            raise InvalidSplit("joint index exceeds capacity")


def joint_encode(n_theta, n_phi, cfg: SplitConfig):
    nt = np.asarray(n_theta, dtype=np.int64)
    nph = np.asarray(n_phi, dtype=np.int64)
    if (nt < 0).any() or (nt > cfg.n_theta_max).any():
        raise InvalidSplit("n_theta out of range for split")
    if (nph < 0).any() or (nph > cfg.n_phi_max).any():
        raise InvalidSplit("n_phi out of range for split")
    return nph * (cfg.n_theta_max + 1) + nt


def joint_decode(n_joint, cfg: SplitConfig):
    joint = np.asarray(n_joint, dtype=np.int64)
    width = cfg.n_theta_max + 1
    return joint % width, joint // width


def _quantize_free(th, ph, ntmax: int, npmax: int):
    """Codec bucket arithmetic for arbitrary bin counts (analysis.py:300-306)."""
    vt = ntmax / 2.0 + th * (ntmax / (2.0 * np.pi))
    vp = ph * (npmax / np.pi)
    nt = np.ceil(np.floor(2.0 * vt) / 2.0).astype(np.int64)
    nph = np.ceil(np.floor(2.0 * vp) / 2.0).astype(np.int64)
    return np.clip(nt, 0, ntmax), np.clip(nph, 0, npmax)


# ---------------------------------------------------------------------------
# companding (analysis.py:342-393)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Compander:
    """Monotone map of a normalised angle psi in [0, 1] before uniform binning:
    uniform, cosine n_max*(1-cos(pi psi))/2, or tanh
    m*n_max*(tanh(gamma*(2 psi-1)) + c), c = tanh(gamma), m = 1/(2c)."""

    kind: str = "uniform"
    gamma: float = 0.5

    def __post_init__(self):
        if self.kind not in ("uniform", "cosine", "tanh"):
            raise ValueError(f"unknown compander {self.kind!r}")
        if self.kind == "tanh" and self.gamma <= 0:
            raise ValueError("tanh compander needs gamma > 0")

    def encode(self, psi, n_max: int):
        psi = np.asarray(psi, dtype=np.float64)
        if self.kind == "uniform":
            raw = psi * n_max
        elif self.kind == "cosine":
            raw = n_max * (1.0 - np.cos(np.pi * psi)) / 2.0
        else:
            c = math.tanh(self.gamma)
            m = 1.0 / (2.0 * c)
            raw = m * n_max * (np.tanh(self.gamma * (2.0 * psi - 1.0)) + c)
        n = np.ceil(np.floor(2.0 * raw) / 2.0).astype(np.int64)
        return np.clip(n, 0, n_max)

    def decode(self, n, n_max: int):
        n = np.asarray(n, dtype=np.float64)
        if self.kind == "uniform":
            return n / n_max
        if self.kind == "cosine":
            return np.arccos(np.clip(1.0 - 2.0 * n / n_max, -1.0, 1.0)) / np.pi
        c = math.tanh(self.gamma)
        m = 1.0 / (2.0 * c)
        u = np.clip(n / (m * n_max) - c, -c, c)
        return np.clip((np.arctanh(u) / self.gamma + 1.0) / 2.0, 0.0, 1.0)


def compand(psi, compander: Compander, n_max: int):
    return compander.encode(psi, n_max)


def compand_inverse(n, compander: Compander, n_max: int):
    return compander.decode(n, n_max)


# ---------------------------------------------------------------------------
# device word formats
# ---------------------------------------------------------------------------
_KIND = {"uniform": _native.VARIANT_UNIFORM, "cosine": _native.VARIANT_COSINE,
         "tanh": _native.VARIANT_TANH}


def c_variant(variant, layout) -> _native.Variant:
    """``vc3_variant`` for a Compander or a SplitConfig."""
    if isinstance(variant, SplitConfig):
        if variant.total_bits != layout.phi_bits + layout.theta_bits:
            raise InvalidSplit(f"split total_bits {variant.total_bits} must equal the layout's "
                               f"angle bits {layout.phi_bits + layout.theta_bits}")
        return _native.Variant(_native.VARIANT_SPLIT, variant.total_bits, variant.n_phi_max, 0.0)
    if isinstance(variant, Compander):
        return _native.Variant(_KIND[variant.kind], 0, 0, float(variant.gamma))
    raise TypeError(f"not a variant: {variant!r}")


def compress_variant(vectors, variant, layout=DEFAULT_LAYOUT):
    """Variant words of float32 (n, 3) vectors (numpy or CUDA tensor)."""
    from .codec import _device_vectors, _host_vectors, _nonfinite_message

    layout = as_layout(layout)
    lib = _native.load()
    host = not _dev.is_device(vectors)
    v = _dev.upload(_host_vectors(vectors)) if host else _device_vectors(vectors)
    out = torch.empty(v.shape[0], dtype=torch.uint64, device=v.device)
    bad = torch.zeros(1, dtype=torch.int32, device=v.device)
    _native.check(lib.vc3_compress_variant(v.data_ptr(), out.data_ptr(), v.shape[0],
                                           _native.c_layout(layout), c_variant(variant, layout),
                                           bad.data_ptr(), _dev.stream_of(v)), "compress_variant")
    nbad = int(bad.item())
    if nbad:
        raise NonFiniteInput(_nonfinite_message(nbad))
    return _dev.download(out) if host else out


def decompress_variant(words, variant, layout=DEFAULT_LAYOUT):
    """(n, 3) float32 vectors from variant words (numpy or CUDA tensor)."""
    layout = as_layout(layout)
    lib = _native.load()
    host = not _dev.is_device(words)
    w = (_dev.upload(np.ascontiguousarray(np.asarray(words, dtype=np.uint64).ravel())) if host
         else words.reshape(-1).contiguous())
    out = torch.empty((w.shape[0], 3), dtype=torch.float32, device=w.device)
    _native.check(lib.vc3_decompress_variant(w.data_ptr(), out.data_ptr(), w.shape[0],
                                             _native.c_layout(layout), c_variant(variant, layout),
                                             _dev.stream_of(w)), "decompress_variant")
    return _dev.download(out) if host else out


def variant_maxima(variant, layout=DEFAULT_LAYOUT) -> tuple[int, int]:
    """(n_theta_max, n_phi_max) of the variant's buckets."""
    import ctypes

    layout = as_layout(layout)
    nt, nph = ctypes.c_int64(), ctypes.c_int64()
    _native.check(_native.load().vc3_variant_maxima(_native.c_layout(layout),
                                                    c_variant(variant, layout),
                                                    ctypes.addressof(nt), ctypes.addressof(nph)),
                  "variant_maxima")
    return nt.value, nph.value


# ---------------------------------------------------------------------------
# studies on the device path
# ---------------------------------------------------------------------------
def _variant_study(domain, variant, layout, normalised=False):
    from .analysis import CHUNK, ChunkMerger, chunk_moments

    acc = ChunkMerger()
    for i in range(domain.n_chunks()):
        v = _dev.upload(domain.chunk(i, domain.chunk_size(i)))
        vh = decompress_variant(compress_variant(v, variant, layout), variant, layout)
        c = chunk_moments(v, vh, normalised, CHUNK)[0].cpu().numpy()
        acc.add(int(c[0]), float(c[1]), float(c[2]), float(c[3]))
    return acc.stats(normalised)


def compand_study(domain, compander: Compander, layout=DEFAULT_LAYOUT):
    """Round-trip error with both angles companded before binning
    (analysis.py:396-417)."""
    if domain.count == 0:
        raise EmptyDomain("compand_study needs at least one sample")
    return _variant_study(domain, compander, as_layout(layout))


def split_sweep(total_bits: int, splits, domain, layout=DEFAULT_LAYOUT):
    """Round-trip error for each joint-coding split (analysis.py:309-337)."""
    if domain.count == 0:
        raise EmptyDomain("split_sweep needs at least one sample")
    layout = as_layout(layout)
    configs = [SplitConfig(total_bits, int(s) - 1) for s in splits]
    return [(cfg, _variant_study(domain, cfg, layout)) for cfg in configs]
