"""Flux-reconstruction flux divergence on compressed fluxes.

The paper's Algorithm 1 (step 10 of its FR table): for each
element ``i`` and equation ``c`` the divergence at solution point ``k`` is

    div[k, c, i] = sum_j sum_d D[d*ns + j, k] * decompress(F[j, c, i])[d]

with ``D`` the (3 ns x ns) divergence operator and the flux row of each
equation stored as one compressed word per solution point.
The reference package has no code for it; the kernel (``csrc/vc3_fr.cu``)
decodes the words straight into the A operand of a tcgen05 TF32 GEMM with
fp32-accurate operand splitting.  Storage follows the flux-reconstruction
convention (PyFR-style, element index fastest): words ``[ns][n_vars][ld]``,
fluxes ``[ns][n_vars][ld][3]``, divergence ``[ns][n_vars][ld]``.

``divergence_operator(k)`` builds D for a hexahedral element with the
tensor product of k+1 Gauss-Legendre points per direction (the paper's
solution points), in reference coordinates.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from ._dev import torch
from .errors import LengthMismatch
from .layout import DEFAULT_LAYOUT, as_layout


def gauss_legendre_nodes(k: int) -> np.ndarray:
    return np.polynomial.legendre.leggauss(k + 1)[0]


def lagrange_derivative_matrix(nodes: np.ndarray) -> np.ndarray:
    """M[a, m] = l_m'(x_a) for the Lagrange basis on ``nodes`` (float64)."""
    x = np.asarray(nodes, dtype=np.float64)
    n = x.size
    w = np.array([1.0 / np.prod([x[m] - x[q] for q in range(n) if q != m]) for m in range(n)])
    M = np.zeros((n, n))
    for a in range(n):
        for m in range(n):
            if a != m:
                M[a, m] = (w[m] / w[a]) / (x[a] - x[m])
        M[a, a] = -M[a].sum()
    return M


def divergence_operator(k: int, dtype=np.float32) -> np.ndarray:
    """(3 ns, ns) operator of a degree-k hexahedron, ns = (k+1)^3, point index
    ``p = ix + (k+1) iy + (k+1)^2 iz``: D[d*ns + j, p] = d l_j / d xi_d at p."""
    n = k + 1
    M = lagrange_derivative_matrix(gauss_legendre_nodes(k))
    eye = np.eye(n)
    ns = n ** 3
    # D_d[p, j] in (iz, iy, ix) Kronecker order: x derivative acts on ix
    dx = np.kron(eye, np.kron(eye, M))
    dy = np.kron(eye, np.kron(M, eye))
    dz = np.kron(M, np.kron(eye, eye))
    D = np.concatenate([dx.T, dy.T, dz.T], axis=0)
    assert D.shape == (3 * ns, ns)
    return D.astype(dtype)


def solution_points(k: int) -> np.ndarray:
    """(ns, 3) reference coordinates of the solution points, same ordering."""
    x = gauss_legendre_nodes(k)
    n = k + 1
    p = np.arange(n ** 3)
    return np.stack([x[p % n], x[(p // n) % n], x[p // n ** 2]], axis=1)


class Operator:
    """A divergence operator staged for the kernel (device memory)."""

    def __init__(self, D):
        _dev.require_torch_cuda()
        lib = _native.load()
        Dt = D if _dev.is_device(D) else _dev.upload(np.ascontiguousarray(D, dtype=np.float32))
        Dt = Dt.to(torch.float32).contiguous()
        if Dt.dim() != 2 or Dt.shape[0] != 3 * Dt.shape[1]:
            raise ValueError(f"operator must be (3 ns, ns), got {tuple(Dt.shape)}")
        self.n_points = int(Dt.shape[1])
        size = int(lib.vc3_fr_operator_floats(self.n_points))
        if size < 0:
            raise ValueError(f"n_points must be in [1, 256], got {self.n_points}")
        self.staged = torch.empty(size, dtype=torch.float32, device=Dt.device)
        _native.check(lib.vc3_fr_prepare_operator(Dt.data_ptr(), self.n_points,
                                                  self.staged.data_ptr(), _dev.stream_of(Dt)),
                      "fr_prepare_operator")
        self.D = Dt


def _geometry(x, op: Operator):
    ns, n_vars, ld = int(x.shape[0]), int(x.shape[1]), int(x.shape[2])
    if ns != op.n_points:
        raise LengthMismatch(f"flux has {ns} solution points, operator {op.n_points}")
    return ns, n_vars, ld


def flux_divergence(words, op: Operator, n_elem: int | None = None, layout=DEFAULT_LAYOUT):
    """Divergence of compressed fluxes: ``words`` is a CUDA uint64 tensor
    ``[ns][n_vars][ld]``; returns float32 ``[ns][n_vars][ld]`` (columns
    ``>= n_elem`` left unwritten)."""
    layout = as_layout(layout)
    lib = _native.load()
    if not _dev.is_device(words) or words.dim() != 3:
        raise ValueError("flux_divergence takes a CUDA uint64 tensor [ns][n_vars][ld]")
    w = words.contiguous()
    ns, n_vars, ld = _geometry(w, op)
    n_elem = ld if n_elem is None else int(n_elem)
    out = torch.empty((ns, n_vars, ld), dtype=torch.float32, device=w.device)
    _native.check(lib.vc3_fr_divergence(w.data_ptr(), op.staged.data_ptr(), out.data_ptr(), n_elem,
                                        n_vars, ld, ns, _native.c_layout(layout), _dev.stream_of(w)),
                  "fr_divergence")
    return out


def flux_divergence_f32(flux, op: Operator, n_elem: int | None = None):
    """The uncompressed baseline: ``flux`` float32 ``[ns][n_vars][ld][3]``."""
    lib = _native.load()
    if not _dev.is_device(flux) or flux.dim() != 4 or flux.shape[3] != 3:
        raise ValueError("flux_divergence_f32 takes a CUDA float32 tensor [ns][n_vars][ld][3]")
    f = flux.to(torch.float32).contiguous()
    ns, n_vars, ld = _geometry(f, op)
    n_elem = ld if n_elem is None else int(n_elem)
    out = torch.empty((ns, n_vars, ld), dtype=torch.float32, device=f.device)
    _native.check(lib.vc3_fr_divergence_f32(f.data_ptr(), op.staged.data_ptr(), out.data_ptr(),
                                            n_elem, n_vars, ld, ns, _dev.stream_of(f)),
                  "fr_divergence_f32")
    return out


def _hex_degree(ns: int) -> int:
    k = round(ns ** (1.0 / 3.0)) - 1
    if (k + 1) ** 3 != ns or not 1 <= k <= 4:
        raise ValueError(f"{ns} points is not a hexahedron of degree 1..4")
    return k


def flux_divergence_hex(words, n_elem: int | None = None, layout=DEFAULT_LAYOUT, m1d=None):
    """Sum-factorised divergence for tensor-product hexahedra (degree 1..4):
    ``words`` CUDA uint64 ``[ns][n_vars][ld]`` with ns = (k+1)^3; the operator
    is ``divergence_operator(k)`` unless ``m1d`` (the 1D derivative matrix)
    is given.  Same result as ``flux_divergence`` to float32 rounding."""
    layout = as_layout(layout)
    lib = _native.load()
    if not _dev.is_device(words) or words.dim() != 3:
        raise ValueError("flux_divergence_hex takes a CUDA uint64 tensor [ns][n_vars][ld]")
    w = words.contiguous()
    ns, n_vars, ld = int(w.shape[0]), int(w.shape[1]), int(w.shape[2])
    k = _hex_degree(ns)
    m = np.ascontiguousarray(lagrange_derivative_matrix(gauss_legendre_nodes(k)) if m1d is None
                             else m1d, dtype=np.float32)
    n_elem = ld if n_elem is None else int(n_elem)
    out = torch.empty((ns, n_vars, ld), dtype=torch.float32, device=w.device)
    _native.check(lib.vc3_fr_divergence_hex(w.data_ptr(), m.ctypes.data, k, out.data_ptr(), n_elem,
                                            n_vars, ld, _native.c_layout(layout), _dev.stream_of(w)),
                  "fr_divergence_hex")
    return out


def flux_divergence_hex_f32(flux, n_elem: int | None = None, m1d=None):
    """Float32 fluxes ``[ns][n_vars][ld][3]`` through the sum-factorised kernel."""
    lib = _native.load()
    if not _dev.is_device(flux) or flux.dim() != 4 or flux.shape[3] != 3:
        raise ValueError("flux_divergence_hex_f32 takes a CUDA float32 tensor [ns][n_vars][ld][3]")
    f = flux.to(torch.float32).contiguous()
    ns, n_vars, ld = int(f.shape[0]), int(f.shape[1]), int(f.shape[2])
    k = _hex_degree(ns)
    m = np.ascontiguousarray(lagrange_derivative_matrix(gauss_legendre_nodes(k)) if m1d is None
                             else m1d, dtype=np.float32)
    n_elem = ld if n_elem is None else int(n_elem)
    out = torch.empty((ns, n_vars, ld), dtype=torch.float32, device=f.device)
    _native.check(lib.vc3_fr_divergence_hex_f32(f.data_ptr(), m.ctypes.data, k, out.data_ptr(), n_elem,
                                                n_vars, ld, _dev.stream_of(f)),
                  "fr_divergence_hex_f32")
    return out


__all__ = ["gauss_legendre_nodes", "lagrange_derivative_matrix", "divergence_operator",
           "solution_points", "Operator", "flux_divergence", "flux_divergence_f32", "flux_divergence_hex",
           "flux_divergence_hex_f32"]
