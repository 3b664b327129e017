"""Synthetic flow fields for the RK-stage workload (BASELINE.json config C4).

The isentropic convecting vortex of PAPER.md:226-252 (Shu): beta = 5,
gamma = 1.4, vortex centre x0 = (10, 10), convective velocity
(u0, v0) = (cos psi, sin psi), on the periodic box [0,20]x[0,20]x[0,2]
divided into 20x20x2 hexahedral elements, each carrying the (k+1)^3
Gauss-Legendre solution points of degree k = 4 flux reconstruction
(125 points, 10^5 in the paper's mesh).

Vectors are stored flux-reconstruction style, solution point major:
row i = upt * n_elements + element (the [n_upts][n_elem] layout of SURVEY
§8d C4), each row a float32 (x, y, z) triple.  For large workloads the
800-element box is tiled: element e lies in copy e // 800 of the box (the
fields repeat; only the storage grows).  The ICV has w = 0, so every
momentum vector sits on the equator (phi = pi/2): n_phi = 65536 for every
word, and the decoded z is the reference's r*cos(pi*65536/131071), not 0
(SURVEY Appendix B).

Input generation only (torch float64 on the device, numpy on the host for
tests); the codec work is in the CUDA library.
"""

from __future__ import annotations

import math

import numpy as np

BETA = 5.0
GAMMA_GAS = 1.4
X0 = (10.0, 10.0)
BOX_ELEMENTS = (20, 20, 2)
DEGREE = 4


def gauss_legendre_nodes(k: int = DEGREE) -> np.ndarray:
    """The k+1 Gauss-Legendre nodes on [-1, 1]."""
    return np.polynomial.legendre.leggauss(k + 1)[0]


def _point_coords(n_elements: int, k: int, xp):
    nodes = xp.asarray(gauss_legendre_nodes(k))
    npts = (k + 1) ** 3
    ex, ey, ez = BOX_ELEMENTS
    per_box = ex * ey * ez
    upt = xp.arange(npts)
    elem = xp.arange(n_elements)
    i, j, l = upt % (k + 1), (upt // (k + 1)) % (k + 1), upt // (k + 1) ** 2
    local = elem % per_box
    cx, cy, cz = local % ex, (local // ex) % ey, local // (ex * ey)
    # row-major [upt][element]
    x = cx[None, :] + 0.5 * (nodes[i][:, None] + 1.0)
    y = cy[None, :] + 0.5 * (nodes[j][:, None] + 1.0)
    z = cz[None, :] + 0.5 * (nodes[l][:, None] + 1.0)
    return x.reshape(-1), y.reshape(-1), z.reshape(-1)


def icv_fields(n_elements: int, psi_deg: float = 0.0, k: int = DEGREE, device=None):
    """(momentum, velocity) float32 arrays of shape (n_elements*(k+1)^3, 3).

    ``device=None``: numpy on the host; otherwise torch tensors on ``device``
    (same float64 arithmetic, so both agree to float32 rounding)."""
    if device is None:
        xp = np
    else:
        import torch

        class _T:  # minimal numpy-like shim over torch float64
            @staticmethod
            def asarray(a):
                return torch.as_tensor(a, dtype=torch.float64, device=device)

            @staticmethod
            def arange(n):
                return torch.arange(n, device=device)

            exp = staticmethod(torch.exp)
            zeros_like = staticmethod(torch.zeros_like)
            stack = staticmethod(lambda arrs, axis: torch.stack(arrs, dim=axis))

        xp = _T
    x, y, _ = _point_coords(n_elements, k, xp)
    u0, v0 = math.cos(math.radians(psi_deg)), math.sin(math.radians(psi_deg))
    dx, dy = x - X0[0], y - X0[1]
    r2 = dx * dx + dy * dy
    f = xp.exp((1.0 - r2) / 2.0)
    u = u0 + BETA / (2.0 * math.pi) * (X0[1] - y) * f
    v = v0 - BETA / (2.0 * math.pi) * (X0[0] - x) * f
    w = xp.zeros_like(u)
    g = GAMMA_GAS
    p = (1.0 - (g - 1.0) * BETA ** 2 / (8.0 * g * math.pi ** 2) * xp.exp(1.0 - r2)) ** (g / (g - 1.0))
    rho = p ** (1.0 / g)
    vel = xp.stack([u, v, w], 1)
    mom = xp.stack([rho * u, rho * v, rho * w], 1)
    if device is None:
        return mom.astype(np.float32), vel.astype(np.float32)
    import torch

    return mom.to(torch.float32), vel.to(torch.float32)


# Carpenter-Kennedy low-storage RK4(5) (2N storage) coefficients, the
# "4th order low-storage explicit Runge-Kutta" of PAPER.md:135.
LSRK_A = (0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
          -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0)
LSRK_B = (1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
          1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
          2277821191437.0 / 14882151754819.0)
