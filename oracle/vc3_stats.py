"""CPU restatement of the K6 error metrics (numpy, float64).

TEST INFRASTRUCTURE ONLY (parity checker for vc3_error_stats; see
vc3_oracle.py for who may import it).  Metric 0/1 follow the reference's
_errors (/root/reference/pkg/src/vc3/analysis.py:148-154); 2 (angular) and 3
(relative magnitude) are not in the reference and are
defined here and in csrc/vc3_kernels.cu err_one with the same operation
order: every product, sum and quotient rounded separately, left to right.
"""

from __future__ import annotations

import numpy as np

L2, L2_NORMALISED, ANGULAR, REL_MAGNITUDE = 0, 1, 2, 3


def _norm(x, y, z):
    return np.sqrt((x * x + y * y) + z * z)


def errors(v, vh, kind: int) -> np.ndarray:
    v = np.asarray(v, dtype=np.float32).astype(np.float64)
    h = np.asarray(vh, dtype=np.float32).astype(np.float64)
    x, y, z = v[:, 0], v[:, 1], v[:, 2]
    a, b, c = h[:, 0], h[:, 1], h[:, 2]
    if kind == ANGULAR:
        cx = y * c - z * b
        cy = z * a - x * c
        cz = x * b - y * a
        dot = (x * a + y * b) + z * c
        return np.arctan2(_norm(cx, cy, cz), dot)
    nv = _norm(x, y, z)
    if kind == REL_MAGNITUDE:
        safe = np.where(nv > 0, nv, 1.0)
        return np.where(nv > 0, np.abs(_norm(a, b, c) - nv) / safe, 0.0)
    e = _norm(x - a, y - b, z - c)
    if kind == L2_NORMALISED:
        e = e / np.where(nv > 0, nv, 1.0)
    return e


def chunk_moments(v, vh, kind: int, chunk: int) -> np.ndarray:
    """(k, 4) rows (count, mean, M2, max) per chunk of ``chunk`` vectors."""
    e = errors(v, vh, kind)
    rows = []
    for lo in range(0, e.size, chunk):
        part = e[lo:lo + chunk]
        mean = part.mean()
        rows.append((part.size, mean, ((part - mean) ** 2).sum(), part.max()))
    return np.array(rows, dtype=np.float64)
