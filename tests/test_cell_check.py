"""CPU restatement of the decode's float32-boundary test (``near_f32_boundary``
in ``csrc/vc3_device.cuh``) and the property the exact decode relies on: if
the test does not fire for (d, 2e), every double within e of d rounds to the
same float32 as d.  Adversarial doubles sit on and next to rounding
midpoints, binade bottoms (where the float32 cell below is half as wide),
the float32 subnormal range and zero."""

from __future__ import annotations

import numpy as np

LOW29 = np.uint64(0x1FFFFFFF)
MID = np.uint64(0x10000000)


def near_f32_boundary(d: np.ndarray, e2: np.ndarray) -> np.ndarray:
    bits = d.view(np.uint64)
    b = ((bits & ~LOW29) | MID).view(np.float64)
    return (np.abs(d - b) <= e2) | ((np.abs(d) < 2.0**-126) & (e2 > 0))


def _adversarial(rng: np.random.Generator, n: int) -> np.ndarray:
    k = rng.integers(-140, 127, n).astype(np.float64)
    f = rng.uniform(1.0, 2.0, n)
    base = f * 2.0**k
    bits = base.view(np.uint64)
    j = rng.integers(-64, 65, n).astype(np.int64)
    pick = rng.integers(0, 4, n)
    mid = ((bits & ~LOW29) | MID).astype(np.int64) + j            # around a midpoint
    bottom = (bits & ~np.uint64((1 << 52) - 1)).astype(np.int64) + np.abs(j)  # binade bottom
    top = (bits | np.uint64((1 << 52) - 1)).astype(np.int64) - np.abs(j)      # binade top
    out = np.where(pick == 0, mid, np.where(pick == 1, bottom, np.where(pick == 2, top, bits.astype(np.int64))))
    d = out.astype(np.uint64).view(np.float64)
    sign = np.where(rng.integers(0, 2, n) == 1, -1.0, 1.0)
    d = d * sign
    d[:8] = [0.0, -0.0, 2.0**-126, -(2.0**-126), 2.0**-149, 1.5 * 2.0**-149, 3.4e38, 1.0]
    return d


def test_cell_check_is_conservative():
    rng = np.random.default_rng(20031)
    n = 400_000
    d = _adversarial(rng, n)
    # e from a few double ulps of d up to ~2^30 ulps, and relative to |d| + a magnitude scale
    ulp = np.spacing(np.abs(d))
    e = ulp * 2.0 ** rng.uniform(0, 30, n)
    e[:8] = [1e-300, 1e-300, 1e-50, 1e-50, 1e-50, 1e-50, 1e25, 1e-17]
    flag = near_f32_boundary(d, e + e)
    f = d.astype(np.float32)
    with np.errstate(over="ignore"):
        for t in np.linspace(-1.0, 1.0, 17):
            dp = d + t * e
            same = dp.astype(np.float32).view(np.uint32) == f.view(np.uint32)
            # sign-of-zero differences are not rounding differences
            same |= (dp.astype(np.float32) == 0) & (f == 0)
            bad = ~flag & ~same
            assert not bad.any(), (d[bad][:4], e[bad][:4], t)
    # the test is not trivially true: most non-adversarial-e cases pass through
    assert flag.mean() < 0.9


def test_cell_check_matches_straddle_rate():
    """On decode-like values (|d| <= r, e = r * 1.6 * 2^-49) the cell check fires
    for at most a few times as many components as the two-conversion straddle
    test it replaces, and never misses one the straddle test catches."""
    rng = np.random.default_rng(7)
    n = 1_000_000
    r = 2.0 ** rng.uniform(-20, 20, n)
    c = rng.uniform(-1, 1, n)
    d = r * c
    e = r * 1.6 * 2.0**-49
    straddle = (d - e).astype(np.float32) != (d + e).astype(np.float32)
    cell = near_f32_boundary(d, e + e)
    assert not (straddle & ~cell).any()
    assert cell.sum() <= 4 * max(1, straddle.sum()) + 64
