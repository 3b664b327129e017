"""Property tests in the style of the reference suite (hypothesis):
host logic on CPU, codec properties on the GPU path."""

import io
from fractions import Fraction
import math

import numpy as np
import pytest
from hypothesis import assume, given, settings, strategies as st

from paper_2003_02633_b200 import BitLayout, nint, parse_layout
from paper_2003_02633_b200.stream import pack_header, parse_header, read_csv, write_csv


def exact_nint(x: Fraction) -> int:
    return math.ceil(math.floor(2 * x) / Fraction(2))


@given(st.integers(-10**6, 10**6), st.sampled_from([0, 1, 2, 3]))
def test_nint_matches_exact_rationals(k, quarter):
    x = Fraction(k) + Fraction(quarter, 4)
    assert nint(float(x)) == exact_nint(x)


@given(st.floats(-1e9, 1e9, allow_nan=False))
def test_nint_within_half_ties_up(x):
    n = nint(x)
    assert abs(n - x) <= 0.5
    if abs(n - x) == 0.5:
        assert n > x


valid_layouts = st.builds(
    lambda s, e, m, p: (s, e, m, p, 64 - s - e - m - p),
    st.sampled_from([0, 1]), st.integers(1, 8), st.integers(1, 23), st.integers(1, 32),
).filter(lambda w: 1 <= w[4] <= 32)


@given(valid_layouts)
def test_layout_spec_and_header_round_trip(w):
    from paper_2003_02633_b200.layout import default_bias

    s, e, m, p, t = w
    lay = BitLayout(s, e, m, p, t, default_bias(e))
    assert parse_layout(lay.spec()) == lay
    assert parse_header(pack_header(lay, 123)) == (lay, 123)


@given(st.lists(st.floats(width=32, allow_nan=False, allow_infinity=False), min_size=3, max_size=30))
def test_csv_round_trip_exact(values):
    n = len(values) // 3
    v = np.array(values[: 3 * n], dtype=np.float32).reshape(-1, 3)
    buf = io.StringIO()
    write_csv(buf, v)
    back = read_csv(io.StringIO(buf.getvalue()))
    assert np.array_equal(back.view(np.uint32), v.view(np.uint32)) or np.array_equal(back, v)


@pytest.mark.gpu
@given(st.lists(st.floats(-1.0, 1.0, width=32), min_size=3, max_size=3))
@settings(max_examples=200, deadline=None)
def test_relative_error_bound_in_unit_cube(cuda, comps):
    """pkg/tests/test_codec.py:109-117 on the GPU codec."""
    import paper_2003_02633_b200 as vc3b

    v = np.array([comps], dtype=np.float32)
    nv = float(np.linalg.norm(v.astype(np.float64)))
    assume(nv > 1e-20)
    vh = vc3b.decompress(vc3b.compress(v))
    err = float(np.linalg.norm(vh.astype(np.float64) - v.astype(np.float64)))
    assert err / nv <= 3e-5


@pytest.mark.gpu
@given(st.floats(2.0 ** -70, 2.0 ** 40), st.floats(2.0 ** -70, 2.0 ** 40))
@settings(max_examples=200, deadline=None)
def test_magnitude_bound_and_monotone(cuda, a, b):
    """pkg/tests/test_magnitude.py:57-70 on the GPU magnitude pieces."""
    import paper_2003_02633_b200 as vc3b

    lo, hi = sorted((a, b))
    r = np.array([lo, hi])
    rh = vc3b.decode_magnitude(vc3b.encode_magnitude(r)).astype(np.float64)
    assert np.all(np.abs(rh - r) / r <= 2.0 ** -22)
    assert rh[0] <= rh[1]
