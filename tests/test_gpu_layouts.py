"""The all-single fused kernels on table layouts other than the default
(RuntimeLayout instantiations and the shared-memory copy sizes of
`fused_copy`, including the reduced replication of the widest layouts), both
numerics modes, against the C oracle.  Needs a B200.

* fused add, VC3_EXACT: bit-exact on adversarial words (rails, endpoints,
  poles, zero fields) and on encoded vectors; VC3_CONTRACT: every differing
  word within one bin / one magnitude step;
* axpy and the RK stage, VC3_EXACT: bit-exact;
* decompress of random words: exact bit-exact, contract <= 1 ulp.
"""
import numpy as np
import pytest
import torch

from test_gpu_fastpath import adversarial_words, encode_of

pytestmark = pytest.mark.gpu


def _layouts():
    from paper_2003_02633_b200.layout import LAYOUT_16_17, LAYOUT_17_17, LAYOUT_BASE_16_16, BitLayout

    return {
        "base_16_16": LAYOUT_BASE_16_16,
        "16_17": LAYOUT_16_17,
        "17_17": LAYOUT_17_17,
        "t20_p15": BitLayout(0, 7, 22, 15, 20, 80),  # theta residual section of 512 entries
        "e6_18_18": BitLayout(0, 6, 22, 18, 18, 40),
        "t20_p20_m19": BitLayout(0, 5, 19, 20, 20, 20),  # widest table layout; m < 20 magnitude path
    }


@pytest.fixture(scope="module", params=list(_layouts()))
def lay(request):
    return _layouts()[request.param]


@pytest.fixture(scope="module")
def pol():
    from paper_2003_02633_b200.layout import ALL_SINGLE_POLICY

    return ALL_SINGLE_POLICY


def _dev(w, cuda):
    return torch.from_numpy(np.ascontiguousarray(w)).to(cuda)


def _within_one_bin(got, want, lay):
    d = got != want
    t, p = lay.theta_bits, lay.phi_bits
    g, w = got[d].astype(np.int64), want[d].astype(np.int64)
    dt = np.abs((g & ((1 << t) - 1)) - (w & ((1 << t) - 1)))
    dt = np.minimum(dt, (1 << t) - dt)
    dp = np.abs(((g >> t) & ((1 << p) - 1)) - ((w >> t) & ((1 << p) - 1)))
    df = np.abs((g >> (t + p)) - (w >> (t + p)))
    return int(d.sum()), bool((dt <= 1).all() and (dp <= 1).all() and (df <= 1).all())


def test_add_both_modes(vc3b, oracle, cuda, lay, pol):
    from paper_2003_02633_b200 import ops

    n = 1 << 16
    a = np.concatenate([adversarial_words(lay, n // 2, 31), encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 32)])
    b = np.concatenate([adversarial_words(lay, n // 2, 33)[::-1], encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 34)])
    want = oracle.add_compressed(a, b, lay, pol, oracle.default_threads())
    got = ops.add_compressed(_dev(a, cuda), _dev(b, cuda), lay, pol).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first a={hex(int(a[bad[0]]))} b={hex(int(b[bad[0]]))}"
    got_c = ops.add_compressed(_dev(a, cuda), _dev(b, cuda), lay, pol, mode="contract").cpu().numpy()
    ndiff, ok = _within_one_bin(got_c, want, lay)
    assert ok and ndiff <= 1e-3 * n, ndiff


def test_axpy_and_rk_exact(vc3b, oracle, cuda, lay, pol):
    from paper_2003_02633_b200 import ops

    n = 1 << 15
    x = np.concatenate([adversarial_words(lay, n // 2, 41), encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 42)])
    y = encode_of(vc3b, oracle, lay, pol, cuda, n, 43)
    got = ops.axpy(-0.75, _dev(x, cuda), _dev(y, cuda), lay, pol).cpu().numpy()
    assert np.array_equal(got, oracle.axpy(-0.75, x, y, lay, pol, oracle.default_threads()))
    q, dq, R = y, x, encode_of(vc3b, oracle, lay, pol, cuda, n, 44)
    a_, b_, dt = np.float32(-0.4178), np.float32(0.6), np.float32(1e-3)
    qd, dqd = _dev(q.copy(), cuda), _dev(dq.copy(), cuda)
    ops.rk_stage(float(a_), float(b_), float(dt), qd, dqd, _dev(R, cuda), lay, pol)
    vq, vd, vr = (oracle.decompress(w, lay) for w in (q, dq, R))
    d_new = (a_ * vd + dt * vr).astype(np.float32)
    q_new = (vq + b_ * d_new).astype(np.float32)
    assert np.array_equal(dqd.cpu().numpy(), oracle.compress(d_new, lay, pol))
    assert np.array_equal(qd.cpu().numpy(), oracle.compress(q_new, lay, pol))


def test_decompress_both_modes(vc3b, oracle, cuda, lay):
    g = np.random.Generator(np.random.Philox(key=(100 * lay.theta_bits + lay.phi_bits, 5)))
    w = g.integers(0, 2 ** 64, 1 << 16, dtype=np.uint64)
    w[:64] = adversarial_words(lay, 64, 51)
    want = oracle.decompress(w, lay).view(np.int32).astype(np.int64)
    got = vc3b.decompress(_dev(w, cuda), lay).cpu().numpy().view(np.int32).astype(np.int64)
    assert np.array_equal(got, want)
    got_c = vc3b.decompress(_dev(w, cuda), lay, mode="contract").cpu().numpy().view(np.int32).astype(np.int64)
    assert int(np.abs(got_c - want).max()) <= 1


@pytest.mark.parametrize("lname", ["t20_p20_m19", "p24_t20"])
def test_compress_near_poles(vc3b, oracle, cuda, pol, lname):
    """All-single compress on wide angle fields (the fast path covers t <= 25,
    p <= 24): vectors whose float32 quotient z / |v| rounds to +-1, where the
    acos argument (1 - |w|) / 2 is 0, and their neighbours."""
    from paper_2003_02633_b200.layout import BitLayout

    lay = {"t20_p20_m19": _layouts()["t20_p20_m19"], "p24_t20": BitLayout(0, 5, 15, 24, 20, 20)}[lname]
    g = np.random.Generator(np.random.Philox(key=(lay.phi_bits, 61)))
    n = 1 << 16
    v = np.empty((n, 3), np.float32)
    z = np.where(g.random(n) < 0.5, -1.0, 1.0) * 10.0 ** g.uniform(-3, 3, n)
    tilt = 10.0 ** g.uniform(-9, -2, n)  # off-axis angle
    ang = g.uniform(-np.pi, np.pi, n)
    v[:, 0] = np.abs(z) * tilt * np.cos(ang)
    v[:, 1] = np.abs(z) * tilt * np.sin(ang)
    v[:, 2] = z
    v[: n // 16, :2] = 0.0  # exactly on the axis
    want = oracle.compress(v, lay, pol)
    got = vc3b.compress(torch.from_numpy(v).to(cuda), lay, pol).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first v={v[bad[0]]} got={hex(int(got[bad[0]]))} want={hex(int(want[bad[0]]))}"
