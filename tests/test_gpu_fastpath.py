"""The all-single fast path (csrc/vc3_fused.cuh) against the C oracle on
adversarial inputs.  Needs a B200.

The fast path replaces the reference's IEEE divide / sqrt calls with their
Newton sequences, widens float32 values from their bits, folds the y == 0
case into a sign test and skips the bucket clamps; every one of those steps
has a range outside which it hands the vector to the generic exact compress.
These tests aim at the range edges: signed zeros in every component,
subnormals, values near FLT_MAX (float32 overflow of the sum of squares),
exact float32 grid magnitudes, and words whose decode hits the theta
endpoints, the phi poles and the magnitude rails.  Bar: bit-exact in
VC3_EXACT mode (compress, add, axpy, RK stage); VC3_CONTRACT words within one
bucket of the oracle.
"""

import itertools

import numpy as np
import pytest
import torch

from conftest import layout_by_name

pytestmark = pytest.mark.gpu

SPECIAL = np.array(
    [0.0, -0.0, 1.0, -1.0, 1.5, -2.5, 2.0 ** -149, -(2.0 ** -149), 2.0 ** -126, -(2.0 ** -126),
     1e-30, -1e-30, 2.0 ** -64, 2.0 ** -63, 3e-20, 1e30, -1e30, 2.0 ** 62, -(2.0 ** 63), 2.0 ** 64,
     3.0e38, -3.4028235e38, 3.4028235e38, 1e-6, -7.0, 0.3333333, 2.0 ** 47, -(2.0 ** 46)],
    dtype=np.float32)


def special_vectors():
    return np.array(list(itertools.product(SPECIAL, repeat=3)), dtype=np.float32)


def random_wide(n, seed):
    """Random float32 vectors with exponents over (most of) the float range and
    random signed zeros."""
    g = np.random.Generator(np.random.Philox(key=(seed, 77)))
    mant = g.uniform(1.0, 2.0, (n, 3))
    expo = g.integers(-140, 127, (n, 3))
    sign = np.where(g.random((n, 3)) < 0.5, -1.0, 1.0)
    v = (sign * mant * np.exp2(expo.astype(np.float64))).astype(np.float32)
    z = g.random((n, 3)) < 0.05
    v[z] = np.where(g.random(int(z.sum())) < 0.5, np.float32(0.0), np.float32(-0.0))
    return v


def unit_scaled(n, seed, lo=-6, hi=6):
    g = np.random.Generator(np.random.Philox(key=(seed, 78)))
    d = g.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = 10.0 ** g.uniform(lo, hi, n)
    v = (d * r[:, None]).astype(np.float32)
    # axis-aligned and planar vectors: exact float grid magnitudes, zeros
    v[: n // 8, 1:] = 0.0
    v[n // 8: n // 4, 2] = -0.0
    v[n // 4: n // 4 + n // 16, 0] = -0.0
    return v


@pytest.fixture(scope="module")
def lay():
    return layout_by_name("17_18")


@pytest.fixture(scope="module")
def pol():
    from paper_2003_02633_b200.layout import ALL_SINGLE_POLICY

    return ALL_SINGLE_POLICY


def gpu_compress(vc3b, v, lay, pol, cuda):
    return vc3b.compress(torch.from_numpy(v).to(cuda), lay, pol).cpu().numpy()


@pytest.mark.parametrize("kind", ["special", "wide", "scaled"])
def test_compress_fast_path_bit_exact(vc3b, oracle, cuda, lay, pol, kind):
    v = {"special": special_vectors, "wide": lambda: random_wide(1 << 18, 1),
         "scaled": lambda: unit_scaled(1 << 18, 2)}[kind]()
    got = gpu_compress(vc3b, v, lay, pol, cuda)
    want = oracle.compress(v, lay, pol, oracle.default_threads())
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (f"{bad.size} mismatches, first {v[bad[0]].view(np.uint32)}: "
                           f"got {hex(int(got[bad[0]]))} want {hex(int(want[bad[0]]))}")


def adversarial_words(lay, n, seed):
    """Words hitting the decode's special entries: theta endpoints, phi
    poles and zero, zero / flush / saturation fields, and random words."""
    g = np.random.Generator(np.random.Philox(key=(seed, 79)))
    t, p = lay.theta_bits, lay.phi_bits
    nt = g.integers(0, 1 << t, n, dtype=np.uint64)
    nph = g.integers(0, 1 << p, n, dtype=np.uint64)
    field = g.integers(0, 1 << (64 - t - p), n, dtype=np.uint64)
    k = n // 8
    nt[:k] = np.uint64(0)
    nt[k: 2 * k] = np.uint64((1 << t) - 1)
    nph[2 * k: 3 * k] = np.uint64(0)
    nph[3 * k: 4 * k] = np.uint64((1 << p) - 1)
    field[4 * k: 4 * k + k // 4] = np.uint64(0)
    field[4 * k + k // 4: 4 * k + k // 2] = np.uint64(2 << lay.mantissa_bits)
    return (field << np.uint64(t + p)) | (nph << np.uint64(t)) | nt


def encode_of(vc3b, oracle, lay, pol, cuda, n, seed):
    v = unit_scaled(n, seed)
    return oracle.compress(v, lay, pol)


@pytest.mark.parametrize("source", ["adversarial", "encoded"])
def test_add_fast_path_bit_exact(vc3b, oracle, cuda, lay, pol, source):
    n = 1 << 17
    if source == "adversarial":
        a, b = adversarial_words(lay, n, 3), adversarial_words(lay, n, 4)[::-1].copy()
    else:
        a, b = encode_of(vc3b, oracle, lay, pol, cuda, n, 5), encode_of(vc3b, oracle, lay, pol, cuda, n, 6)
        b[: n // 4] = a[: n // 4] ^ np.uint64(1)  # near-cancelling pairs: tiny and zero sums
        b[n // 4: n // 2] = a[n // 4: n // 2]
    got = vc3b.add_compressed(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), lay,
                              pol).cpu().numpy()
    want = oracle.add_compressed(a, b, lay, pol, oracle.default_threads())
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first a={hex(int(a[bad[0]]))} b={hex(int(b[bad[0]]))}"


def test_add_contract_mode_within_one_bin(vc3b, oracle, cuda, lay, pol):
    from paper_2003_02633_b200 import ops

    n = 1 << 18
    a = encode_of(vc3b, oracle, lay, pol, cuda, n, 7)
    b = encode_of(vc3b, oracle, lay, pol, cuda, n, 8)
    got = ops.add_compressed(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), lay, pol,
                             mode="contract").cpu().numpy()
    want = oracle.add_compressed(a, b, lay, pol, oracle.default_threads())
    d = got != want
    assert d.mean() < 1e-4
    t, p = lay.theta_bits, lay.phi_bits
    g, w = got[d].astype(np.int64), want[d].astype(np.int64)
    dt = np.abs((g & ((1 << t) - 1)) - (w & ((1 << t) - 1)))
    dt = np.minimum(dt, (1 << t) - dt)
    dp = np.abs(((g >> t) & ((1 << p) - 1)) - ((w >> t) & ((1 << p) - 1)))
    df = np.abs((g >> (t + p)) - (w >> (t + p)))
    assert (dt <= 1).all() and (dp <= 1).all() and (df <= 1).all()


def test_axpy_fast_path_bit_exact(vc3b, oracle, cuda, lay, pol):
    n = 1 << 17
    x = np.concatenate([adversarial_words(lay, n // 2, 9), encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 10)])
    y = np.concatenate([adversarial_words(lay, n // 2, 11), encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 12)])
    for alpha in (0.75, -1.0, 1e-3):
        got = vc3b.ops.axpy(alpha, torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda), lay,
                            pol).cpu().numpy()
        want = oracle.axpy(alpha, x, y, lay, pol, oracle.default_threads())
        assert np.array_equal(got, want), f"alpha={alpha}: {(got != want).sum()} mismatches"


def test_rk_stage_fast_path_bit_exact(vc3b, oracle, cuda, lay, pol):
    n = 1 << 16
    q = encode_of(vc3b, oracle, lay, pol, cuda, n, 13)
    dq = np.concatenate([adversarial_words(lay, n // 2, 14), encode_of(vc3b, oracle, lay, pol, cuda, n // 2, 15)])
    R = encode_of(vc3b, oracle, lay, pol, cuda, n, 16)
    a, b, dt = np.float32(-0.4178), np.float32(0.6), np.float32(1e-3)
    qd, dqd = torch.from_numpy(q.copy()).to(cuda), torch.from_numpy(dq.copy()).to(cuda)
    vc3b.ops.rk_stage(float(a), float(b), float(dt), qd, dqd, torch.from_numpy(R).to(cuda), lay, pol)
    # composition oracle: decode, float32 ops in the documented order, encode
    vq, vd, vr = (oracle.decompress(w, lay) for w in (q, dq, R))
    d_new = (a * vd + dt * vr).astype(np.float32)
    q_new = (vq + b * d_new).astype(np.float32)
    assert np.array_equal(dqd.cpu().numpy(), oracle.compress(d_new, lay, pol))
    assert np.array_equal(qd.cpu().numpy(), oracle.compress(q_new, lay, pol))
