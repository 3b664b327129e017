"""CUDA path vs the reference (golden fixtures) and the C oracle.  Needs a B200.

Parity bar (BASELINE.json north star):
  * bit-unpacking and magnitude coding: bit-exact;
  * compressed words: bit-exact, except quantisation-bin ties caused by
    transcendental ulp differences, each within one bin.  Policies whose
    angles are all single precision never call a double transcendental
    (the float32 trig is the reference's own polynomial), so they must be
    bit-exact; double-angle policies go through CUDA's libm, where ties are
    allowed and counted;
  * decompressed components: bit-exact to the reference decode of the same
    word (fast table decode; components within the measured decode tolerance
    of a float32 rounding boundary are re-evaluated from the reference's own
    tables; vc3_decode_tolerance).
"""

import numpy as np
import pytest
import torch

from conftest import LAYOUT_NAMES, layout_by_name, policy_by_code

pytestmark = pytest.mark.gpu

VEC_SETS = ["mixed", "kat", "edge", "sphere", "cube", "spread"]
ALL_CODES = ["SSS", "SSD", "SDS", "SDD", "DSS", "DSD", "DDS", "DDD"]


def _fields(words, lay):
    w = np.asarray(words, dtype=np.uint64)
    nt = (w & np.uint64(lay.n_theta_max)).astype(np.int64)
    nph = ((w >> np.uint64(lay.theta_bits)) & np.uint64(lay.n_phi_max)).astype(np.int64)
    field = (w >> np.uint64(lay.theta_bits + lay.phi_bits)).astype(np.int64)
    return nt, nph, field


def assert_words_match(got, want, lay, code, label=""):
    got = np.asarray(got, dtype=np.uint64)
    want = np.asarray(want, dtype=np.uint64)
    assert got.shape == want.shape
    diff = got != want
    if code[0] == "S" and code[1] == "S":
        assert not diff.any(), f"{label}: {int(diff.sum())} word mismatches on an all-single policy"
        return 0
    g_nt, g_np, g_f = _fields(got[diff], lay)
    w_nt, w_np, w_f = _fields(want[diff], lay)
    assert np.array_equal(g_f, w_f), f"{label}: magnitude field differs"
    # a tie flips exactly one bucket by one (theta wraps only at the clamp ends)
    assert (np.abs(g_nt - w_nt) <= 1).all() and (np.abs(g_np - w_np) <= 1).all(), label
    assert diff.mean() <= 1e-3, f"{label}: tie rate {diff.mean():.2e}"
    return int(diff.sum())


def ulp32(a, b):
    ia = np.asarray(a, dtype=np.float32).view(np.int32).astype(np.int64)
    ib = np.asarray(b, dtype=np.float32).view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 31)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 31)) - ib, ib)
    return np.abs(ia - ib)


def assert_vectors_match(got, want, label=""):
    got = np.asarray(got, dtype=np.float32)
    want = np.asarray(want, dtype=np.float32)
    assert got.shape == want.shape
    u = ulp32(got, want)
    assert u.max() <= 2, f"{label}: max ulp {u.max()}"
    assert (u == 0).mean() >= 0.9999, f"{label}: exact fraction {(u == 0).mean()}"


# ---------------------------------------------------------------------------
# golden fixtures (reference outputs)
# ---------------------------------------------------------------------------
def test_compress_golden_default_layout_all_policies(golden, vc3b, cuda):
    lay = layout_by_name("17_18")
    ties = 0
    for code in ALL_CODES:
        for vname in VEC_SETS:
            want = golden[f"cw_17_18_{code}_{vname}"]
            v = golden[f"vec_{vname}"][: want.size]
            ties += assert_words_match(vc3b.compress(v, lay, policy_by_code(code)), want, lay,
                                       code, f"host {code} {vname}")
            dv = torch.from_numpy(v).to(cuda)
            got = vc3b.compress(dv, lay, policy_by_code(code)).cpu().numpy()
            assert_words_match(got, want, lay, code, f"device {code} {vname}")
    print(f"double-policy bin ties on the golden sets: {ties}")


@pytest.mark.parametrize("lname", LAYOUT_NAMES[1:])
def test_compress_golden_other_layouts(golden, vc3b, cuda, lname):
    lay = layout_by_name(lname)
    for code in ["SDS", "SSS", "DDD"]:
        for vname in ["mixed", "kat", "edge", "spread"]:
            want = golden[f"cw_{lname}_{code}_{vname}"]
            v = golden[f"vec_{vname}"][: want.size]
            assert_words_match(vc3b.compress(v, lay, policy_by_code(code)), want, lay, code,
                               f"{lname} {code} {vname}")


@pytest.mark.parametrize("lname", LAYOUT_NAMES)
def test_decompress_golden(golden, vc3b, cuda, lname):
    lay = layout_by_name(lname)
    assert_vectors_match(vc3b.decompress(golden["words_random"], lay),
                         golden[f"dv_{lname}_random"], f"{lname} random words")
    for code in ("SSS", "SDS"):
        for vname in ("mixed", "edge", "kat", "spread"):
            words = golden[f"cw_{lname}_{code}_{vname}"]
            want = golden[f"dv_{lname}_{code}_{vname}"]
            assert_vectors_match(vc3b.decompress(words, lay), want, f"{lname} {code} {vname}")
            got = vc3b.decompress(torch.from_numpy(words).to(cuda), lay).cpu().numpy()
            assert_vectors_match(got, want, f"device {lname} {code} {vname}")


def test_every_random_word_decodes_finite(golden, vc3b, cuda):
    for lname in LAYOUT_NAMES:
        out = vc3b.decompress(golden["words_random"], layout_by_name(lname))
        assert np.isfinite(out).all()


@pytest.mark.parametrize("key,lname,code", [
    ("17_18_SSS", "17_18", "SSS"), ("17_18_SDS", "17_18", "SDS"), ("17_18_DDD", "17_18", "DDD"),
    ("base_16_16_SSS", "base_16_16", "SSS"), ("wide_10_25_SSS", "wide_10_25", "SSS")])
def test_add_compressed_golden(golden, vc3b, cuda, key, lname, code):
    lay, pol = layout_by_name(lname), policy_by_code(code)
    a, b = golden[f"add_a_{key}"], golden[f"add_b_{key}"]
    want = golden[f"add_c_{key}"]
    assert_words_match(vc3b.add_compressed(a, b, lay, pol), want, lay, code, f"host {key}")
    da, db = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    got = vc3b.add_compressed(da, db, lay, pol).cpu().numpy()
    assert_words_match(got, want, lay, code, f"device {key}")


def test_add_compressed_adversarial_words(golden, vc3b, cuda):
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    w = golden["words_random"]
    assert_words_match(vc3b.add_compressed(w[:10_000], w[10_000:], lay, pol),
                       golden["add_c_random_SSS"], lay, "SSS", "random words")
    kw = golden["cw_17_18_SSS_kat"]
    got = vc3b.add_compressed(kw[:4], kw[3::-1].copy(), lay, pol)
    assert [hex(int(x)) for x in got] == ["0xa4d413d400028000", "0xa27311b9913e7fff",
                                          "0xa27311b9913e7fff", "0xa4d413d400028000"]


def test_add_raw_golden(golden, vc3b, cuda):
    got = vc3b.add_raw(golden["add_va"], golden["add_vb"])
    assert np.array_equal(got, golden["add_raw_c"])
    dv = vc3b.add_raw(torch.from_numpy(golden["add_va"]).to(cuda),
                      torch.from_numpy(golden["add_vb"]).to(cuda)).cpu().numpy()
    assert np.array_equal(dv, golden["add_raw_c"])


def test_pieces_golden(golden, vc3b, cuda):
    lay = layout_by_name("17_18")
    pv = golden["piece_vec"]
    for code in ("SDS", "SSS", "DDD", "DSS"):
        pol = policy_by_code(code)
        r, th, ph = vc3b.to_spherical(pv, pol)
        assert np.array_equal(r, golden[f"sph_r_{code}"])
        wt, wp = golden[f"sph_th_{code}"], golden[f"sph_ph_{code}"]
        if code[0] == "S":
            assert np.array_equal(th, wt)
        else:  # CUDA vs glibc double atan2: last-ulp differences only
            assert np.abs(th - wt).max() <= 4 * np.spacing(np.pi)
        if code[1] == "S":
            assert np.array_equal(ph, wp)
        else:
            assert np.abs(ph - wp).max() <= 4 * np.spacing(np.pi)
        # bucket arithmetic is pure IEEE: bit-exact on the reference's angles
        nt, nph = vc3b.quantize_angles(wt, wp, lay, pol)
        assert np.array_equal(nt, golden[f"q_nt_{code}"])
        assert np.array_equal(nph, golden[f"q_nph_{code}"])
    for code in ("SSS", "DDD"):
        nt, nph = vc3b.quantize_angles(golden["qin_th"], golden["qin_ph"], lay, policy_by_code(code))
        assert np.array_equal(nt, golden[f"qout_nt_{code}"])
        assert np.array_equal(nph, golden[f"qout_nph_{code}"])
    idx = np.arange(0, 1 << 18, 61)
    th, ph = vc3b.dequantize_angles(idx, idx >> 1, lay)
    assert np.array_equal(th, golden["deq_th"]) and np.array_equal(ph, golden["deq_ph"])


@pytest.mark.parametrize("lname", LAYOUT_NAMES)
def test_magnitude_golden(golden, vc3b, cuda, lname):
    lay = layout_by_name(lname)
    r = golden["mag_r"]
    r = r[np.isfinite(r)]
    f = vc3b.encode_magnitude(r, lay)
    assert np.array_equal(f, golden[f"mag_field_{lname}"][: r.size])
    d = vc3b.decode_magnitude(f, lay)
    assert np.array_equal(d.view(np.uint32), golden[f"mag_dec_{lname}"][: r.size].view(np.uint32))


def test_magnitude_events_golden(golden, vc3b, cuda):
    lay = layout_by_name("17_18")
    assert vc3b.magnitude_event_counts(golden["vec_mixed"], lay) == tuple(golden["mag_events_mixed"])
    assert vc3b.magnitude_event_counts(golden["vec_edge"], lay) == tuple(golden["mag_events_edge"])


def test_scalar_api_kats(vc3b, cuda):
    # pkg/tests/test_codec.py:30-47 and SURVEY Appendix B
    assert vc3b.compress_one((1.0, 0.0, 0.0)) == ((80 << 22) << 35) | (65536 << 18) | 131072
    assert vc3b.compress_one((0.0, 0.0, 0.0)) == 0
    assert vc3b.decompress_one(0) == (0.0, 0.0, 0.0)
    assert vc3b.decompress_one(vc3b.compress_one((0.0, 0.0, 1.0))) == (0.0, 0.0, 1.0)
    assert vc3b.compress_one((-1.0, -0.0, 0.0), policy=vc3b.ORACLE_POLICY) == 0xa000000400000000
    assert vc3b.compress_one((-1.0, -0.0, 0.0)) == 0xa00000040003ffff
    for bits in (0, 123456, (1 << 35) - 1):
        assert vc3b.decompress_one(bits) == (0.0, 0.0, 0.0)
    assert vc3b.encode_magnitude(1.0) == 80 << 22
    assert vc3b.decode_magnitude(80 << 22) == 1.0
    assert vc3b.quantize_angles(0.0, 0.0, vc3b.BitLayout(0, 7, 23, 17, 17, 80),
                                vc3b.ORACLE_POLICY) == (65536, 0)


# ---------------------------------------------------------------------------
# errors and edge shapes
# ---------------------------------------------------------------------------
def test_nonfinite_raises(vc3b, cuda):
    bad = np.array([[1, np.nan, 0], [0, 0, np.inf], [1, 2, 3]], dtype=np.float32)
    with pytest.raises(vc3b.NonFiniteInput, match="2 vector"):
        vc3b.compress(bad)
    with pytest.raises(vc3b.NonFiniteInput):
        vc3b.compress(torch.from_numpy(bad).to(cuda))
    with pytest.raises(vc3b.NonFiniteInput):
        vc3b.to_spherical(bad)
    with pytest.raises(vc3b.NonFiniteInput):
        vc3b.encode_magnitude(np.inf)
    with pytest.raises(ValueError):
        vc3b.encode_magnitude(-1.0)


def test_shape_and_length_errors(vc3b, cuda):
    with pytest.raises(ValueError):
        vc3b.compress(np.zeros((4, 2), np.float32))
    with pytest.raises(vc3b.LengthMismatch):
        vc3b.add_compressed(np.zeros(4, np.uint64), np.zeros(5, np.uint64))
    with pytest.raises(vc3b.LengthMismatch):
        vc3b.add_raw(np.zeros((4, 3), np.float32), np.zeros((5, 3), np.float32))
    with pytest.raises(ValueError):
        vc3b.quantize_angles(np.zeros(3), np.zeros(4))


@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 7, 1023, 4097])
def test_ragged_sizes(vc3b, oracle, cuda, n):
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    g = np.random.Generator(np.random.Philox(n))
    v = (g.normal(size=(n, 3)) * 10.0 ** g.uniform(-3, 3, (n, 1))).astype(np.float32)
    w = vc3b.compress(v, lay, pol)
    assert w.shape == (n,) and np.array_equal(w, oracle.compress(v, lay, pol))
    d = vc3b.decompress(w, lay)
    assert d.shape == (n, 3) and np.array_equal(d, oracle.decompress(w, lay))
    s = vc3b.add_compressed(w, w[::-1].copy(), lay, pol)
    assert np.array_equal(s, oracle.add_compressed(w, w[::-1].copy(), lay, pol))


def test_misaligned_device_views(vc3b, oracle, cuda):
    """Views starting one element in take the unvectorised path."""
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    g = np.random.Generator(np.random.Philox(5))
    v = g.normal(size=(1001, 3)).astype(np.float32)
    dv = torch.from_numpy(v).to(cuda)[1:]
    w = vc3b.compress(dv, lay, pol)
    assert np.array_equal(w.cpu().numpy(), oracle.compress(v[1:], lay, pol))
    full = torch.from_numpy(oracle.compress(v, lay, pol)).to(cuda)
    a, b = full[1:], full[:-1]
    got = vc3b.add_compressed(a, b, lay, pol).cpu().numpy()
    want = oracle.add_compressed(a.cpu().numpy(), b.cpu().numpy(), lay, pol)
    assert np.array_equal(got, want)
    assert np.array_equal(vc3b.decompress(a, lay).cpu().numpy(), oracle.decompress(a.cpu().numpy(), lay))


# ---------------------------------------------------------------------------
# larger seeded inputs vs the C oracle (all host cores)
# ---------------------------------------------------------------------------
N_MID = 1 << 21


@pytest.fixture(scope="module")
def mid_inputs():
    g = np.random.Generator(np.random.Philox(key=(2003, 2633)))
    dirs = g.normal(size=(N_MID, 3))
    mags = 10.0 ** g.uniform(-6, 6, (N_MID, 1))
    v = (dirs * mags).astype(np.float32)
    cube = g.uniform(-1.0, 1.0, (N_MID, 3)).astype(np.float32)
    return v, cube


def test_mid_compress_vs_oracle(vc3b, oracle, cuda, mid_inputs):
    v, _ = mid_inputs
    lay = layout_by_name("17_18")
    nthr = oracle.default_threads()
    for code in ("SSS", "SDS", "DDD"):
        pol = policy_by_code(code)
        got = vc3b.compress(torch.from_numpy(v).to(cuda), lay, pol).cpu().numpy()
        ties = assert_words_match(got, oracle.compress(v, lay, pol, nthreads=nthr), lay, code, code)
        print(f"{code}: {ties} ties in {N_MID} words ({ties / N_MID:.2e})")


def test_mid_decompress_vs_oracle(vc3b, oracle, cuda):
    g = np.random.Generator(np.random.Philox(77))
    w = g.integers(0, 2 ** 64, N_MID, dtype=np.uint64)
    lay = layout_by_name("17_18")
    got = vc3b.decompress(torch.from_numpy(w).to(cuda), lay).cpu().numpy()
    want = oracle.decompress(w, lay, nthreads=oracle.default_threads())
    assert_vectors_match(got, want, "random words")
    print(f"decode mismatching components: {int((got != want).sum())} of {3 * N_MID}")


def test_mid_add_vs_oracle(vc3b, oracle, cuda, mid_inputs):
    _, cube = mid_inputs
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    nthr = oracle.default_threads()
    a = oracle.compress(cube, lay, pol, nthreads=nthr)
    b = oracle.compress(cube[::-1].copy(), lay, pol, nthreads=nthr)
    got = vc3b.add_compressed(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), lay, pol)
    assert_words_match(got.cpu().numpy(), oracle.add_compressed(a, b, lay, pol, nthreads=nthr),
                       lay, "SSS", "fused add")


def test_axpy_and_rk_vs_composition(vc3b, oracle, cuda, mid_inputs):
    v, cube = mid_inputs
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    n = 1 << 18
    x = oracle.compress(v[:n], lay, pol)
    y = oracle.compress(cube[:n], lay, pol)
    alpha = np.float32(-0.37)
    got = vc3b.axpy(alpha, torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda), lay, pol)
    want = oracle.axpy(alpha, x, y, lay, pol)
    assert_words_match(got.cpu().numpy(), want, lay, "SSS", "axpy")
    # composition with float32 numpy arithmetic, op order as documented
    xd, yd = oracle.decompress(x, lay), oracle.decompress(y, lay)
    assert np.array_equal(want, oracle.compress(alpha * xd + yd, lay, pol))
    # RK stage
    R = oracle.compress(cube[n:2 * n] * np.float32(3.0), lay, pol)
    ca, cb, dt = np.float32(-0.4178904745), np.float32(1.4965783), np.float32(1e-3)
    q = torch.from_numpy(x.copy()).to(cuda)
    dq = torch.from_numpy(y.copy()).to(cuda)
    vc3b.rk_stage(ca, cb, dt, q, dq, torch.from_numpy(R).to(cuda), lay, pol)
    qd, dqd, Rd = oracle.decompress(x, lay), oracle.decompress(y, lay), oracle.decompress(R, lay)
    dq_new = ca * dqd + dt * Rd
    q_new = qd + cb * dq_new
    assert_words_match(dq.cpu().numpy(), oracle.compress(dq_new, lay, pol), lay, "SSS", "rk dq")
    assert_words_match(q.cpu().numpy(), oracle.compress(q_new, lay, pol), lay, "SSS", "rk q")


# ---------------------------------------------------------------------------
# full BASELINE size (2^28 vectors): size-independent properties
# ---------------------------------------------------------------------------
def test_full_size_fused_equals_composed_and_commutes(vc3b, cuda):
    n = 1 << 28
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    gen = torch.Generator(device=cuda).manual_seed(7)
    a = vc3b.compress(torch.rand((n, 3), device=cuda, generator=gen) * 2 - 1, lay, pol)
    b = vc3b.compress(torch.rand((n, 3), device=cuda, generator=gen) * 2 - 1, lay, pol)
    c = vc3b.add_compressed(a, b, lay, pol)
    assert torch.equal(c.view(torch.int64), vc3b.add_compressed(b, a, lay, pol).view(torch.int64))
    # fused == composed (pkg/tests/test_bench.py:40-53), checked on a strided sample
    idx = torch.arange(0, n, 97, device=cuda)
    a_s, b_s = a.view(torch.int64)[idx], b.view(torch.int64)[idx]  # uint64 has no gather kernel
    composed = vc3b.compress(vc3b.decompress(a_s, lay) + vc3b.decompress(b_s, lay), lay, pol)
    assert torch.equal(c.view(torch.int64)[idx], composed.view(torch.int64))
    # decoded words are fixed points of the double-policy round trip
    w1 = vc3b.compress(vc3b.decompress(a_s, lay), lay, vc3b.ORACLE_POLICY)
    v1 = vc3b.decompress(w1, lay)
    w2 = vc3b.compress(v1, lay, vc3b.ORACLE_POLICY)
    assert torch.equal(w1.view(torch.int64), w2.view(torch.int64))
    assert torch.isfinite(vc3b.decompress(c.view(torch.int64)[idx], lay)).all()


def test_rk_stage_on_icv_field_vs_composition(vc3b, oracle, cuda):
    """BASELINE config C4 at the paper's mesh size (10^5 points):
    five low-storage RK stages on compressed momentum match the oracle
    composition (decompress, float32 update, compress) stage by stage."""
    from paper_2003_02633_b200 import fields

    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    mom, vel = fields.icv_fields(800, 30.0)
    assert mom.shape == (100_000, 3) and (mom[:, 2] == 0).all()
    q = oracle.compress(mom, lay, pol)
    assert (((q >> np.uint64(18)) & np.uint64(lay.n_phi_max)) == 65536).all()  # equator
    dq = oracle.compress(vel * np.float32(1e-3), lay, pol)
    R = oracle.compress(vel, lay, pol)
    tq, tdq, tR = (torch.from_numpy(x.copy()).to(cuda) for x in (q, dq, R))
    dt = np.float32(1e-3)
    for s in range(5):
        a, b = np.float32(fields.LSRK_A[s]), np.float32(fields.LSRK_B[s])
        vc3b.rk_stage(a, b, dt, tq, tdq, tR, lay, pol)
        qd, dqd, Rd = (oracle.decompress(x, lay) for x in (q, dq, R))
        dq_new = a * dqd + dt * Rd
        q_new = qd + b * dq_new
        dq, q = oracle.compress(dq_new, lay, pol), oracle.compress(q_new, lay, pol)
        assert_words_match(tdq.cpu().numpy(), dq, lay, "SSS", f"stage {s} dq")
        assert_words_match(tq.cpu().numpy(), q, lay, "SSS", f"stage {s} q")


def test_decode_tolerance_is_tight(vc3b, cuda):
    """The exact decode's boundary tolerance is measured per layout over every
    table index; it must stay near the double-rounding floor (a loose bound
    only costs speed, a zero one would skip the boundary re-evaluation)."""
    import ctypes

    from paper_2003_02633_b200 import _native

    lib = _native.load()
    for lname in LAYOUT_NAMES:
        lay = layout_by_name(lname)
        tol = ctypes.c_double(-1.0)
        assert lib.vc3_decode_tolerance(_native.c_layout(lay), ctypes.byref(tol)) == 0
        if lay.theta_bits <= 20 and lay.phi_bits <= 20:  # table-decoded layouts
            assert 2.0 ** -49 < tol.value < 2.0 ** -46, (lname, tol.value)
        else:
            assert tol.value == 0.0


def test_rk_stage_f32_baseline(vc3b, cuda):
    g = torch.Generator(device=cuda).manual_seed(3)
    q, dq, R = (torch.rand(3 * 1001, device=cuda, generator=g) for _ in range(3))
    q0, dq0 = q.clone(), dq.clone()
    vc3b.ops.rk_stage_f32(0.5, 0.25, 1e-3, q, dq, R)
    dq_ref = (torch.tensor(0.5, device=cuda) * dq0 + torch.tensor(1e-3, device=cuda) * R)
    assert torch.equal(dq, dq_ref)
    assert torch.equal(q, q0 + 0.25 * dq_ref)


@pytest.mark.parametrize("lname", ["base_16_16", "wide_10_25", "17_17"])
@pytest.mark.parametrize("code", ["SSS", "SDS"])
def test_fused_ops_other_layouts_vs_oracle(vc3b, oracle, cuda, lname, code):
    """Fused add / axpy on the generic-layout kernels (runtime layout, and the
    reference-angle decode for the 25-bit theta layout) against the oracle."""
    lay, pol = layout_by_name(lname), policy_by_code(code)
    g = np.random.Generator(np.random.Philox(key=(len(lname), 9)))
    n = 20_001
    va = (g.normal(size=(n, 3)) * 10.0 ** g.uniform(-4, 4, (n, 1))).astype(np.float32)
    vb = g.uniform(-1, 1, (n, 3)).astype(np.float32)
    a, b = oracle.compress(va, lay, pol), oracle.compress(vb, lay, pol)
    ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    assert_words_match(vc3b.add_compressed(ta, tb, lay, pol).cpu().numpy(),
                       oracle.add_compressed(a, b, lay, pol), lay, code, f"add {lname}")
    al = np.float32(0.73)
    assert_words_match(vc3b.axpy(al, ta, tb, lay, pol).cpu().numpy(),
                       oracle.axpy(al, a, b, lay, pol), lay, code, f"axpy {lname}")
    assert_vectors_match(vc3b.decompress(ta, lay).cpu().numpy(), oracle.decompress(a, lay),
                         f"decompress {lname}")


@pytest.mark.gpu
def test_lsrk_step_graph_matches_eager(vc3b, cuda):
    """A CUDA-graph-captured LSRK step (5 rk_stage launches) is bit-identical
    to the eager stages, over several steps."""
    import torch

    from paper_2003_02633_b200 import fields, ops

    mom, vel = fields.icv_fields(800, 30.0, device="cuda")
    pol = vc3b.ALL_SINGLE_POLICY
    q0 = vc3b.compress(mom, vc3b.DEFAULT_LAYOUT, pol)
    dq0 = vc3b.compress(vel * 1e-3, vc3b.DEFAULT_LAYOUT, pol)
    R = vc3b.compress(vel, vc3b.DEFAULT_LAYOUT, pol)
    qa, dqa, qb, dqb = q0.clone(), dq0.clone(), q0.clone(), dq0.clone()
    ga = ops.LSRKStep(qa, dqa, R, 1e-3).capture()
    eb = ops.LSRKStep(qb, dqb, R, 1e-3)
    for _ in range(3):
        ga.step()
        eb.step_eager()
    torch.cuda.synchronize()
    assert torch.equal(qa, qb) and torch.equal(dqa, dqb)
    assert not torch.equal(qa, q0)


@pytest.mark.gpu
def test_host_entry_points_multi_chunk(vc3b, cuda):
    """vc3_*_host stream 2^23-vector chunks over three CUDA streams: several
    chunks plus a ragged tail equal the device-buffer results word for word."""
    n = 3 * (1 << 22) + 777
    g = torch.Generator(device=cuda).manual_seed(11)
    va = torch.rand((n, 3), device=cuda, generator=g).mul_(2).sub_(1)
    vb = torch.rand((n, 3), device=cuda, generator=g).mul_(2).sub_(1)
    lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
    a_dev, b_dev = vc3b.compress(va, lay, pol), vc3b.compress(vb, lay, pol)
    a_host = vc3b.compress(va.cpu().numpy(), lay, pol)            # vc3_compress_host
    assert np.array_equal(a_host, a_dev.cpu().numpy())
    c_host = vc3b.add_compressed(a_host, b_dev.cpu().numpy(), lay, pol)  # vc3_add_compressed_host
    assert np.array_equal(c_host, vc3b.add_compressed(a_dev, b_dev, lay, pol).cpu().numpy())
    d_host = vc3b.decompress(c_host, lay)                            # vc3_decompress_host
    d_dev = vc3b.decompress(torch.from_numpy(c_host.view(np.int64)).to(cuda).view(torch.uint64), lay)
    assert np.array_equal(d_host.view(np.uint32), d_dev.cpu().numpy().view(np.uint32))


@pytest.mark.gpu
def test_empty_inputs_everywhere(vc3b, cuda, tmp_path):
    """n = 0 through every entry point, host and device arrays."""
    from paper_2003_02633_b200 import ops, stream

    lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
    ev = torch.empty((0, 3), dtype=torch.float32, device=cuda)
    ew = torch.empty(0, dtype=torch.uint64, device=cuda)
    assert vc3b.compress(ev).numel() == 0 and vc3b.decompress(ew).shape == (0, 3)
    assert vc3b.compress(np.empty((0, 3), np.float32)).shape == (0,)
    assert vc3b.decompress(np.empty(0, np.uint64)).shape == (0, 3)
    assert vc3b.add_compressed(ew, ew).numel() == 0
    assert vc3b.add_compressed(np.empty(0, np.uint64), np.empty(0, np.uint64)).shape == (0,)
    assert vc3b.add_raw(np.empty((0, 3), np.float32), np.empty((0, 3), np.float32)).shape == (0, 3)
    assert ops.axpy(2.0, ew, ew).numel() == 0
    q, dq = ops.rk_stage(0.5, 0.5, 0.1, ew.clone(), ew.clone(), ew)
    assert q.numel() == 0 and dq.numel() == 0
    assert vc3b.magnitude_event_counts(ev) == (0, 0)
    stream.write_stream(tmp_path / "e.vc3", ew)
    words, lay2 = stream.read_stream(tmp_path / "e.vc3")
    assert words.size == 0 and lay2 == lay and (tmp_path / "e.vc3").stat().st_size == 20


@pytest.mark.gpu
@pytest.mark.parametrize("lname,code", [("17_18", "SSS"), ("17_18", "SDS"), ("base_16_16", "DDD"),
                                        ("wide_10_25", "SSS")])
def test_compress_with_events_fused(golden, vc3b, cuda, lname, code):
    """K8: the fused pass gives the compress words and the event counts of the
    separate kernels (and the reference's counts on its fixtures)."""
    from paper_2003_02633_b200 import codec

    lay, pol = layout_by_name(lname), policy_by_code(code)
    for key in ("vec_mixed", "vec_edge"):
        v = golden[key]
        words, ev = codec.compress_with_events(v, lay, pol)
        assert np.array_equal(words, vc3b.compress(v, lay, pol))
        assert ev == vc3b.magnitude_event_counts(v, lay)
        if lname == "17_18":
            assert ev == tuple(golden["mag_events_" + key[4:]])
    tv = torch.from_numpy(golden["vec_mixed"]).to(cuda)
    dw, dev_ev = codec.compress_with_events(tv, lay, pol)
    assert dw.is_cuda and dev_ev == vc3b.magnitude_event_counts(golden["vec_mixed"], lay)
