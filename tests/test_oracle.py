"""Pin the C oracle (oracle/vc3_oracle.c) to the reference's own outputs.

The golden fixtures were produced by importing the reference package
(tests/golden/make_golden.py).  Everything here is bit-exact: the oracle runs
the reference's operation sequence with the same libm, so any difference is
a restatement bug.  CPU only.
"""

import numpy as np
import pytest

from conftest import LAYOUT_NAMES, layout_by_name, policy_by_code

VEC_SETS = ["mixed", "kat", "edge", "sphere", "cube", "spread"]


def test_compress_all_policies_default_layout(golden, oracle):
    lay = layout_by_name("17_18")
    for code in ["SSS", "SSD", "SDS", "SDD", "DSS", "DSD", "DDS", "DDD"]:
        for vname in VEC_SETS:
            want = golden[f"cw_17_18_{code}_{vname}"]
            got = oracle.compress(golden[f"vec_{vname}"][: want.size], lay, policy_by_code(code))
            assert np.array_equal(got, want), (code, vname, int(np.sum(got != want)))


@pytest.mark.parametrize("lname", LAYOUT_NAMES[1:])
def test_compress_other_layouts(golden, oracle, lname):
    lay = layout_by_name(lname)
    for code in ["SDS", "SSS", "DDD"]:
        for vname in ["mixed", "kat", "edge", "spread"]:
            want = golden[f"cw_{lname}_{code}_{vname}"]
            v = golden[f"vec_{vname}"][: want.size]
            assert np.array_equal(oracle.compress(v, lay, policy_by_code(code)), want)


@pytest.mark.parametrize("lname", LAYOUT_NAMES)
def test_decompress(golden, oracle, lname):
    lay = layout_by_name(lname)
    got = oracle.decompress(golden["words_random"], lay)
    assert np.array_equal(got.view(np.uint32), golden[f"dv_{lname}_random"].view(np.uint32))
    for code in ("SSS", "SDS"):
        for vname in ("mixed", "edge", "kat", "spread"):
            words = golden[f"cw_{lname}_{code}_{vname}"]
            want = golden[f"dv_{lname}_{code}_{vname}"]
            assert np.array_equal(oracle.decompress(words, lay).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("key,lname,code", [
    ("17_18_SSS", "17_18", "SSS"), ("17_18_SDS", "17_18", "SDS"), ("17_18_DDD", "17_18", "DDD"),
    ("base_16_16_SSS", "base_16_16", "SSS"), ("wide_10_25_SSS", "wide_10_25", "SSS")])
def test_add_compressed(golden, oracle, key, lname, code):
    lay, pol = layout_by_name(lname), policy_by_code(code)
    a, b = golden[f"add_a_{key}"], golden[f"add_b_{key}"]
    assert np.array_equal(oracle.compress(golden["add_va"], lay, pol), a)
    assert np.array_equal(oracle.add_compressed(a, b, lay, pol), golden[f"add_c_{key}"])


def test_add_compressed_adversarial_and_kat(golden, oracle):
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    w = golden["words_random"]
    assert np.array_equal(oracle.add_compressed(w[:10_000], w[10_000:], lay, pol),
                          golden["add_c_random_SSS"])
    kw = golden["cw_17_18_SSS_kat"]
    got = oracle.add_compressed(kw[:4], kw[3::-1].copy(), lay, pol)
    assert np.array_equal(got, golden["add_c_kat_SSS"])
    # SURVEY Appendix B
    assert [hex(x) for x in got] == ["0xa4d413d400028000", "0xa27311b9913e7fff",
                                     "0xa27311b9913e7fff", "0xa4d413d400028000"]


def test_add_raw(golden, oracle):
    got = oracle.add_raw(golden["add_va"], golden["add_vb"])
    assert np.array_equal(got, golden["add_raw_c"])


def test_pieces(golden, oracle):
    lay = layout_by_name("17_18")
    pv = golden["piece_vec"]
    for code in ("SDS", "SSS", "DDD", "DSS"):
        pol = policy_by_code(code)
        r, th, ph = oracle.to_spherical(pv, pol)
        assert np.array_equal(r, golden[f"sph_r_{code}"])
        assert np.array_equal(th, golden[f"sph_th_{code}"])
        assert np.array_equal(ph, golden[f"sph_ph_{code}"])
        nt, nph = oracle.quantize_angles(th, ph, lay, pol)
        assert np.array_equal(nt, golden[f"q_nt_{code}"])
        assert np.array_equal(nph, golden[f"q_nph_{code}"])
    for code in ("SSS", "DDD"):
        nt, nph = oracle.quantize_angles(golden["qin_th"], golden["qin_ph"], lay, policy_by_code(code))
        assert np.array_equal(nt, golden[f"qout_nt_{code}"])
        assert np.array_equal(nph, golden[f"qout_nph_{code}"])


@pytest.mark.parametrize("lname", LAYOUT_NAMES)
def test_magnitude(golden, oracle, lname):
    lay = layout_by_name(lname)
    f = oracle.encode_magnitude(golden["mag_r"], lay)
    assert np.array_equal(f.astype(np.uint64), golden[f"mag_field_{lname}"])
    d = oracle.decode_magnitude(f, lay)
    assert np.array_equal(d.view(np.uint32), golden[f"mag_dec_{lname}"].view(np.uint32))


def test_appendix_b_kats(golden, oracle):
    lay = layout_by_name("17_18")
    kat = golden["vec_kat"]
    want = {
        "SDS": [0xa000000400020000, 0xa000000000020000, 0xa176cf626ec67fff, 0xa480000400029720, 0,
                0xa00000040003ffff, 0xa2000007fffe0000, 0x40000065e72b46f, 0xfdfffffb22758000,
                0x9e4a91dc8f6bb46f],
        "SSS": [0xa000000400020000, 0xa000000000020000, 0xa176cf626ec67fff, 0xa480000400029720, 0,
                0xa00000040003ffff, 0xa2000007fffe0000, 0x40000000002b46f, 0xfdfffffc00018000,
                0x9e4a91dc8f6bb46f],
        "DDD": [0xa000000400020000, 0xa000000000020000, 0xa176cf626ec67fff, 0xa480000400029720, 0,
                0xa000000400000000, 0xa2000007fffe0000, 0x40000065e72b46f, 0xfdfffffb22758000,
                0x9e4a91dc8f6bb46f],
    }
    for code, words in want.items():
        assert [int(x) for x in oracle.compress(kat, lay, policy_by_code(code))] == words
    dec = oracle.decompress(oracle.compress(kat, lay, policy_by_code("SSS")), lay).view(np.uint32)
    assert [tuple(int(x) for x in row) for row in dec[[0, 5, 7, 8]]] == [
        (0x3f800000, 0x3749100d, 0xb749103f), (0xbf800000, 0x250d3132, 0xb749103f),
        (0, 0, 0x18800000), (0x56b5055c, 0xd6b50487, 0xcec9103e)]


def test_trig_kats(oracle):
    # pkg/tests/test_trig.py:14-20, 46-50
    f32 = np.float32
    assert oracle.atan2_f32(0, 0) == 0.0
    assert oracle.atan2_f32(0, -2) == f32(np.pi)
    assert oracle.atan2_f32(3, 0) == f32(np.pi / 2)
    assert oracle.atan2_f32(-3, 0) == -f32(np.pi / 2)
    assert oracle.acos_f32(1) == 0.0
    assert oracle.acos_f32(-1) == f32(np.pi)
    assert oracle.acos_f32(0) == f32(np.pi / 2)


def test_threaded_equals_serial(golden, oracle):
    lay, pol = layout_by_name("17_18"), policy_by_code("SSS")
    a, b = golden["add_a_17_18_SSS"], golden["add_b_17_18_SSS"]
    assert np.array_equal(oracle.add_compressed(a, b, lay, pol, nthreads=4),
                          oracle.add_compressed(a, b, lay, pol, nthreads=1))
    v = golden["vec_mixed"]
    assert np.array_equal(oracle.compress(v, lay, pol, nthreads=3), oracle.compress(v, lay, pol))


COMPANDERS = {"uniform": ("uniform", 0.5), "cosine": ("cosine", 0.5),
              "tanh05": ("tanh", 0.5), "tanh2": ("tanh", 2.0)}


@pytest.mark.parametrize("cname", list(COMPANDERS))
def test_variant_oracle_compand(golden, oracle, cname):
    import vc3_variants

    kind, gamma = COMPANDERS[cname]
    nt, nph, vh = vc3_variants.compand_round_trip(golden["var_vec"], layout_by_name("17_18"),
                                                  kind, gamma)
    assert np.array_equal(nt, golden[f"cmp_{cname}_nt"])
    assert np.array_equal(nph, golden[f"cmp_{cname}_nph"])
    assert np.array_equal(vh.view(np.uint32), golden[f"cmp_{cname}_vh"].view(np.uint32))


def test_variant_oracle_split(golden, oracle):
    import vc3_variants

    for s in golden["split_values"]:
        J, vh = vc3_variants.split_round_trip(golden["var_vec"], layout_by_name("17_18"), 35,
                                              int(s) - 1)
        assert np.array_equal(J, golden[f"split_{s}_J"])
        assert np.array_equal(vh.view(np.uint32), golden[f"split_{s}_vh"].view(np.uint32))
