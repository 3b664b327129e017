"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the reference package ``vc3`` (/root/reference/pkg/src/vc3) and
records inputs and outputs of its public API on the reference tests' own
fixtures (pkg/tests/conftest.py:18-34), the SURVEY Appendix B known-answer
vectors, adversarial edge cases and random words.  The fixtures pin both the C
oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

import vc3
from vc3 import analysis, bench
from vc3.layout import (
    ALL_SINGLE_POLICY,
    DEFAULT_LAYOUT,
    DEFAULT_POLICY,
    LAYOUT_16_17,
    LAYOUT_17_17,
    LAYOUT_BASE_16_16,
    ORACLE_POLICY,
    BitLayout,
    PrecisionPolicy,
)

OUT = Path(__file__).resolve().parent

LAYOUTS = {
    "17_18": DEFAULT_LAYOUT,
    "base_16_16": LAYOUT_BASE_16_16,
    "16_17": LAYOUT_16_17,
    "17_17": LAYOUT_17_17,
    "wide_10_25": BitLayout(0, 7, 22, 10, 25, 80),  # direct (no-table) decode path
}
ALL_POLICIES = {
    f"{t[0].upper()}{p[0].upper()}{q[0].upper()}": PrecisionPolicy(t, p, q)
    for t in ("single", "double") for p in ("single", "double") for q in ("single", "double")
}


def mixed_vectors():
    # pkg/tests/conftest.py:23-34
    g = np.random.Generator(np.random.Philox(key=(404, 0)))
    v = g.normal(size=(20_000, 3))
    scales = 10.0 ** g.uniform(-6, 6, size=20_000)
    v = (v * scales[:, None]).astype(np.float32)
    axes = np.array([
        [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
        [0, 0, 0], [1, 1, 1], [3, 4, 0], [-2, 0, 2],
    ], dtype=np.float32)
    return np.concatenate([axes, v])


def kat_vectors():
    # SURVEY.md Appendix B rows
    return np.array([
        [1, 0, 0], [0, 0, 1], [1, 1, 1], [3, 4, 0], [0, 0, 0], [-1, -0.0, 0],
        [0, 0, -2], [1e-30, 2e-30, -3e-30], [1e20, -1e20, 5e19], [-0.5, 0.25, -0.125],
    ], dtype=np.float32)


def edge_vectors():
    """Adversarial inputs: signed zeros, subnormals, f32 square under/overflow,
    rails, axis and near-pole directions, exact ties of |x| == |y|."""
    f = np.float32
    tiny = np.finfo(np.float32).tiny
    mx = np.finfo(np.float32).max
    sub = f(1e-45)
    rows = [
        [0, 0, 0], [-0.0, 0, 0], [0, -0.0, 0], [0, 0, -0.0], [-0.0, -0.0, -0.0],
        [sub, 0, 0], [0, sub, 0], [0, 0, sub], [-sub, -sub, sub], [sub, -sub, 0],
        [tiny, tiny, tiny], [tiny / 4, 0, tiny], [1e-38, -1e-39, 1e-40],
        [mx, 0, 0], [0, mx, 0], [0, 0, -mx], [mx, mx, mx], [-mx, mx, -mx],
        [3e38, 3e38, 0], [1e19, 1e19, 1e19], [1.9e19, 0, 0], [1.8446743e19, 0, 0],
        [2.0 ** -78, 0, 0], [2.0 ** -79, 0, 0], [2.0 ** -77, 2.0 ** -77, 0],
        [2.0 ** 46, 0, 0], [2.0 ** 47, 0, 0], [1.4e14, 0, 0],
        [1, 1, 0], [-1, 1, 0], [-1, -1, 0], [1, -1, 0], [2, 2, 2], [-3, -3, 3],
        [1, 1e-30, 0], [-1, 1e-30, 0], [-1, -1e-30, 0], [1, 0, 1e-30],
        [1e-30, 0, 1], [0, 1e-30, -1], [-1e-20, 1e-20, 5], [1e-7, 0, -1],
        [0.1, 0.2, 0.3], [-0.7, 0.7, 0.1], [5, 0, 0], [0, 0, 3], [0, 0, 1536],
        [0, 0, 0.015625], [0, 0, 5], [0, 0, -5], [1e-20, 1e-20, 1e-20],
        [-1.5e-23, 2.5e-23, 1e-22], [65504, -65504, 1], [123456.79, -0.001, 42],
    ]
    v = np.array(rows, dtype=np.float64)
    with np.errstate(over="ignore"):
        return v.astype(np.float32)


def main():
    d = {}
    mixed = mixed_vectors()
    kat = kat_vectors()
    edge = edge_vectors()
    sphere = analysis.sample(analysis.SampleDomain("unit_sphere", 5_000, 71))
    cube = analysis.sample(analysis.SampleDomain("cube", 5_000, 5))
    # magnitude-spread cube (log-uniform magnitudes, like BASELINE config C1)
    g = np.random.Generator(np.random.Philox(key=(1, 0)))
    spread = (cube.astype(np.float64) * (10.0 ** g.uniform(-6, 6, 5_000))[:, None]).astype(np.float32)

    vec_sets = {"mixed": mixed, "kat": kat, "edge": edge, "sphere": sphere, "cube": cube,
                "spread": spread}
    for name, v in vec_sets.items():
        d[f"vec_{name}"] = v

    # compress: every policy on the default layout; 3 policies on the others
    for lname, lay in LAYOUTS.items():
        pols = ALL_POLICIES if lname == "17_18" else {
            "SDS": DEFAULT_POLICY, "SSS": ALL_SINGLE_POLICY, "DDD": ORACLE_POLICY}
        for pname, pol in pols.items():
            for vname, v in vec_sets.items():
                if lname != "17_18" and vname in ("sphere", "cube"):
                    continue
                if lname != "17_18" and vname == "mixed":
                    v = v[:5010]
                d[f"cw_{lname}_{pname}_{vname}"] = vc3.compress(v, lay, pol)

    # decompress: codec words + random words (pkg/tests/test_codec.py:142-147)
    g = np.random.Generator(np.random.Philox(99))
    rand_words = g.integers(0, 2 ** 64, 20_000, dtype=np.uint64)
    d["words_random"] = rand_words
    for lname, lay in LAYOUTS.items():
        d[f"dv_{lname}_random"] = vc3.decompress(rand_words, lay)
        for pname in ("SSS", "SDS"):
            for vname in ("mixed", "edge", "kat", "spread"):
                key = f"cw_{lname}_{pname}_{vname}"
                if vname == "mixed":
                    d[key] = d[key][:5010]
                d[f"dv_{lname}_{pname}_{vname}"] = vc3.decompress(d[key], lay)

    # fused add (pkg/tests/test_bench.py:40-53 inputs) + Appendix B add KAT
    g = np.random.Generator(np.random.Philox(21))
    va = g.normal(size=(8_000, 3)).astype(np.float32)
    vb = g.normal(size=(8_000, 3)).astype(np.float32)
    d["add_va"], d["add_vb"] = va, vb
    for lname, pname, lay, pol in [("17_18", "SSS", DEFAULT_LAYOUT, ALL_SINGLE_POLICY),
                                   ("17_18", "SDS", DEFAULT_LAYOUT, DEFAULT_POLICY),
                                   ("17_18", "DDD", DEFAULT_LAYOUT, ORACLE_POLICY),
                                   ("base_16_16", "SSS", LAYOUT_BASE_16_16, ALL_SINGLE_POLICY),
                                   ("wide_10_25", "SSS", LAYOUTS["wide_10_25"], ALL_SINGLE_POLICY)]:
        a = vc3.compress(va, lay, pol)
        b = vc3.compress(vb, lay, pol)
        d[f"add_a_{lname}_{pname}"] = a
        d[f"add_b_{lname}_{pname}"] = b
        d[f"add_c_{lname}_{pname}"] = bench.add_compressed(a, b, lay, pol)
    # adversarial words summed (random words + each other, reversed)
    d["add_c_random_SSS"] = bench.add_compressed(rand_words[:10_000], rand_words[10_000:],
                                                 DEFAULT_LAYOUT, ALL_SINGLE_POLICY)
    kw = vc3.compress(kat, DEFAULT_LAYOUT, ALL_SINGLE_POLICY)
    d["add_c_kat_SSS"] = bench.add_compressed(kw[:4], kw[3::-1], DEFAULT_LAYOUT, ALL_SINGLE_POLICY)
    d["add_raw_c"] = bench.add_raw(va, vb)

    # pieces on the mixed and edge sets
    pv = np.concatenate([mixed[:4000], edge])
    d["piece_vec"] = pv
    for pname in ("SDS", "SSS", "DDD", "DSS"):
        pol = ALL_POLICIES[pname]
        r, th, ph = vc3.to_spherical(pv, pol)
        d[f"sph_r_{pname}"], d[f"sph_th_{pname}"], d[f"sph_ph_{pname}"] = r, th, ph
        nt, nph = vc3.quantize_angles(th, ph, DEFAULT_LAYOUT, pol)
        d[f"q_nt_{pname}"], d[f"q_nph_{pname}"] = nt, nph
    g = np.random.Generator(np.random.Philox(17))
    qth = g.uniform(-np.pi * 1.0001, np.pi * 1.0001, 8_000)
    qph = g.uniform(-1e-3, np.pi * 1.0001, 8_000)
    d["qin_th"], d["qin_ph"] = qth, qph
    for pname in ("SSS", "DDD"):
        nt, nph = vc3.quantize_angles(qth, qph, DEFAULT_LAYOUT, ALL_POLICIES[pname])
        d[f"qout_nt_{pname}"], d[f"qout_nph_{pname}"] = nt, nph
    dt, dp = vc3.dequantize_angles(np.arange(0, 1 << 18, 61), np.arange(0, 1 << 18, 61) >> 1,
                                   DEFAULT_LAYOUT)
    d["deq_th"], d["deq_ph"] = dt, dp
    rr = np.concatenate([
        np.sqrt((mixed[:4000].astype(np.float64) ** 2).sum(axis=1)),
        10.0 ** np.random.Generator(np.random.Philox(3)).uniform(-45, 39, 5_000),
        [0.0, 1.0, 3.0, 5.0, 2.0 ** -100, 2.0 ** -78, 1e30, 1e38, 3.5e38, 1e300],
    ])
    d["mag_r"] = rr
    for lname, lay in LAYOUTS.items():
        f = np.atleast_1d(np.asarray(vc3.encode_magnitude(rr, lay), dtype=np.uint64))
        d[f"mag_field_{lname}"] = f
        d[f"mag_dec_{lname}"] = vc3.decode_magnitude(f, lay)
    d["mag_events_mixed"] = np.array(vc3.magnitude_event_counts(mixed, DEFAULT_LAYOUT))
    d["mag_events_edge"] = np.array(vc3.magnitude_event_counts(edge, DEFAULT_LAYOUT))

    # error statistics (analysis.py:157-167)
    for pname in ("SDS", "DDD"):
        for norm in (False, True):
            st = analysis.error_study(analysis.SampleDomain("unit_sphere", 60_000, 21),
                                      DEFAULT_LAYOUT, ALL_POLICIES[pname], normalised=norm)
            d[f"err_sphere_{pname}_{int(norm)}"] = np.array(
                [st.mean, st.max, st.stddev, st.count], dtype=np.float64)

    # K7 variants (analysis.py:259-417): per-vector indices and reconstructions
    # exactly as compand_study / split_sweep compute them, plus the studies.
    vv = np.concatenate([sphere, mixed[:2000]])
    d["var_vec"] = vv
    r, th, ph = vc3.to_spherical(vv, ORACLE_POLICY)
    rh = vc3.decode_magnitude(vc3.encode_magnitude(r, DEFAULT_LAYOUT), DEFAULT_LAYOUT).astype(np.float64)
    ntmax, npmax = DEFAULT_LAYOUT.n_theta_max, DEFAULT_LAYOUT.n_phi_max
    comps = {"uniform": analysis.Compander("uniform"), "cosine": analysis.Compander("cosine"),
             "tanh05": analysis.Compander("tanh", 0.5), "tanh2": analysis.Compander("tanh", 2.0)}
    for cname, comp in comps.items():
        nt = comp.encode((th + np.pi) / (2.0 * np.pi), ntmax)
        nph = comp.encode(ph / np.pi, npmax)
        th2 = 2.0 * np.pi * comp.decode(nt, ntmax) - np.pi
        ph2 = np.pi * comp.decode(nph, npmax)
        sp = np.sin(ph2)
        vh = np.stack([rh * np.cos(th2) * sp, rh * np.sin(th2) * sp, rh * np.cos(ph2)],
                      axis=1).astype(np.float32)
        d[f"cmp_{cname}_nt"], d[f"cmp_{cname}_nph"], d[f"cmp_{cname}_vh"] = nt, nph, vh
        st = analysis.compand_study(analysis.SampleDomain("unit_sphere", 100_000, 11), comp)
        d[f"cmp_{cname}_study"] = np.array([st.mean, st.max, st.stddev, st.count])
    splits = [1 << 16, 98304, 1 << 17, 196608, 1 << 18]
    d["split_values"] = np.array(splits)
    for s_ in splits:
        cfg = analysis.SplitConfig(35, s_ - 1)
        nt, nph = analysis._quantize_free(th, ph, cfg.n_theta_max, cfg.n_phi_max)
        J = analysis.joint_encode(nt, nph, cfg)
        nt2, nph2 = analysis.joint_decode(J, cfg)
        th2 = np.pi * (2.0 * nt2 / cfg.n_theta_max - 1.0)
        ph2 = np.pi * nph2 / cfg.n_phi_max
        sp = np.sin(ph2)
        vh = np.stack([rh * np.cos(th2) * sp, rh * np.sin(th2) * sp, rh * np.cos(ph2)],
                      axis=1).astype(np.float32)
        d[f"split_{s_}_J"], d[f"split_{s_}_vh"] = J, vh
    rows = analysis.split_sweep(35, splits, analysis.SampleDomain("unit_sphere", 100_000, 7))
    d["split_study"] = np.array([[st.mean, st.max, st.stddev, st.count] for _, st in rows])

    # characterisation studies (analysis.py:236-254, 446-486)
    d["binmiss_sphere"] = np.array(analysis.bin_miss_study(
        analysis.SampleDomain("unit_sphere", 300_000, 3)))
    d["binmiss_cube"] = np.array(analysis.bin_miss_study(analysis.SampleDomain("cube", 300_000, 3)))
    for pname in ("SDS", "DDD", "SSS"):
        r = analysis.idempotence_study(analysis.SampleDomain("unit_sphere", 300_000, 4),
                                       DEFAULT_LAYOUT, ALL_POLICIES[pname])
        d[f"idem_{pname}"] = np.array([r.word_miss_fraction, r.predicted_bound,
                                       r.third_cycle_stable_fraction, r.count])

    # VC3C stream bytes (stream.py:1-87) and CSV text
    import io as _io
    from vc3 import stream as _stream
    for lname in ("17_18", "base_16_16"):
        buf = _io.BytesIO()
        _stream.write_stream(buf, d[f"cw_{lname}_SSS_kat"], LAYOUTS[lname])
        d[f"stream_{lname}"] = np.frombuffer(buf.getvalue(), dtype=np.uint8)
    sbuf = _io.StringIO()
    _stream.write_csv(sbuf, edge)
    d["csv_edge"] = np.frombuffer(sbuf.getvalue().encode(), dtype=np.uint8)

    # anisotropy map, precision comparison, Smith bins (analysis.py:170-233, 420-443)
    means, counts, _, _ = analysis.anisotropy_map(DEFAULT_LAYOUT, ORACLE_POLICY, (8, 4), 200_000, 3)
    d["aniso_means"], d["aniso_counts"] = means, counts
    rows = analysis.precision_comparison(100_000, 1)
    d["prec_cmp"] = np.array([[r["mean"], r["max"], r["stddev"], r["count"]] for r in rows])
    smith = []
    for phi, npm, tau in ((0.3, 64, 0.05), (1.5, 1000, 0.01), (2.9, 131071, 1e-4), (1.0, 8, 0.5)):
        smith.append(analysis.smith_theta_bins(phi, npm, tau))
    d["smith_bins"] = np.array(smith)

    np.savez_compressed(OUT / "golden.npz", **d)
    total = sum(v.nbytes for v in d.values())
    print(f"wrote {len(d)} arrays ({total / 1e6:.1f} MB raw) to {OUT / 'golden.npz'}")


if __name__ == "__main__":
    main()
