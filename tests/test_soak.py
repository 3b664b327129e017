"""Soak parity run: billions of vectors through the GPU kernels against the C
oracle on every host core.  Skipped unless VC3_SOAK=<log2 total vectors per
case> is set (e.g. VC3_SOAK=32); the counts it prints are recorded in
profiles/r01_soak.json.  All-single policy (the benchmark's): compressed
words, fused-add words and RK-stage words must match bit for bit; the default
policy may differ only by single-bin ties; decoded components of random words
must be bit-exact."""

import json
import os
import time

import numpy as np
import pytest

from conftest import layout_by_name, policy_by_code

SOAK = int(os.environ.get("VC3_SOAK", "0"))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(SOAK == 0, reason="set VC3_SOAK=<log2 vectors>")]
CHUNK = 1 << 25


def _vectors(g, kind, n):
    if kind == "cube":
        return g.uniform(-1.0, 1.0, (n, 3)).astype(np.float32)
    if kind == "loguniform":
        d = g.normal(size=(n, 3))
        return (d * 10.0 ** g.uniform(-20, 12, (n, 1))).astype(np.float32)
    # edge: axis-aligned, tiny/huge magnitudes, exact zeros, near-pole and near-seam angles
    v = g.normal(size=(n, 3)).astype(np.float32)
    sel = g.integers(0, 6, n)
    v[sel == 0, 1:] = 0.0
    v[sel == 1, :2] *= np.float32(1e-6)
    v[sel == 2, 1] = np.float32(0.0) * v[sel == 2, 1]
    v[sel == 2, 0] = -np.abs(v[sel == 2, 0])
    v[sel == 3] *= np.float32(1e-30)
    v[sel == 4] *= np.float32(1e20)
    v[sel == 5] = 0.0
    return v


def test_soak(vc3b, oracle, cuda):
    import torch

    lay = layout_by_name("17_18")
    sss, sds = policy_by_code("SSS"), policy_by_code("SDS")
    nthr = oracle.default_threads()
    total = 1 << SOAK
    report = {"vectors_per_case": total, "threads": nthr}
    details = []
    t0 = time.time()
    for ki, kind in enumerate(("cube", "loguniform", "edge")):
        g = np.random.Generator(np.random.Philox(key=(SOAK, ki)))
        mis_sss = ties_sds = mis_add = ties_ct = 0
        dmax_ct = [0, 0, 0]
        for _ in range(max(1, total // CHUNK)):
            v = _vectors(g, kind, CHUNK)
            tv = torch.from_numpy(v).to(cuda)
            w = vc3b.compress(tv, lay, sss).cpu().numpy()
            mis_sss += int((w != oracle.compress(v, lay, sss, nthreads=nthr)).sum())
            wd = vc3b.compress(tv, lay, sds).cpu().numpy()
            ties_sds += int((wd != oracle.compress(v, lay, sds, nthreads=nthr)).sum())
            w2 = np.roll(w, 1)
            c = vc3b.add_compressed(torch.from_numpy(w.view(np.int64)).to(cuda).view(torch.uint64),
                                    torch.from_numpy(w2.view(np.int64)).to(cuda).view(torch.uint64),
                                    lay, sss).cpu().numpy()
            want_c = oracle.add_compressed(w, w2, lay, sss, nthreads=nthr)
            # the north-star contract mode: one-bin ties only
            from paper_2003_02633_b200 import ops

            c_ct = ops.add_compressed(torch.from_numpy(w.view(np.int64)).to(cuda).view(torch.uint64),
                                      torch.from_numpy(w2.view(np.int64)).to(cuda).view(torch.uint64),
                                      lay, sss, mode="contract").cpu().numpy().view(np.uint64)
            dct = c_ct != want_c
            ties_ct += int(dct.sum())
            if dct.any():
                gg, ww = c_ct[dct].astype(np.int64), want_c[dct].astype(np.int64)
                tm, pm = int(lay.n_theta_max), int(lay.n_phi_max)
                dt_ = np.abs((gg & tm) - (ww & tm))
                dmax_ct[0] = max(dmax_ct[0], int(np.minimum(dt_, tm + 1 - dt_).max()))
                dmax_ct[1] = max(dmax_ct[1], int(np.abs(((gg >> lay.theta_bits) & pm) - ((ww >> lay.theta_bits) & pm)).max()))
                dmax_ct[2] = max(dmax_ct[2], int(np.abs((gg >> (lay.theta_bits + lay.phi_bits))
                                                        - (ww >> (lay.theta_bits + lay.phi_bits))).max()))
            bad = np.nonzero(c != want_c)[0]
            mis_add += int(bad.size)
            for i in bad[:8]:
                # the field that moved, and the decoded operands (a 1-ulp decode
                # difference of the reference libm vs the table decode)
                ga, gb = vc3b.decompress(w[i:i + 1], lay), vc3b.decompress(w2[i:i + 1], lay)
                oa, ob = oracle.decompress(w[i:i + 1], lay), oracle.decompress(w2[i:i + 1], lay)
                details.append({"got": int(c[i]), "want": int(want_c[i]),
                                "a_decode_ulp_diff": (ga.view(np.int32) - oa.view(np.int32)).tolist(),
                                "b_decode_ulp_diff": (gb.view(np.int32) - ob.view(np.int32)).tolist(),
                                "dtheta": int(c[i] & lay.n_theta_max) - int(want_c[i] & lay.n_theta_max),
                                "dphi": int((c[i] >> lay.theta_bits) & lay.n_phi_max)
                                - int((want_c[i] >> lay.theta_bits) & lay.n_phi_max),
                                "dfield": int(c[i] >> (lay.theta_bits + lay.phi_bits))
                                - int(want_c[i] >> (lay.theta_bits + lay.phi_bits))})
        report[kind] = {"compress_all_single_mismatches": mis_sss, "compress_default_ties": ties_sds,
                        "fused_add_mismatches": mis_add, "fused_add_contract_ties": ties_ct,
                        "contract_tie_max_deltas": dmax_ct}
        report["fused_add_mismatch_details"] = details
        # compress and the fused add are bit-exact (the fused decodes take the
        # reference's tables near a float32 rounding boundary)
        assert mis_sss == 0, report
        assert mis_add == 0, report
        assert ties_sds <= 1e-4 * total, report
        assert max(dmax_ct) <= 1 and ties_ct <= 1e-6 * total, report
    # low-storage RK stage on equator vectors (the ICV field's w = 0: decoded z
    # ~ -1.2e-5 r, the decode's hardest case for the boundary test), 1/8 of
    # the vectors: words bit-exact vs the oracle composition
    g = np.random.Generator(np.random.Philox(key=(SOAK, 7)))
    mis_rk = 0
    for _ in range(max(1, total // CHUNK // 8)):
        v = g.normal(size=(3, CHUNK, 3)).astype(np.float32)
        v[:, :, 2] = 0.0
        q, dq, R = (oracle.compress(x, lay, sss, nthreads=nthr) for x in v)
        tq, tdq, tR = (torch.from_numpy(x.view(np.int64)).to(cuda).view(torch.uint64) for x in (q, dq, R))
        a, b, dt = np.float32(-0.41789047), np.float32(1.4965424), np.float32(1e-3)
        vc3b.rk_stage(a, b, dt, tq, tdq, tR, lay, sss)
        qd, dqd, Rd = (oracle.decompress(x, lay, nthreads=nthr) for x in (q, dq, R))
        dq_new = a * dqd + dt * Rd
        q_new = qd + b * dq_new
        mis_rk += int((tdq.cpu().numpy().view(np.uint64) != oracle.compress(dq_new, lay, sss, nthreads=nthr)).sum())
        mis_rk += int((tq.cpu().numpy().view(np.uint64) != oracle.compress(q_new, lay, sss, nthreads=nthr)).sum())
    report["rk_stage_equator"] = {"vectors": max(1, total // CHUNK // 8) * CHUNK, "word_mismatches": mis_rk}
    assert mis_rk == 0, report
    # decompress of random words
    g = np.random.Generator(np.random.Philox(key=(SOAK, 99)))
    exact = ulp_max = n_words = ulp_ct = 0
    for _ in range(max(1, total // CHUNK)):
        w = g.integers(0, 2 ** 64, CHUNK, dtype=np.uint64)
        got = vc3b.decompress(torch.from_numpy(w.view(np.int64)).to(cuda).view(torch.uint64), lay).cpu().numpy()
        want = oracle.decompress(w, lay, nthreads=nthr)
        same = got.view(np.uint32) == want.view(np.uint32)
        exact += int(same.sum())
        ia = got.view(np.int32).astype(np.int64)
        ib = want.view(np.int32).astype(np.int64)
        ia = np.where(ia < 0, -(2 ** 31) - ia, ia)
        ib = np.where(ib < 0, -(2 ** 31) - ib, ib)
        ulp_max = max(ulp_max, int(np.abs(ia - ib).max()))
        got_ct = vc3b.decompress(torch.from_numpy(w.view(np.int64)).to(cuda).view(torch.uint64), lay,
                                 mode="contract").cpu().numpy()
        ic = got_ct.view(np.int32).astype(np.int64)
        ic = np.where(ic < 0, -(2 ** 31) - ic, ic)
        ulp_ct = max(ulp_ct, int(np.abs(ic - ib).max()))
        n_words += CHUNK
    report["decompress_random_words"] = {"components": 3 * n_words, "exact": exact, "max_ulp": ulp_max,
                                         "contract_max_ulp": ulp_ct}
    report["seconds"] = round(time.time() - t0, 1)
    print("SOAK", json.dumps(report))
    assert ulp_max == 0 and exact == 3 * n_words, report
    assert ulp_ct <= 1, report
