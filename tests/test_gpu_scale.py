"""Parity at scale in the regular GPU suite: 2^26 vectors
per input family against the C oracle, both numerics modes.  Needs a B200.

* compress (all-single): bit-exact;
* fused add, VC3_EXACT: bit-exact; VC3_CONTRACT: every differing word within
  one bucket / one magnitude step, rate reported;
* axpy, VC3_EXACT: bit-exact;
* decompress of random words, VC3_EXACT: bit-exact; VC3_CONTRACT: <= 1 ulp.
The opt-in soak (tests/test_soak.py, VC3_SOAK=<log2>) runs the same checks on
billions of vectors.
"""

import json
import os
import time

import numpy as np
import pytest
import torch

from conftest import layout_by_name, policy_by_code
from test_soak import _vectors

pytestmark = pytest.mark.gpu
LOG2 = int(os.environ.get("VC3_SCALE_LOG2", "26"))


def _dev_words(w, cuda):
    return torch.from_numpy(w.view(np.int64)).to(cuda).view(torch.uint64)


def _deltas(got, want, lay):
    d = got != want
    t, p = lay.theta_bits, lay.phi_bits
    g, w = got[d].astype(np.int64), want[d].astype(np.int64)
    tm, pm = (1 << t) - 1, (1 << p) - 1
    dt = np.abs((g & tm) - (w & tm))
    dt = np.minimum(dt, tm + 1 - dt)
    dp = np.abs(((g >> t) & pm) - ((w >> t) & pm))
    df = np.abs((g >> (t + p)) - (w >> (t + p)))
    return int(d.sum()), (int(dt.max()) if d.any() else 0, int(dp.max()) if d.any() else 0,
                          int(df.max()) if d.any() else 0)


def test_parity_at_scale(vc3b, oracle, cuda):
    from paper_2003_02633_b200 import ops

    lay, sss = layout_by_name("17_18"), policy_by_code("SSS")
    nthr = oracle.default_threads()
    n = 1 << LOG2
    report = {"vectors_per_family": n}
    t0 = time.time()
    for ki, kind in enumerate(("cube", "loguniform", "edge")):
        g = np.random.Generator(np.random.Philox(key=(LOG2, 100 + ki)))
        v = _vectors(g, kind, n)
        w = vc3b.compress(torch.from_numpy(v).to(cuda), lay, sss).cpu().numpy()
        mis_c = int((w != oracle.compress(v, lay, sss, nthreads=nthr)).sum())
        del v
        w2 = np.roll(w, 1)
        want = oracle.add_compressed(w, w2, lay, sss, nthreads=nthr)
        da, db = _dev_words(w, cuda), _dev_words(w2, cuda)
        mis_ex = int((ops.add_compressed(da, db, lay, sss).cpu().numpy() != want).sum())
        ties, (dt, dp, df) = _deltas(ops.add_compressed(da, db, lay, sss, mode="contract").cpu().numpy(),
                                     want, lay)
        want_ax = oracle.axpy(-0.75, w, w2, lay, sss, nthreads=nthr)
        mis_ax = int((ops.axpy(-0.75, da, db, lay, sss).cpu().numpy() != want_ax).sum())
        report[kind] = {"compress_mismatches": mis_c, "add_exact_mismatches": mis_ex,
                        "add_contract_ties": ties, "tie_max_deltas": [dt, dp, df],
                        "axpy_exact_mismatches": mis_ax}
        del da, db
        assert mis_c == 0 and mis_ex == 0 and mis_ax == 0, report
        assert max(dt, dp, df) <= 1 and ties <= 1e-5 * n, report
    g = np.random.Generator(np.random.Philox(key=(LOG2, 199)))
    wr = g.integers(0, 2 ** 64, n, dtype=np.uint64)
    want = oracle.decompress(wr, lay, nthreads=nthr).view(np.int32).astype(np.int64)
    dw = _dev_words(wr, cuda)
    got_ex = vc3b.decompress(dw, lay).cpu().numpy().view(np.int32).astype(np.int64)
    got_ct = vc3b.decompress(dw, lay, mode="contract").cpu().numpy().view(np.int32).astype(np.int64)
    ulp_ct = np.abs(got_ct - want)
    report["decompress_random_words"] = {"exact_mismatches": int((got_ex != want).sum()),
                                         "contract_max_ulp": int(ulp_ct.max()),
                                         "contract_differing": int((ulp_ct != 0).sum())}
    report["seconds"] = round(time.time() - t0, 1)
    print("SCALE", json.dumps(report))
    assert report["decompress_random_words"]["exact_mismatches"] == 0, report
    assert report["decompress_random_words"]["contract_max_ulp"] <= 1, report
