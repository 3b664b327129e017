"""A/B of fused-add builds on one GPU: timing, bit-identity and tie statistics.

    python tools/fused_ab.py [--n LOG2] [--ref tools/libvc3_r1.so] [--steps K]

Loads the current library (lib/libvc3_b200.so) and a reference build (the
round-1 library by default) in the same process, generates 2^n cube vectors
on the device (as bench.py), compresses them, and for each fused operation:
  * times exact and contract modes of the current build and the reference
    build's exact kernel (CUDA events, L2-flushing working set);
  * checks current-exact == reference-exact bit for bit on all 2^n pairs;
  * reports the contract-mode words that differ from the exact words:
    rate and the largest theta / phi / magnitude-field deltas.
Prints one JSON object.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2003_02633_b200 import _native  # noqa: E402
import paper_2003_02633_b200 as vc3b  # noqa: E402


def load_ref(path):
    lib = ctypes.CDLL(str(path))
    for name in ("vc3_add_compressed", "vc3_compress", "vc3_decompress", "vc3_axpy", "vc3_rk_stage"):
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = _native.SIGNATURES[name]
    return lib


def timeit(fn, steps, stream):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / steps


def word_deltas(x: torch.Tensor, y: torch.Tensor, t=18, p=17):
    x, y = x.view(torch.int64), y.view(torch.int64)
    d = x != y
    cnt = int(d.sum())
    out = {"n_diff": cnt, "rate": cnt / x.numel()}
    if cnt:
        xi = x[d]
        yi = y[d]
        tm, pm = (1 << t) - 1, (1 << p) - 1
        dt = ((xi & tm) - (yi & tm)).abs()
        dt = torch.minimum(dt, tm + 1 - dt)  # theta wraps at +-pi
        dp = (((xi >> t) & pm) - ((yi >> t) & pm)).abs()
        df = ((xi >> (t + p)) - (yi >> (t + p))).abs()
        out.update(max_dn_theta=int(dt.max()), max_dn_phi=int(dp.max()), max_dfield=int(df.max()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ref", default=str(ROOT / "tools" / "libvc3_r1.so"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = _native.load()
    ref = load_ref(args.ref) if Path(args.ref).exists() else None
    lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
    cl = _native.c_layout(lay)
    n = 1 << args.n
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    gen = torch.Generator(device=dev).manual_seed(1234)
    va = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    vb = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    a = vc3b.compress(va, lay, pol)
    b = vc3b.compress(vb, lay, pol)
    if ref is not None:  # the compress itself must agree with the reference build
        a2 = torch.empty_like(a)
        ref.vc3_compress(va.data_ptr(), a2.data_ptr(), n, cl, pol.mask, None, sp)
        torch.cuda.synchronize()
        compress_same = bool(torch.equal(a, a2))
        del a2
    del va, vb
    res = {"n": n}
    if ref is not None:
        res["compress_equal_ref"] = compress_same
    c_ex, c_ct = torch.empty_like(a), torch.empty_like(a)
    f_ex = lambda: lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), c_ex.data_ptr(), n, cl,
                                             pol.mask, 0, sp)
    f_ct = lambda: lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), c_ct.data_ptr(), n, cl,
                                             pol.mask, 1, sp)
    t_ex, t_ct = timeit(f_ex, args.steps, stream), timeit(f_ct, args.steps, stream)
    res["add"] = {"exact_gvec_s": n / t_ex / 1e6, "contract_gvec_s": n / t_ct / 1e6}
    if ref is not None:
        c_r = torch.empty_like(a)
        f_r = lambda: ref.vc3_add_compressed(a.data_ptr(), b.data_ptr(), c_r.data_ptr(), n, cl,
                                             pol.mask, sp)
        res["add"]["ref_exact_gvec_s"] = n / timeit(f_r, args.steps, stream) / 1e6
        res["add"]["exact_equal_ref"] = bool(torch.equal(c_ex, c_r))
        res["add"]["exact_vs_ref"] = word_deltas(c_ex, c_r)
        del c_r
    res["add"]["contract_vs_exact"] = word_deltas(c_ct, c_ex)
    # standalone compress (the all-single fast path vs the reference build)
    vx = torch.rand((n, 3), device=dev, generator=gen).mul_(2).sub_(1)
    cw = torch.empty_like(a)
    f_c = lambda: lib.vc3_compress(vx.data_ptr(), cw.data_ptr(), n, cl, pol.mask, None, sp)
    res["compress"] = {"gvec_s": n / timeit(f_c, args.steps, stream) / 1e6}
    if ref is not None:
        cw2 = torch.empty_like(a)
        f_c2 = lambda: ref.vc3_compress(vx.data_ptr(), cw2.data_ptr(), n, cl, pol.mask, None, sp)
        res["compress"]["ref_gvec_s"] = n / timeit(f_c2, args.steps, stream) / 1e6
        res["compress"]["equal_ref"] = bool(torch.equal(cw, cw2))
        del cw2
    del vx, cw
    # axpy y' = 0.75 x + y (out of place) and the RK stage (in place, on copies)
    for mode in (0, 1):
        o = torch.empty_like(a)
        f = lambda: lib.vc3_axpy_ex(0.75, a.data_ptr(), b.data_ptr(), o.data_ptr(), n, cl, pol.mask, mode, sp)
        res.setdefault("axpy", {})[("exact" if mode == 0 else "contract") + "_gvec_s"] = n / timeit(f, args.steps, stream) / 1e6
        if mode == 0:
            o_ex = o
    if ref is not None:
        o2 = torch.empty_like(a)
        ref.vc3_axpy(0.75, a.data_ptr(), b.data_ptr(), o2.data_ptr(), n, cl, pol.mask, sp)
        torch.cuda.synchronize()
        res["axpy"]["exact_equal_ref"] = bool(torch.equal(o_ex, o2))
        del o2
    del o, o_ex
    q0, d0 = a.clone(), b.clone()
    for mode in (0, 1):
        q, d = q0.clone(), d0.clone()
        f = lambda: lib.vc3_rk_stage_ex(0.5, 0.25, 1e-3, q.data_ptr(), d.data_ptr(), c_ex.data_ptr(), n, cl,
                                        pol.mask, mode, sp)
        res.setdefault("rk", {})[("exact" if mode == 0 else "contract") + "_gvec_s"] = n / timeit(f, args.steps, stream) / 1e6
        if mode == 0:
            q, d = q0.clone(), d0.clone()
            f()
            torch.cuda.synchronize()
            q_ex, d_ex = q, d
    if ref is not None:
        q, d = q0.clone(), d0.clone()
        ref.vc3_rk_stage(0.5, 0.25, 1e-3, q.data_ptr(), d.data_ptr(), c_ex.data_ptr(), n, cl, pol.mask, sp)
        torch.cuda.synchronize()
        res["rk"]["exact_equal_ref"] = bool(torch.equal(q, q_ex) and torch.equal(d, d_ex))
    del q, d, q0, d0
    # decompress both modes
    out = torch.empty((n, 3), dtype=torch.float32, device=dev)
    out2 = torch.empty_like(out)
    d_ex = lambda: lib.vc3_decompress_ex(a.data_ptr(), out.data_ptr(), n, cl, 0, sp)
    d_ct = lambda: lib.vc3_decompress_ex(a.data_ptr(), out2.data_ptr(), n, cl, 1, sp)
    res["decompress"] = {"exact_gword_s": n / timeit(d_ex, args.steps, stream) / 1e6,
                         "contract_gword_s": n / timeit(d_ct, args.steps, stream) / 1e6}
    ulp = (out.view(torch.int32).to(torch.int64) - out2.view(torch.int32).to(torch.int64)).abs()
    res["decompress"]["contract_max_ulp"] = int(ulp.max())
    res["decompress"]["contract_frac_diff"] = float((ulp != 0).float().mean())
    if ref is not None:
        ref.vc3_decompress(a.data_ptr(), out2.data_ptr(), n, cl, sp)
        torch.cuda.synchronize()
        res["decompress"]["exact_equal_ref"] = bool(torch.equal(out, out2))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
