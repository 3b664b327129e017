"""Run one fused operation a few times (ncu / sanitizer driver).

    python tools/run_op.py [--op add|decompress|compress|axpy|rk] [--mode exact|contract]
                           [--n LOG2] [--steps K]
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2003_02633_b200 as vc3b  # noqa: E402
from paper_2003_02633_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="add")
ap.add_argument("--mode", default="contract")
ap.add_argument("--n", type=int, default=26)
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
lib = _native.load()
lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
cl = _native.c_layout(lay)
n = 1 << args.n
flags = 1 if args.mode == "contract" else 0
s = torch.cuda.current_stream(dev).cuda_stream
g = torch.Generator(device=dev).manual_seed(7)
va = torch.rand((n, 3), device=dev, generator=g).mul_(2).sub_(1)
vb = torch.rand((n, 3), device=dev, generator=g).mul_(2).sub_(1)
a = vc3b.compress(va, lay, pol)
b = vc3b.compress(vb, lay, pol)
c = torch.empty_like(a)
for _ in range(args.steps):
    if args.op == "add":
        rc = lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, cl, pol.mask, flags, s)
    elif args.op == "decompress":
        rc = lib.vc3_decompress_ex(a.data_ptr(), va.data_ptr(), n, cl, flags, s)
    elif args.op == "compress":
        rc = lib.vc3_compress(va.data_ptr(), c.data_ptr(), n, cl, pol.mask, None, s)
    elif args.op == "axpy":
        rc = lib.vc3_axpy_ex(0.75, a.data_ptr(), b.data_ptr(), c.data_ptr(), n, cl, pol.mask, flags, s)
    elif args.op == "rk":
        rc = lib.vc3_rk_stage_ex(0.5, 0.25, 1e-3, a.data_ptr(), b.data_ptr(), c.data_ptr(), n, cl,
                                 pol.mask, flags, s)
    _native.check(rc, args.op)
torch.cuda.synchronize()
print("ok", args.op, args.mode, n)
