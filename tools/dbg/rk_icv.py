"""Time the RK stage on the ICV field (bench C4 setup) in both modes, and check
exact-mode words against the oracle composition on a sample."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, torch
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import fields, _native
lib = _native.load()
dev = torch.device("cuda", 0)
lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
cl = _native.c_layout(lay)
n_elem = (1 << 28) // 125
mom, vel = fields.icv_fields(n_elem, 30.0, device=dev)
npts = mom.shape[0]
q = vc3b.compress(mom, lay, pol); dq = vc3b.compress(vel * 1e-3, lay, pol); R = vc3b.compress(vel, lay, pol)
s = torch.cuda.current_stream().cuda_stream
def step(flags):
    lib.vc3_rk_stage_ex(-0.4178, 0.6, 1e-3, q.data_ptr(), dq.data_ptr(), R.data_ptr(), npts, cl, pol.mask, flags, s)
for flags in (0, 1):
    step(flags); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): step(flags)
    e1.record(); e1.synchronize()
    print(["exact", "contract"][flags], npts / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9, "Gvec/s")
# parity sample (exact)
import vc3_oracle as oracle
oracle.build()
m = 1 << 22
qs, dqs, Rs = (x[:m].cpu().numpy().view(np.uint64).copy() for x in (q.view(torch.int64), dq.view(torch.int64), R.view(torch.int64)))
tq, tdq, tR = (torch.from_numpy(x.view(np.int64)).to(dev).view(torch.uint64) for x in (qs, dqs, Rs))
vc3b.rk_stage(np.float32(-0.4178), np.float32(0.6), np.float32(1e-3), tq, tdq, tR, lay, pol)
a_, b_, dt = np.float32(-0.4178), np.float32(0.6), np.float32(1e-3)
vq, vd, vr = (oracle.decompress(x, lay) for x in (qs, dqs, Rs))
d_new = (a_ * vd + dt * vr).astype(np.float32)
q_new = (vq + b_ * d_new).astype(np.float32)
mis = int((tdq.cpu().numpy().view(np.uint64) != oracle.compress(d_new, lay, pol)).sum()) + \
      int((tq.cpu().numpy().view(np.uint64) != oracle.compress(q_new, lay, pol)).sum())
print("exact parity mismatches on", m, "ICV points:", mis)
