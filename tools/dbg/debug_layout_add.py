"""Debug: one fused-add mismatch on <1,8,23>-16-16 (large magnitudes)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, torch
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import ops
from paper_2003_02633_b200.layout import LAYOUT_BASE_16_16 as lay, ALL_SINGLE_POLICY as pol
import vc3_oracle as oracle
oracle.build()
a = np.array([0x7f451af9b9bb0000], dtype=np.uint64)
b = np.array([0x7f17bb10dd35612b], dtype=np.uint64)
dev = torch.device("cuda", 0)
t = lambda w: torch.from_numpy(w.view(np.int64)).to(dev).view(torch.uint64)
va_o, vb_o = oracle.decompress(a, lay), oracle.decompress(b, lay)
va_g, vb_g = vc3b.decompress(t(a), lay).cpu().numpy(), vc3b.decompress(t(b), lay).cpu().numpy()
print("decode a oracle", va_o, "gpu", va_g, np.array_equal(va_o.view(np.int32), va_g.view(np.int32)))
print("decode b oracle", vb_o, "gpu", vb_g, np.array_equal(vb_o.view(np.int32), vb_g.view(np.int32)))
s = (va_o + vb_o).astype(np.float32)
print("sum", s)
w_o = oracle.compress(s, lay, pol)
w_g = vc3b.compress(torch.from_numpy(s).to(dev), lay, pol).cpu().numpy() if np.isfinite(s).all() else None
print("compress oracle", hex(int(w_o[0])), "gpu", None if w_g is None else hex(int(w_g[0])))
add_o = oracle.add_compressed(a, b, lay, pol)
add_g = ops.add_compressed(t(a), t(b), lay, pol).cpu().numpy().view(np.uint64)
add_c = ops.add_compressed(t(a), t(b), lay, pol, mode="contract").cpu().numpy().view(np.uint64)
print("add oracle", hex(int(add_o[0])), "gpu exact", hex(int(add_g[0])), "gpu contract", hex(int(add_c[0])))
# the same sum through the generic compress with each policy path
for n in (1, 4, 5):
    aa, bb = np.repeat(a, n), np.repeat(b, n)
    g = ops.add_compressed(t(aa), t(bb), lay, pol).cpu().numpy().view(np.uint64)
    print(n, [hex(int(x)) for x in g])
