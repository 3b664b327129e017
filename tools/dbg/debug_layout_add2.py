"""Debug: fused add mismatches on <0,5,19>-20-20@20."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import ops
from paper_2003_02633_b200.layout import BitLayout, ALL_SINGLE_POLICY as pol
import vc3_oracle as oracle
oracle.build()
from test_gpu_fastpath import adversarial_words, encode_of, unit_scaled
lay = BitLayout(0, 5, 19, 20, 20, 20)
dev = torch.device("cuda", 0)
t = lambda w: torch.from_numpy(np.ascontiguousarray(w).view(np.int64)).to(dev).view(torch.uint64)
n = 1 << 15
v = unit_scaled(n, 32)
wo = oracle.compress(v, lay, pol)
wg = vc3b.compress(torch.from_numpy(v).to(dev), lay, pol).cpu().numpy().view(np.uint64)
print("compress mismatches", int((wo != wg).sum()))
zero = np.zeros(n, np.uint64)
for name, a in (("encoded", wo), ("adversarial", adversarial_words(lay, n, 31))):
    want = oracle.add_compressed(a, zero, lay, pol)
    got = ops.add_compressed(t(a), t(zero), lay, pol).cpu().numpy().view(np.uint64)
    bad = np.nonzero(got != want)[0]
    print(name, "add(a, 0) mismatches", bad.size)
    for i in bad[:5]:
        va = oracle.decompress(a[i:i+1], lay)
        vg = vc3b.decompress(t(a[i:i+1]), lay).cpu().numpy()
        print("  a", hex(int(a[i])), "want", hex(int(want[i])), "got", hex(int(got[i])), "dec", va, vg,
              "recompress oracle", hex(int(oracle.compress(va, lay, pol)[0])))
    gotc = ops.add_compressed(t(a), t(zero), lay, pol, mode="contract").cpu().numpy().view(np.uint64)
    print(name, "contract mismatches", int((gotc != want).sum()))
