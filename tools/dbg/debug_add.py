"""Debug: mismatching fused adds of the golden set (prints the pieces)."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests")); sys.path.insert(0, str(ROOT / "oracle"))
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import _native
import vc3_oracle
g = np.load(ROOT / "tests/golden/golden.npz")
lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
dev = torch.device("cuda", 0)
for key in [k[6:] for k in g.files if k.startswith("add_a_")]:
    if not key.endswith("SSS"): continue
    a, b, want = g[f"add_a_{key}"], g[f"add_b_{key}"], g[f"add_c_{key}"]
    if key != "17_18_SSS": continue
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    got = vc3b.add_compressed(da, db, lay, pol).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    print(key, "mismatches", bad.size)
    va = vc3_oracle.decompress(a, lay); vb = vc3_oracle.decompress(b, lay)
    s = (va + vb).astype(np.float32)
    cw = vc3b.compress(torch.from_numpy(s).to(dev), lay, pol).cpu().numpy()
    print("generic compress of oracle sums == want:", np.array_equal(cw, want))
    # fast path on the exact sums: add x + 0 (word 0 decodes to zeros)
    for i in bad[:10]:
        print(i, hex(int(a[i])), hex(int(b[i])), "got", hex(int(got[i])), "want", hex(int(want[i])),
              "sum", s[i], [hex(int(v)) for v in s[i].view(np.uint32)])
