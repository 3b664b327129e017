import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2003_02633_b200 as vc3b
g = np.load(ROOT / "tests/golden/golden.npz")
lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY
for vname in ["edge", "kat", "mixed", "spread"]:
    want = g[f"cw_17_18_SSS_{vname}"]
    v = g[f"vec_{vname}"][: want.size]
    got = vc3b.compress(v, lay, pol)
    bad = np.nonzero(got != want)[0]
    print(vname, bad.size)
    for i in bad[:10]:
        print(" ", [hex(int(x)) for x in v[i].view(np.uint32)], v[i], hex(int(got[i])), hex(int(want[i])))
