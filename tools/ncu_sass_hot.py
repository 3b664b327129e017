"""Summarise an ncu SASS source page (csv): instructions executed and stall
samples per opcode, the top stalled instructions, and executed-per-item.

    ncu -i rep --page source --csv --print-source sass > page.csv
    python tools/ncu_sass_hot.py page.csv [--items N]
"""
import csv
import sys
from collections import Counter, defaultdict

path = sys.argv[1]
items = float(sys.argv[sys.argv.index("--items") + 1]) if "--items" in sys.argv else None
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
body = rows[2:]
ex = Counter()
st = Counter()
tot_ex = 0
tot_st = 0
per_ins = []
for r in body:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    e = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += e
    st[op] += s
    tot_ex += e
    tot_st += s
    per_ins.append((s, e, r[ix["Address"]][-5:], src))
print(f"warp instructions executed {tot_ex}, stall samples {tot_st}")
if items:
    print(f"thread instructions per item: {tot_ex * 32 / items:.1f}")
print("opcode: executed share / stall share")
for op, e in ex.most_common(30):
    print(f"  {op:10s} {e / tot_ex:6.1%}  {st[op] / max(tot_st, 1):6.1%}"
          + (f"  ({e * 32 / items:.1f}/item)" if items else ""))
print("top stalled instructions:")
for s, e, a, src in sorted(per_ins, reverse=True)[:25]:
    print(f"  {s:6d} {e:10d} {a} {src[:80]}")
