"""Per-source-line executed instruction counts from an ncu source export
(ncu -i X.ncu-rep --page source --csv --print-source cuda,sass)."""
import collections
import csv
import sys


def toi(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, n_items, top=60):
    rows = list(csv.reader(open(path)))
    file = None
    lines, sass = [], []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0] and len(r) > 7 and r[2] == "-":
            lines.append((file, r[0], r[1], toi(r[7])))
        elif r[0] == "" and len(r) > 7:
            sass.append((r[3].strip(), toi(r[7])))
    tot = sum(x[3] for x in lines)
    print(f"thread-instructions per item: {tot * 32 / n_items:.1f}")
    for f, ln, src, c in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"{c * 32 / n_items:6.1f}  {f}:{ln}  {src[:95]}")
    ops = collections.Counter()
    for s, c in sass:
        parts = s.split()
        if not parts:
            continue
        o = parts[1] if parts[0].startswith("@") else parts[0]
        ops[o.split(".")[0]] += c
    print([(o, round(c * 32 / n_items, 1)) for o, c in ops.most_common(40)])


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 60)
