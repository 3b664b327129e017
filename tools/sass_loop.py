"""Per-stage SASS instruction budget of a kernel's hot loop.

    python tools/sass_loop.py <cubin|so|o> <function-substring> [--per N]

Finds the function, takes its largest backward-branch loop and prints the
instruction histogram of that loop body grouped by issue pipe, divided by
--per (vectors per iteration).  Instructions inside forward-branched regions
guarded by a predicate (the rare slow paths: `@P BRA` over a block) are
listed separately as "cold"; the rest is the straight-line hot path.
"""
from __future__ import annotations

import re
import subprocess
import sys
from collections import Counter

PIPES = {
    "fp64": {"DFMA", "DMUL", "DADD", "DSETP", "DMNMX"},
    "xu": {"MUFU", "F2F", "I2F", "F2I", "FRND", "I2FP", "F2IP"},
    "fp32": {"FFMA", "FMUL", "FADD", "FFMA2", "FMUL2", "FADD2", "FSETP", "FSEL", "FMNMX", "FCHK",
             "FSWZADD"},
    "int": {"IMAD", "IADD3", "VIADD", "LOP3", "SHF", "ISETP", "SEL", "LEA", "VIMNMX", "IMNMX",
            "PRMT", "IABS", "MOV", "PLOP3", "FLO", "POPC", "BMSK", "SGXT", "IADD", "P2R", "R2P",
            "CS2R", "S2R", "S2UR"},
    "mem": {"LDS", "STS", "LDG", "STG", "LDC", "LDL", "STL", "LD", "ST", "ATOMG", "RED", "REDG",
            "ATOMS"},
    "ctrl": {"BRA", "BSSY", "BSYNC", "CALL", "RET", "EXIT", "NOP", "WARPSYNC", "BAR"},
}


def pipe_of(op: str) -> str:
    if op.startswith("U"):
        return "uniform"
    for k, v in PIPES.items():
        if op in v:
            return k
    return "other"


def sass_of(path: str) -> str:
    return subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout


def parse(fn_text: str):
    ins = []
    for line in fn_text.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        body = m.group(2).strip()
        toks = body.split()
        pred = None
        if toks[0].startswith("@"):
            pred = toks[0]
            toks = toks[1:]
        op = toks[0]
        target = None
        if op.startswith("BRA"):
            tm = re.search(r"0x([0-9a-f]+)", body.split(" ", 1)[1] if " " in body else "")
            if tm:
                target = int(tm.group(1), 16)
        ins.append((addr, pred, op, target, body))
    return ins


def main():
    path, sub = sys.argv[1], sys.argv[2]
    per = 1
    if "--per" in sys.argv:
        per = int(sys.argv[sys.argv.index("--per") + 1])
    txt = sass_of(path)
    funcs = re.split(r"\n\s+Function : ", txt)
    for f in funcs[1:]:
        name = f.split("\n")[0].strip()
        if sub not in name:
            continue
        ins = parse(f)
        # largest backward branch = main loop
        loops = [(a, t) for a, p, o, t, b in ins if o.startswith("BRA") and t is not None and t < a]
        if not loops:
            print(name, "no loop")
            continue
        end, start = max(loops, key=lambda x: x[0] - x[1])
        body = [x for x in ins if start <= x[0] <= end]
        # cold regions: predicated forward branches skipping over code inside the loop
        cold = set()
        for a, p, o, t, b in body:
            if o.startswith("BRA") and p is not None and t is not None and a < t <= end:
                span = [x[0] for x in body if a < x[0] < t]
                if len(span) > 6:  # a real block, not a short select-by-branch
                    cold.update(span)
        hot = [x for x in body if x[0] not in cold]
        print(f"{name[:140]}")
        print(f"  loop 0x{start:x}-0x{end:x}: {len(body)} instructions, hot {len(hot)}, "
              f"cold {len(body) - len(hot)}; per item (/{per}): hot {len(hot) / per:.1f}")
        for label, sel in (("hot", hot),):
            pc = Counter(pipe_of(x[2].split(".")[0]) for x in sel)
            oc = Counter(x[2].split(".")[0] for x in sel)
            print(f"  {label} by pipe (/item): " +
                  ", ".join(f"{k} {v / per:.1f}" for k, v in pc.most_common()))
            print(f"  {label} by opcode (/item): " +
                  ", ".join(f"{k} {v / per:.1f}" for k, v in oc.most_common()))


if __name__ == "__main__":
    main()
