"""Summarise `ncu --set full` reports of the fused kernels as a markdown table.

    python tools/ncu_summary.py NAME=path.ncu-rep [NAME=path.ncu-rep ...] [--n LOG2] [--bytes B ...]

For each report: duration, DRAM read + write, warp instructions (and per
unit, 2^n units per launch), issue-active, FP64 / XU pipe use, warps active,
shared-memory wavefronts (and the bank-conflict share) and the top stall
reasons from the PC sampling.  Also writes <path>.raw.csv next to each
report (the `--page raw --csv` export).
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def raw(path: str) -> tuple[list[str], list[str], list[str]]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    open(path.replace(".ncu-rep", ".raw.csv"), "w").write(out)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def num(v: str, unit: str = "") -> float:
    """Value in bytes (byte units) or microseconds (time units)."""
    if v in ("", "n/a"):
        return float("nan")
    return float(v.replace(",", "")) * SCALE.get(unit, 1.0)


def main() -> None:
    args = [a for a in sys.argv[1:] if "=" in a]
    n = 26
    if "--n" in sys.argv:
        n = int(sys.argv[sys.argv.index("--n") + 1])
    units = 2 ** n
    cols = []
    for a in args:
        name, path = a.split("=", 1)
        h, u, v = raw(path)
        g = lambda k: num(v[h.index(k)], u[h.index(k)]) if k in h else float("nan")  # noqa: E731
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v[i]) for i, k in enumerate(h)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
              and v[i] not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        top = ", ".join(f"{k} {100 * x / tot:.1f}" for k, x in sorted(st.items(), key=lambda t: -t[1])[:5])
        wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        bc = g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
        cols.append((name, {
            "kernel": v[h.index("Kernel Name")].split("(")[0][:60],
            "duration": f"{g('gpu__time_duration.sum'):.1f} us",
            "DRAM read + write": f"{g('dram__bytes_read.sum') / 1e6:.1f} + {g('dram__bytes_write.sum') / 1e6:.1f} MB",
            "instructions (warp)": f"{g('smsp__inst_executed.sum') / 1e6:.1f} M = "
                                   f"{32 * g('smsp__inst_executed.sum') / units:.1f} / unit",
            "issue active": f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} %",
            "FP64 pipe": f"{g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} %",
            "XU pipe": f"{g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} %",
            "warps active": f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} %",
            "registers / CTAs per SM": f"{g('launch__registers_per_thread'):.0f} / "
                                       f"{min(g('launch__occupancy_limit_registers'), g('launch__occupancy_limit_shared_mem')):.0f}",
            "shared wavefronts (conflicts)": f"{wf / 1e6:.1f} M ({100 * bc / wf:.0f} %)" if wf == wf and wf else "-",
            "top stalls (% of samples)": top,
        }))
    keys = list(cols[0][1])
    print("| metric | " + " | ".join(c[0] for c in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for k in keys:
        print(f"| {k} | " + " | ".join(c[1][k] for c in cols) + " |")


if __name__ == "__main__":
    main()
