"""Headline metrics of one kernel from an ncu report (raw page CSV)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(rep):
    if rep.endswith(".csv"):  # a saved raw page
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    print(v[h.index("Kernel Name")][:100])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {v[i]} {u[i]}")
    stalls = [(float(v[i]), n) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")
              and v[i] not in ("", "n/a")]
    for val, n in sorted(stalls, reverse=True)[:8]:
        print(f"  stall {n[34:-30]:40s} {val:.2f}")


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
