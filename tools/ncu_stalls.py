"""Stall reasons (warps per issued instruction) and pipe utilisation of one ncu report."""
import csv
import subprocess
import sys

KEYS = ["smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    for k in KEYS:
        print(f"  {k:70s} {d.get(k)}")
    st = []
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for k, v in d.items():
        if k.startswith(pre) and k.endswith(suf):
            try:
                st.append((float(v), k[len(pre):-len(suf)]))
            except ValueError:
                pass
    print("  stalls (warps/issue): " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    for r in sys.argv[1:]:
        print(r)
        main(r)
