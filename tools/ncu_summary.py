"""Summarize an ncu --set full report: per kernel time, pipes, occupancy, DRAM, stalls.

usage: ncu -i rep.ncu-rep --page raw --csv > raw.csv ; python tools/ncu_summary.py raw.csv
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thr"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd_thr"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul_thr"),
]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units, data = rows[0], rows[1], rows[2:]
    stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("per_issue_active.ratio")]
    for r in data:
        print("----", r[h.index("Kernel Name")][:80])
        parts = []
        for k, lab in KEYS:
            if k in h and r[h.index(k)] not in ("", "n/a"):
                parts.append(f"{lab}={r[h.index(k)]}{units[h.index(k)] if lab in ('time', 'dram_rd', 'dram_wr') else ''}")
        print("   " + "  ".join(parts))
        st = []
        for c in stall:
            v = r[h.index(c)]
            try:
                st.append((float(v), c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
        st.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
