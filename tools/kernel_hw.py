"""Per-kernel ncu numbers for bench.py's rooflines, from a tools/profile_round.sh output directory.

usage: python tools/kernel_hw.py <profile dir> > profiles/round2/kernel_hw.json
Reads metric_<kernel>.summary.txt (tools/ncu_summary.py lines: time, tensor%,
fp64%, dram_rd, dram_wr of one launch) for the three largest kernels of the
metric workload, and residual_hw.json (executed FP64 work of k_residual).
"""
import json
import os
import re
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6,
         "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}


def num(s):
    m = re.match(r"([0-9.eE+-]+)([A-Za-z]*)", s)
    return float(m.group(1)) * UNITS.get(m.group(2), 1.0)


def main():
    d = sys.argv[1]
    out = {}
    for k in ("k_residual", "k_interp_mma", "k_anterp2"):
        p = os.path.join(d, f"metric_{k}.summary.txt")
        if not os.path.exists(p):
            continue
        txt = open(p).read()
        f = dict(re.findall(r"(\w+%?)=(\S+)", txt))
        out[k] = {"time_s": num(f["time"]), "tensor_pct": float(f["tensor%"]), "fp64_pct": float(f["fp64%"]),
                  "dram_bytes_per_launch": num(f["dram_rd"]) + num(f["dram_wr"]),
                  "source": f"ncu --set full, one launch at the metric (tools/profile_round.sh -> {p})"}
    hw = os.path.join(d, "residual_hw.json")
    if os.path.exists(hw) and "k_residual" in out:
        r = json.load(open(hw))
        out["k_residual"]["hw_fp64_tflops"] = r["hw_fp64_tflops"]
        out["k_residual"]["hw_fp64_flop"] = r["hw_fp64_flop"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
