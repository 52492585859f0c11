"""Per-CUDA-source-line stall samples and instruction counts from an ncu report.

usage: python tools/ncu_lines.py report.ncu-rep [top_n]
Runs `ncu -i report --page source --csv --print-source cuda,sass` and folds
the SASS rows onto the CUDA line that precedes them.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hdr]
    iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    samp, inst = collections.Counter(), collections.Counter()
    for r in rows[hdr + 1:]:
        if not r or not r[0] or len(r) <= iex:  # SASS rows carry an empty line number
            continue
        key = (r[0] + ": " + r[1].strip())[:120]
        try:
            samp[key] += int(r[iss] or 0)
            inst[key] += int(r[iex] or 0)
        except ValueError:
            pass
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"{'stall%':>7} {'inst%':>6}  line")
    for k, v in samp.most_common(top):
        print(f"{100 * v / ts:7.2f} {100 * inst[k] / ti:6.2f}  {k}")


if __name__ == "__main__":
    main()
