"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list.

usage: python tools/launch_summary.py launches.csv [--last-fraction 0.5]
Aggregates per kernel over the trailing fraction of launches (the warm rep).
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    frac = float(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--last-fraction" else 0.5
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = rows[hdr + 1:]
    data = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"sdmkb::<unnamed>::|void ", "", name)[:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'ms':>9} {'share':>6} {'n':>4}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / 1e6:9.3f} {100 * v[1] / tot:5.1f}% {v[0]:4d}  {k}")
    print(f"{tot / 1e6:9.3f} total ms over {len(data)} launches")


if __name__ == "__main__":
    main()
