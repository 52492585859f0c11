"""FP64 work the hardware executed in one k_residual launch, from an ncu --set full capture.

usage: python tools/residual_hw.py <source.csv> <raw.csv> > profiles/round2/residual_hw.json
  source.csv: ncu -i rep --page source --csv --print-source sass
  raw.csv:    ncu -i rep --page raw --csv
Counts predicated-on thread instructions of the SASS source page (DFMA counts
2 FLOP, DMUL and DADD 1) and divides by gpu__time_duration; DRAM bytes are
dram__bytes_read.sum + dram__bytes_write.sum of the same launch.
"""
import csv
import json
import re
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hdr]
    src, pon = h.index("Source"), h.index("Predicated-On Thread Instructions Executed")
    cnt = {"DFMA": 0, "DMUL": 0, "DADD": 0}
    for r in rows[hdr + 1:]:
        if len(r) <= pon:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", r[src])
        if m and m.group(2) in cnt:
            cnt[m.group(2)] += int(r[pon] or 0)
    raw = list(csv.reader(open(sys.argv[2])))
    rh, units, rv = raw[0], raw[1], raw[2]

    def val(key):
        v = float(rv[rh.index(key)].replace(",", ""))
        u = units[rh.index(key)]
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "s": 1.0,
                 "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        return v * scale

    t = val("gpu__time_duration.sum")
    flop = 2 * cnt["DFMA"] + cnt["DMUL"] + cnt["DADD"]
    out = {
        "kernel": rv[rh.index("Kernel Name")][:60] + " (metric, N=1e7 3D Stokeslet)",
        "time_s": t,
        "dfma_thread_inst": cnt["DFMA"],
        "dmul_thread_inst": cnt["DMUL"],
        "dadd_thread_inst": cnt["DADD"],
        "hw_fp64_flop": flop,
        "hw_fp64_tflops": flop / t / 1e12,
        "source": "ncu --set full capture of the current kernel (tools/profile_round.sh), predicated-on thread "
                  "instructions of the SASS source page: 2 DFMA + DMUL + DADD over gpu__time_duration",
        "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
