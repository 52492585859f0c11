"""Summarize `nvcc -Xptxas -v` logs: kernel -> registers, spills, smem."""
import glob
import re
import subprocess
import sys

logs = sys.argv[1:] or glob.glob("paper_2509_21471_b200/csrc/build/kernels/*.ptxas.log")
for path in sorted(logs):
    cur = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            try:
                name = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            except Exception:  # noqa: BLE001
                pass
            name = re.sub(r"sdmkb::\(anonymous namespace\)::", "", name)
            name = re.sub(r"\(.*", "", name)
            cur = {"name": name}
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            cur["spill"] = f"{m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if m:
            cur["regs"] = int(m.group(1))
            sm = re.search(r"(\d+) bytes smem", line)
            if "cub::" not in cur["name"]:
                print(f"{cur['regs']:4d} regs  spill {cur.get('spill', '0/0'):>9}  "
                      f"smem {sm.group(1) if sm else 0:>6}  {cur['name'][:90]}")
            cur = None
