#!/bin/bash
# One GPU call after a kernel change: the parity / guard / reference-case GPU
# tests, then the bench line.  usage: tools/quick_check.sh <outdir> [pytest files...]
out=${1:-gpurun_out/q}; shift
mkdir -p "$out"
files=${@:-tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_reference_cases.py}
python -m pytest $files -q -x > "$out/t.log" 2>&1; echo rc=$? >> "$out/t.log"
python bench.py > "$out/bench.json" 2> "$out/bench.log"
tail -2 "$out/t.log"
python - "$out/bench.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
k = d["roofline"]["kernels"]
print("step_ms", round(d["ms_per_step"], 2), "value", d["value"], "e2e", d["e2e"]["value"],
      {n: round(v["ms"], 2) for n, v in k.items()}, "pw", d["kernels"]["stokeslet"]["pass_s"]["t_planewave"])
PY
