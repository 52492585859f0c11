#!/bin/bash
# Final evidence of the round on one B200: bench line, launch lists and ncu
# captures (tools/profile_round.sh), kernel_hw.json, full-size parity at every
# BASELINE configuration.  usage: tools/final_evidence.sh <outdir>
set -u
out=${1:-gpurun_out/final}
mkdir -p "$out"
python bench.py > "$out/bench.json" 2> "$out/bench.log" || { echo bench failed; tail -20 "$out/bench.log"; exit 1; }
bash tools/profile_round.sh "$out/prof" > "$out/prof.log" 2>&1
python tools/kernel_hw.py "$out/prof" > "$out/kernel_hw.json"
python tools/parity_configs.py --out "$out/parity_full_size.jsonl" > "$out/parity.log" 2>&1
