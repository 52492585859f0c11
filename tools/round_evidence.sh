#!/bin/bash
# Round evidence on one B200: bench line, launch list, ncu --set full of the
# residual kernel, one-GPU scaling projections.  Usage: tools/round_evidence.sh <outdir>
set -u
out=${1:-gpurun_out/ev}
mkdir -p "$out"
python bench.py > "$out/bench.json" 2> "$out/bench.log" || { echo bench failed; tail -20 "$out/bench.log"; exit 1; }
python bench.py --impl reference --steps 2 --warmup 1 > "$out/bench_ref.json" 2> "$out/bench_ref.log"
cmd="python tools/prof_step.py --n 10000000 --reps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" $cmd > /dev/null 2>&1
python tools/launch_summary.py "$out/launches.csv" > "$out/launches.txt" 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual -c 1 -o "$out/k_residual" \
    python tools/prof_step.py --n 10000000 --reps 1 > /dev/null 2>&1
python tools/shard_projection.py --n 1e7 > "$out/proj_1e7.json" 2>&1
python tools/shard_projection.py --n 1.6e7 --dist cfg5 > "$out/proj_cfg5.json" 2>&1
