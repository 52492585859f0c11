#!/bin/bash
# Evidence for profiles/<round>: the bench command's launch list and one
# ncu --set full capture per dominant kernel (largest launch of each), run on
# the GPU box after the same command has exited 0 without ncu.
# usage: tools/profile_round.sh <outdir>
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
cmd="python tools/prof_step.py --n 10000000 --reps 2"
$cmd > "$out/plain.log" 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" $cmd > /dev/null 2>&1
python tools/launch_summary.py "$out/launches.csv" > "$out/launches.txt"
# kernel regex : launches to skip (the big level-5 launch where a kernel runs per level)
for spec in k_residual:0 k_interp_mma:0 k_anterp2:0 k_tensor_up:4 k_tensor_down:3 k_inv_xy2:8 k_acc_group:8 k_fwd_xy2:8 k_zi2:8 k_zf2:8; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip -c 1 \
      -o "$out/$k" python tools/prof_step.py --n 10000000 --reps 1 > /dev/null 2>&1
done
