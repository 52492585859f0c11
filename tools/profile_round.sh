#!/bin/bash
# Evidence for profiles/<round>: launch lists of one warm evaluation (the
# metric, N = 1e7 3D Stokeslet; and BASELINE cfg4, 2D) and one ncu --set full
# capture per kernel on those paths (the largest / level-5 launch), run on the
# GPU box after the same commands have exited 0 without ncu.
# usage: tools/profile_round.sh <outdir>
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
m="python tools/prof_step.py --n 10000000 --reps 2"
c4="python tools/prof_step.py --cfg cfg4 --reps 2"
$m > "$out/plain_metric.log" 2>&1 || exit 1
$c4 > "$out/plain_cfg4.log" 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_metric.csv" $m > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_cfg4.csv" $c4 > /dev/null 2>&1
python tools/launch_summary.py "$out/launches_metric.csv" > "$out/launches_metric.txt"
python tools/launch_summary.py "$out/launches_cfg4.csv" > "$out/launches_cfg4.txt"
one="python tools/prof_step.py --n 10000000 --reps 1"
# kernel regex : launches to skip (the big level-5 launch where a kernel runs per level)
for spec in k_residual:0 k_interp_mma:0 k_anterp2:0 k_basis:0 k_tensor_up:0 k_tensor_down:4 k_inv_xy3:8 k_acc_group:8 \
            k_fwd_xy3:5 k_zi3:8 k_zf3:5 k_morton:0 k_gather_points:0 k_pack_sources:0 k_combine:0; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip -c 1 \
      -o "$out/metric_$k" $one > /dev/null 2>&1
done
one4="python tools/prof_step.py --cfg cfg4 --reps 1"
for k in k_residual k_inv_xy k_tensor k_fwd_xy k_interp_mma k_anterp_mma k_basis k_acc_group k_inv_z k_fwd_z; do
  ncu --set full --clock-control none --import-source on -k regex:"$k\\b" -c 1 -o "$out/cfg4_$k" $one4 > /dev/null 2>&1
done

# the residual kernel's executed FP64 work (bench.py's roofline reads it)
ncu -i "$out/metric_k_residual.ncu-rep" --page source --csv --print-source sass > "$out/metric_k_residual.sass.csv" 2>/dev/null
ncu -i "$out/metric_k_residual.ncu-rep" --page raw --csv > "$out/metric_k_residual.raw.csv" 2>/dev/null
python tools/residual_hw.py "$out/metric_k_residual.sass.csv" "$out/metric_k_residual.raw.csv" > "$out/residual_hw.json"
python tools/ncu_lines.py "$out/metric_k_residual.ncu-rep" 60 > "$out/metric_k_residual.lines.txt" 2>&1
rm -f "$out/metric_k_residual.sass.csv"
# text summaries on the box (the reports themselves exceed what gpurun copies back)
for r in "$out"/*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  python tools/ncu_summary.py "${r%.ncu-rep}.raw.csv" > "${r%.ncu-rep}.summary.txt" 2>&1
done
cat "$out"/metric_*.summary.txt > "$out/ncu_kernels_metric.txt"
cat "$out"/cfg4_*.summary.txt > "$out/ncu_kernels_cfg4.txt"
mkdir -p "$out/keep" && cp "$out/metric_k_residual.ncu-rep" "$out/metric_k_inv_xy3.ncu-rep" "$out/keep/" 2>/dev/null
rm -f "$out"/*.ncu-rep "$out"/*.raw.csv "$out"/launches_*.csv
du -sh "$out"
