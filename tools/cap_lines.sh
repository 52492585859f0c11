#!/bin/bash
# ncu --set full captures with source-line stall attribution of chosen kernels
# at the metric (N = 1e7 Stokeslet).  usage: tools/cap_lines.sh <outdir> <kernel:skip> ...
set -u
out=$1; shift
mkdir -p $out
one="python tools/prof_step.py --n 10000000 --reps 1"
$one > $out/plain.log 2>&1 || { echo plain failed; exit 1; }
for spec in "$@"; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip -c 1 -o $out/$k $one > /dev/null 2>&1
  python tools/ncu_lines.py $out/$k.ncu-rep 45 > $out/$k.lines.txt 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/$k.raw.csv 2>/dev/null
  python tools/ncu_summary.py $out/$k.raw.csv > $out/$k.summary.txt 2>&1
done
rm -f $out/*.ncu-rep $out/*.raw.csv
