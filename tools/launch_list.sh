#!/bin/bash
# Per-kernel launch list of one warm N = 1e7 evaluation (ncu, serialized):
# usage: tools/launch_list.sh <out.txt> [prof_step args]
out=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out.csv" \
    python tools/prof_step.py --n 10000000 --reps 2 "$@" > /dev/null 2>&1
python tools/launch_summary.py "$out.csv" > "$out"
rm -f "$out.csv"
