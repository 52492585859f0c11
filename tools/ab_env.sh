#!/bin/bash
# A/B of one environment switch at the metric (and the stresslet): per-pass
# times of a warm evaluation.  usage: tools/ab_env.sh VAR value...
var=$1; shift
for v in "$@"; do
  for k in 0 1; do
    env $var=$v python tools/prof_step.py --n 10000000 --kernel $k --reps 4 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$var=$v', $k, 'step', round(d['t_total']-d['t_h2d']-d['t_d2h'],5), 'tree', d['t_tree'], 'up', d['t_upward'], 'root', d['t_root'], 'down', d['t_downward'], 'res', d['t_residual'])"
  done
done
