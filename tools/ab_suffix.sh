for v in 0 1; do
  if [ $v = 1 ]; then export SDMK_TENSOR_NOSUFFIX=1; fi
  for k in 0 1; do
    python tools/prof_step.py --n 10000000 --kernel $k --reps 3 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('nosuffix=$v', $k, 'total', d['t_total'], 'up', d['t_upward'])"
  done
done
