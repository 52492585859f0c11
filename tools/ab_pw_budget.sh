for b in 2048 6144 512; do
  for r in 1; do SDMK_PW_BUDGET_MB=$b python tools/prof_step.py --n 10000000 --reps 3 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$b', d['t_total'], d['t_downward'], d['t_planewave'], d['t_residual_kernel'])"; done
done
