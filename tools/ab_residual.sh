# A/B timing of residual-kernel variants built as paper_2509_21471_b200/libsdmk_<name>.so
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=paper_2509_21471_b200/libsdmk_$v.so; fi
  for k in 0 1; do
    SDMK_LIB=$L python tools/prof_step.py --n 10000000 --kernel $k --reps 3 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$v', $k, d['t_residual_kernel'], d['t_total'])"
  done
done
