# A/B: per-pass times from one warm N=1e7 evaluation for each build
# (base = in-tree library, others = paper_2509_21471_b200/libsdmk_<name>.so)
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=paper_2509_21471_b200/libsdmk_$v.so; fi
  for k in 0 1; do
    SDMK_LIB=$L python tools/prof_step.py --n 10000000 --kernel $k --reps 3 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$v', $k, 'total', d['t_total'], 'up', d['t_upward'], 'down', d['t_downward'], 'pw', d['t_planewave'], 'res', d['t_residual_kernel'])"
  done
done
