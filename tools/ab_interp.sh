#!/bin/bash
# A/B of K11 builds on one GPU: parity tests, then the kernel's CUDA-event time
# at the metric.  usage: tools/ab_interp.sh <outdir> <variant>...  (base = in-tree library)
out=$1; shift
mkdir -p "$out"
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=paper_2509_21471_b200/libsdmk_$v.so; fi
  SDMK_LIB=$L python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_cases.py -q -x > "$out/t_$v.log" 2>&1
  echo "$v tests: $(tail -1 "$out/t_$v.log")"
  for k in 0 1; do
    SDMK_LIB=$L python tools/prof_step.py --n 10000000 --kernel $k --reps 3 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$v', $k, 'total', d['t_total'], 'interp', d['t_interp_kernel'], 'tree', d['t_tree'], 'down', d['t_downward'])"
  done
done
