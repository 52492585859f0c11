# A/B of one kernel's ncu launch time (cold, serialized) across builds:
# tools/ab_kernel.sh <kernel regex> <variant>...
k=$1; shift
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=paper_2509_21471_b200/libsdmk_$v.so; fi
  SDMK_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$k --csv --log-file gpurun_out/ab_$v.csv python tools/prof_step.py --n 10000000 --reps 1 > /dev/null 2>&1
  echo "$v $(python tools/launch_summary.py gpurun_out/ab_$v.csv | tail -1)"
done
