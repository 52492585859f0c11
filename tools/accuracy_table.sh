mkdir -p gpurun_out/acc
for d in 3 2; do for k in stokeslet stresslet rotlet; do for e in 1e-3 1e-6 1e-9 1e-12; do
  python tools/experiments.py accuracy --kernel $k --dim $d --eps $e --n 100000 --out gpurun_out/acc/${k}_${d}d_${e}.csv 2>> gpurun_out/acc/summary.txt || echo "rc=$? $k $d $e" >> gpurun_out/acc/summary.txt
done; done; done
python tools/experiments.py scaling --kernel stokeslet --dim 3 --eps 1e-6 --n-list 1e5,1e6,4e6,1e7,1.6e7 --repetitions 2 --out gpurun_out/acc/scaling_stokeslet_3d.csv 2>> gpurun_out/acc/summary.txt
cat gpurun_out/acc/summary.txt
