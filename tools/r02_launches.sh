# full GPU suite + serialised launch lists at n = 400, 1600, 10k (one evaluation each after warm-up)
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests_full.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02_gpu_tests_full.log
for n in 400 1600 10000; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launch_n$n.csv \
      python tools/n10k_once.py $n > gpurun_out/r02_launch_n$n.log 2>&1
done
