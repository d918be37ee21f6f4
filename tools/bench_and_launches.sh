set -x
python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/plain_bench_c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_bench_c.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_c.log 2>&1
