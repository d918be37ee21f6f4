set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_nb1024.log 2>&1
python bench.py > gpurun_out/bench_nb1024.json 2> gpurun_out/bench_nb1024.err
timeout 300 python tools/quick_timing.py 100000 > gpurun_out/qt_nb1024.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:SyrkMap -s 1 -c 1 \
    -o gpurun_out/prof_u2_nb1024 python tools/quick_timing.py 100000 > gpurun_out/ncu_nb1024.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/plain_bench_g.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_nb1024.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_g.log 2>&1
