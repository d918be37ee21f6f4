# Profiling recipe used for profiles/ (run under gpurun from the repo root).
set -x
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/quick_timing.py 100000 > gpurun_out/qt100k.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:SyrkMap -s 1 -c 1 \
    -o gpurun_out/prof_u2_100k python tools/quick_timing.py 100000 > gpurun_out/ncu_full.log 2>&1
