# Final round-1 measurements: bench (default), launch list of a 1-step bench, ncu --set full of
# the new K2 at n=100k, small-n and config timings. Run under gpurun from the repo root.
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/plain_bench_f.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_f.log 2>&1
timeout 300 python tools/quick_timing.py 100000 > gpurun_out/qt100k_f.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:potrf_block -s 200 -c 1 \
    -o gpurun_out/prof_potrf_final python tools/quick_timing.py 100000 > gpurun_out/ncu_potrf_f.log 2>&1
