# Round-2 closing run (after the right-looking panel and the pool's joint polling): full GPU
# suite, smoke, bench, executor timing, MLE timing, launch list of one n=100k evaluation.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02f4_tests.log 2>&1; tail -3 gpurun_out/r02f4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f4_smoke.log 2>&1; tail -2 gpurun_out/r02f4_smoke.log
python bench.py > gpurun_out/r02f4_bench.json 2> gpurun_out/r02f4_bench.err
head -c 300 gpurun_out/r02f4_bench.json; echo
python tools/tile_tasks_timing.py 400 800 1600 2400 3200 > gpurun_out/r02f4_exec_timing.txt 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02f4_mle.txt 2>&1
python tools/tile_task_trace.py 1600 > gpurun_out/r02f4_trace_n1600.txt 2>&1
python tools/tile_task_trace.py 400 > gpurun_out/r02f4_trace_n400.txt 2>&1
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02f4_launches_100k.csv python tools/once.py 100000 0 0 > gpurun_out/r02f4_ncu_launch.log 2>&1
