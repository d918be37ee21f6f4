# Round-2 closing measurements after the chain prefetch by the factor warps and the next-step
# pointers on warp 7: executor timing, MLE, traces, bench, full GPU suite, smoke.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02f5_tests.log 2>&1; tail -3 gpurun_out/r02f5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f5_smoke.log 2>&1; tail -2 gpurun_out/r02f5_smoke.log
python tools/tile_tasks_timing.py 400 800 1600 2400 3200 > gpurun_out/r02f5_exec_timing.txt 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02f5_mle.txt 2>&1
python tools/tile_task_trace.py 1600 > gpurun_out/r02f5_trace_n1600.txt 2>&1
python tools/tile_task_trace.py 400 > gpurun_out/r02f5_trace_n400.txt 2>&1
python bench.py > gpurun_out/r02f5_bench.json 2> gpurun_out/r02f5_bench.err
head -c 200 gpurun_out/r02f5_bench.json; echo
