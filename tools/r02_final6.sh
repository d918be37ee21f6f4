# Round-2 closing run after the pool ticket lookahead: full GPU suite, smoke, executor timing, MLE, traces, bench.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02f6_tests.log 2>&1; tail -3 gpurun_out/r02f6_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f6_smoke.log 2>&1; tail -2 gpurun_out/r02f6_smoke.log
python tools/tile_tasks_timing.py 400 800 1600 2400 3200 > gpurun_out/r02f6_exec_timing.txt 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02f6_mle.txt 2>&1
python tools/tile_task_trace.py 1600 > gpurun_out/r02f6_trace_n1600.txt 2>&1
python tools/tile_task_trace.py 400 > gpurun_out/r02f6_trace_n400.txt 2>&1
python bench.py > gpurun_out/r02f6_bench.json 2> gpurun_out/r02f6_bench.err
head -c 200 gpurun_out/r02f6_bench.json; echo
