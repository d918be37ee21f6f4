set -x
timeout 900 python -m pytest tests/test_gpu_tile_tasks.py tests/test_gpu_graphs.py tests/test_gpu_mle.py -q -x > gpurun_out/r02_tt_tests.log 2>&1; echo "tt tests rc=$?"
tail -2 gpurun_out/r02_tt_tests.log
timeout 600 python tools/tile_tasks_timing.py 400 1600 3000 > gpurun_out/r02_tt_timing.log 2>&1
cat gpurun_out/r02_tt_timing.log
for n in 400 1600; do timeout 120 python tools/tile_task_trace.py $n > gpurun_out/r02_tt_trace_$n.log 2>&1; done
