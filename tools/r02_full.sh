set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_full2.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_gpu_full2.log
timeout 600 python tools/tile_tasks_timing.py 400 1600 3000 3500 > gpurun_out/r02_tt_timing2.log 2>&1
cat gpurun_out/r02_tt_timing2.log
for n in 400 1600; do timeout 120 python tools/tile_task_trace.py $n > gpurun_out/r02_tt_trace_$n.log 2>&1; done
