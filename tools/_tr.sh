for n in 400 1600; do timeout 120 python tools/tile_task_trace.py $n > gpurun_out/r02_tt_trace_$n.log 2>&1; done
