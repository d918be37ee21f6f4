timeout 900 python -m pytest tests/test_gpu_tile_tasks.py -q -x > gpurun_out/r02_tt_tests.log 2>&1; tail -2 gpurun_out/r02_tt_tests.log
for a in "5000 128" "8192 256" "10000 256" "16384 384" "20000 512"; do python tools/tail_sweep.py $a 0,1536,2048,2560,3200,4096; done > gpurun_out/r02_tail_sweep.log 2>&1
cat gpurun_out/r02_tail_sweep.log
