# K2 changes: GPU tests, small/mid n latency, executor timing.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_k2_tests.log 2>&1; tail -3 gpurun_out/r02_k2_tests.log
python tools/tile_tasks_timing.py 400 1600 3200 4000 > gpurun_out/r02_k2_tt.log 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02_k2_mle.log 2>&1
python tools/graph_timing.py 5000 8192 10000 20000 > gpurun_out/r02_k2_gt.log 2>&1
for a in "5000 128" "8192 512" "10000 512"; do python tools/tail_sweep.py $a 0,2048,2900,3600,4400 >> gpurun_out/r02_k2_tail.log 2>&1; done
