set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile_tasks.py -q -x > gpurun_out/r02_persist_tests.log 2>&1; tail -2 gpurun_out/r02_persist_tests.log
for v in 0 1; do
  EXAGEO_U2_PERSIST=$v python tools/nb_sweep.py 8192,10000,20000 256,512 > gpurun_out/r02_persist_$v.log 2>&1
  EXAGEO_U2_PERSIST=$v python tools/u2_trace.py 10000 256 > gpurun_out/r02_persist_u2_$v.log 2>&1
  EXAGEO_U2_PERSIST=$v python tools/quick_timing.py 60000 100000 >> gpurun_out/r02_persist_$v.log 2>&1
done
cat gpurun_out/r02_persist_0.log gpurun_out/r02_persist_1.log; head -4 gpurun_out/r02_persist_u2_*.log
