for a in "8192 512" "10000 512" "20000 1024" "40000 1024"; do python tools/tail_sweep.py $a 0,2048,2560,3200,4096,5120; done > gpurun_out/r02_tail_sweep2.log 2>&1
cat gpurun_out/r02_tail_sweep2.log
