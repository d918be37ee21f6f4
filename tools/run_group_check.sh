# super-panel trailing update: tuner timing per group size, ncu DRAM bytes of U2(0), GPU suite
set -x
timeout 400 ./tools/gemm_tune 100000 > gpurun_out/tune_group.log 2>&1
timeout 300 python tools/quick_timing.py 100000 > gpurun_out/qt100k_group.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:SyrkMap -s 1 -c 1 \
    -o gpurun_out/prof_u2_group python tools/quick_timing.py 100000 > gpurun_out/ncu_group.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_group.log 2>&1
