# Secondary-kernel profiles (K1 generation, K2 POTRF, panel GEMM) and the n=150k single-GPU point.
# Run under gpurun from the repo root; each ncu capture only after the same command exited 0.
set -x
timeout 400 python tools/quick_timing.py 150000 > gpurun_out/qt150k.log 2>&1
THETA=1.0,0.03,1.0 timeout 200 python tools/quick_timing.py 20000 40000 > gpurun_out/qt_nu1.log 2>&1
timeout 300 python tools/quick_timing.py 100000 > gpurun_out/qt100k_b.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_panels -c 1 \
    -o gpurun_out/prof_gen_100k python tools/quick_timing.py 100000 > gpurun_out/ncu_gen.log 2>&1
THETA=1.0,0.03,1.0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_panels -c 1 \
    -o gpurun_out/prof_gen_nu1_40k python tools/quick_timing.py 40000 > gpurun_out/ncu_gen_nu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:potrf_block -s 200 -c 1 \
    -o gpurun_out/prof_potrf_100k python tools/quick_timing.py 100000 > gpurun_out/ncu_potrf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:DenseMap -s 300 -c 1 \
    -o gpurun_out/prof_panel_100k python tools/quick_timing.py 100000 > gpurun_out/ncu_panel.log 2>&1
ls -la gpurun_out
