# K1 generator rework check: GPU suite, per-phase timings (nu = 0.5 and general nu), probes,
# ncu of the generator. Run under gpurun from the repo root.
set -x
timeout 60 ./tools/probes/bar_lat > gpurun_out/bar_lat.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_gen.log 2>&1
timeout 300 python tools/quick_timing.py 20000 40000 100000 > gpurun_out/qt_gen_nu05.log 2>&1
THETA=1.0,0.03,1.0 timeout 300 python tools/quick_timing.py 20000 40000 > gpurun_out/qt_gen_nu1.log 2>&1
THETA=1.0,0.03,0.8 timeout 300 python tools/quick_timing.py 20000 40000 > gpurun_out/qt_gen_nu08.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_panels -c 1 \
    -o gpurun_out/prof_gen2_100k python tools/quick_timing.py 100000 > gpurun_out/ncu_gen2.log 2>&1
THETA=1.0,0.03,1.0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_panels -c 1 \
    -o gpurun_out/prof_gen2_nu1_40k python tools/quick_timing.py 40000 > gpurun_out/ncu_gen2_nu1.log 2>&1
