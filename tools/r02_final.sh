# Round-2 closing measurements: full GPU suite, smoke, bench (default), launch list of one n=100k
# evaluation, cuSOLVER comparison, executor timing. Run under gpurun from the repo root.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02f_tests.log 2>&1; tail -3 gpurun_out/r02f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f_smoke.log 2>&1; tail -2 gpurun_out/r02f_smoke.log
python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
head -c 400 gpurun_out/r02f_bench.json; echo
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02f_launches_100k.csv python tools/once.py 100000 > gpurun_out/r02f_ncu_launch.log 2>&1
timeout 900 python tools/chol_vs_vendor.py > gpurun_out/r02f_chol_vs_cusolver.log 2>&1
tail -8 gpurun_out/r02f_chol_vs_cusolver.log
python tools/tile_tasks_timing.py 400 800 1600 2400 3200 > gpurun_out/r02f_exec_timing.txt 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02f_mle.txt 2>&1
