# Round-2 measurements after the CUTLASS-mainloop trailing update: bench (default), launch list of
# one n=100k evaluation, ncu --set full of U2(0) at n=100k, U2 timeline, cuSOLVER comparison.
set -x
python bench.py > gpurun_out/r02_bench_final3.json 2> gpurun_out/r02_bench_final3.err
head -c 300 gpurun_out/r02_bench_final3.json; echo
python tools/u2_trace.py 100000 > gpurun_out/r02_u2_100k.log 2>&1
python tools/u2_trace.py 10000 > gpurun_out/r02_u2_10k.log 2>&1
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02_launches_100k.csv python tools/once.py 100000 > gpurun_out/r02_ncu_launch.log 2>&1
EVALS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:SyrkMap -s 1 -c 1 -o gpurun_out/r02_prof_u2_100k -f python tools/once.py 100000 > gpurun_out/r02_ncu_u2.log 2>&1
timeout 900 python tools/chol_vs_vendor.py > gpurun_out/r02_chol_vs_cusolver.log 2>&1
tail -8 gpurun_out/r02_chol_vs_cusolver.log
