# Round-2 measurements at the nb = 2048 headline layout: bench (default), serialised launch list of
# one n=100k evaluation, ncu --set full of U2(0) at n=100k, the per-step U2 timeline.
set -x
python bench.py > gpurun_out/r02_bench_final2.json 2> gpurun_out/r02_bench_final2.err
head -c 300 gpurun_out/r02_bench_final2.json; echo
python tools/u2_trace.py 100000 > gpurun_out/r02_u2_100k.log 2>&1
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02_launches_100k.csv python tools/once.py 100000 > gpurun_out/r02_ncu_launch.log 2>&1
EVALS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:SyrkMap -s 1 -c 1 -o gpurun_out/r02_prof_u2_100k -f python tools/once.py 100000 > gpurun_out/r02_ncu_u2.log 2>&1
ls -la gpurun_out/ | grep -E "r02_prof_u2_100k|r02_launches_100k"
