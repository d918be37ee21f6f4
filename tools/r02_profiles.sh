# Round-2 measurements: bench (default), serialised launch list of one n=100k evaluation,
# ncu --set full of U2(0) at n=100k and of the tile-task executor at n=400 and n=1600.
set -x
python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err
cat gpurun_out/r02_bench_final.json | head -c 600; echo
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02_launches_100k.csv python tools/once.py 100000 > gpurun_out/r02_ncu_launch.log 2>&1
EVALS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:SyrkMap -s 1 -c 1 -o gpurun_out/r02_prof_u2_100k -f python tools/once.py 100000 > gpurun_out/r02_ncu_u2.log 2>&1
for n in 400 1600; do
  EVALS=2 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:dag_factor -s 1 -c 1 -o gpurun_out/r02_prof_dag_$n -f python tools/once.py $n 0 0 > gpurun_out/r02_ncu_dag_$n.log 2>&1
done
ls -la gpurun_out/
