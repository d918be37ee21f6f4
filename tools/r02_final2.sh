# Launch list of one n=100k evaluation in the bench's configuration (automatic nb and tail hand-off)
# and ncu --set full of the executor kernel at n=400 / 1600 (current code).
set -x
EVALS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/r02f_launches_100k.csv python tools/once.py 100000 0 0 > gpurun_out/r02f_ncu_launch.log 2>&1
for n in 400 1600; do
  EVALS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dag_factor -s 1 -c 1 \
      -o gpurun_out/r02_prof_dag_$n -f python tools/once.py $n 0 1 > gpurun_out/r02_ncu_dag_$n.log 2>&1
done
