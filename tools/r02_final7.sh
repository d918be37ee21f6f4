# ncu --set full of the executor kernel at n=400 / 1600 with the closing code.
set -x
for n in 400 1600; do
  EVALS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dag_factor -s 1 -c 1 \
      -o gpurun_out/r02_prof_dag_$n -f python tools/once.py $n 0 1 > gpurun_out/r02_ncu_dag_$n.log 2>&1
done
