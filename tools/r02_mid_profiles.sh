# ncu --set full of the first bulk trailing update U2(0) at mid n: nb = 128 (round-1 tiling) vs the
# automatic nb = 512 at n = 10k, and n = 20k at nb = 512 (tools/summarize_profiles.py --mid).
set -x
for cfg in "10000 128" "10000 512" "20000 512"; do
  set -- $cfg
  EVALS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:SyrkMap -s 1 -c 1 \
      -o gpurun_out/r02_prof_u2_n$1_nb$2 -f python tools/once.py $1 $2 > gpurun_out/r02_ncu_u2_n$1_nb$2.log 2>&1
done
