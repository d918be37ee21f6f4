# ncu --set full of the secondary kernels at n = 100k: K1 (nu = 1/2 closed form, nu = 0.8 via the
# K1T table) and the backward-solve GEMV (predict), plus the launch list of one predict.
set -x
for th in "1.0,0.1,0.5" "1.0,0.1,0.8"; do
  tag=$(echo $th | tr ',' '_')
  THETA=$th EVALS=1 timeout 900 ncu --set full --clock-control none --kernel-name-base mangled -k regex:gen_panels \
      -c 1 -o gpurun_out/r02_prof_k1_$tag -f python tools/once.py 100000 > gpurun_out/r02_ncu_k1_$tag.log 2>&1
done
timeout 900 ncu --set full --clock-control none --kernel-name-base mangled -k regex:gemv_t -c 1 \
    -o gpurun_out/r02_prof_gemvt -f python tools/predict_once.py 100000 1000 > gpurun_out/r02_ncu_gemvt.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base mangled -k regex:"gemv_t|tile_solve|krige" --csv --log-file gpurun_out/r02_predict_launches.csv \
    python tools/predict_once.py 100000 1000 > gpurun_out/r02_ncu_predict.log 2>&1
ls -la gpurun_out | grep r02_prof
