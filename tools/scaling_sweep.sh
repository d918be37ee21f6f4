#!/bin/bash
# Multi-GPU scaling sweep of bench.py on one node (SURVEY §8(d) cfg 4; BASELINE configs[3]):
#   weak scaling at constant tile memory per GPU: n = 106k / 150k / 212k / 300k on 1 / 2 / 4 / 8
#   GPUs (process grids 1x1, 1x2, 2x2, 2x4; n^2 / GPUs constant, 45 GB of tiles per GPU);
#   strong scaling at n = 100k (fits one GPU) and n = 150k over 1 / 2 / 4 / 8 GPUs.
# One JSON line per run in $OUT (default gpurun_out/scaling/). Needs as many GPUs as the largest
# N; runs only the N that fit (nvidia-smi -L). Not run on the one-GPU build box.
set -u
OUT=${OUT:-gpurun_out/scaling}
STEPS=${STEPS:-2}
WARMUP=${WARMUP:-1}
mkdir -p "$OUT"
NGPU=$(nvidia-smi -L | wc -l)
run() {  # run N n tag
  local N=$1 n=$2 tag=$3
  [ "$N" -le "$NGPU" ] || { echo "skip $tag: needs $N GPUs, have $NGPU"; return; }
  if [ "$N" -eq 1 ]; then
    python bench.py --n "$n" --steps "$STEPS" --warmup "$WARMUP" --no-extras --no-cpu-baseline \
      > "$OUT/$tag.json" 2> "$OUT/$tag.err"
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus "$N" --n "$n" --steps "$STEPS" --warmup "$WARMUP" \
      --no-extras --no-cpu-baseline > "$OUT/$tag.json" 2> "$OUT/$tag.err"
  fi
  echo "$tag: $(tail -1 "$OUT/$tag.json" | cut -c1-200)"
}
for pair in "1 106000" "2 150000" "4 212000" "8 300000"; do
  set -- $pair
  run "$1" "$2" "weak_N$1_n$2"
done
for n in 100000 150000; do
  for N in 1 2 4 8; do run "$N" "$n" "strong_N${N}_n$n"; done
done
