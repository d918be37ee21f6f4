#!/bin/bash
# FP64 roofline denominators on this B200 (run under gpurun from the repo root):
#   DMMA (mma.sync m8n8k4 f64) and DFMA sustained loops (tools/probes/fp64_peak.cu),
#   cuBLAS DGEMM 4096^3/8192^3 and cuSOLVER potrf (tools/probes/vendor_fp64.py),
#   SM clocks and throttle reasons sampled by nvidia-smi during the probes.
# Output: profiles/fp64_peak.txt (committed; bench.py reads the DMMA and DGEMM lines).
set -e
out=${1:-gpurun_out/fp64_peak.txt}
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/fp64_peak tools/probes/fp64_peak.cu
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active \
  --format=csv,noheader -lms 200 > gpurun_out/fp64_peak_clocks.csv &
smi=$!
{
  echo "# FP64 peaks measured on $(nvidia-smi --query-gpu=name,driver_version --format=csv,noheader) $(date -u +%FT%TZ)"
  echo "# tools/fp64_peak.sh: tools/probes/fp64_peak.cu (DMMA/DFMA loops) + tools/probes/vendor_fp64.py"
  ./tools/probes/fp64_peak
  python tools/probes/vendor_fp64.py
} > "$out" 2>&1
kill $smi || true
python - "$out" <<'PY'
import csv, statistics, sys
rows = [r for r in csv.reader(open("gpurun_out/fp64_peak_clocks.csv")) if len(r) >= 5]
sm = [float(r[1].split()[0]) for r in rows if r[1].strip().split()[0].isdigit()]
mx = [float(r[2].split()[0]) for r in rows if r[2].strip().split()[0].isdigit()]
reasons = sorted({r[4].strip() for r in rows})
with open(sys.argv[1], "a") as f:
    f.write(f"clocks: samples {len(sm)} sm_mhz median {statistics.median(sm) if sm else 'na'} "
            f"min {min(sm) if sm else 'na'} max_mhz {max(mx) if mx else 'na'} reasons {reasons}\n")
PY
cat "$out"
