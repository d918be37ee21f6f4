#!/bin/bash
# Build tools/potrf_bench (K2 latency + correctness, panel GEMM timings) against the product kernels.
set -e
cd "$(dirname "$0")/.."
C=paper_1708_02835_b200/csrc
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -I include -I $C \
  tools/potrf_bench.cu $C/potrf_reduce.cu $C/gemm_dmma.cu -I $(python -c "import sys; sys.path.insert(0,'.'); from paper_1708_02835_b200.build import cutlass_include as c; print(c())") -o tools/potrf_bench
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -I include -I $C -DEXAGEO_POTRF_TRACE \
  tools/potrf_bench.cu $C/potrf_reduce.cu $C/gemm_dmma.cu -I $(python -c "import sys; sys.path.insert(0,'.'); from paper_1708_02835_b200.build import cutlass_include as c; print(c())") -o tools/potrf_bench_trace
