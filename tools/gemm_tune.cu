// gemm_tune.cu -- timing harness for DMMA contraction configurations (development tool).
// Times the step-k trailing update (SyrkMap) over a synthetic panel workspace.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1708_02835_b200/csrc \
//        -o tools/gemm_tune tools/gemm_tune.cu
#include <cstdio>
#include <cstdlib>

#include "gemm_dmma.cuh"

using namespace exageo;
using namespace exageo::gemm;

__global__ void fill(double* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 1e-3 * (double)((i * 2654435761ull) % 1000) / 1000.0;
}

template <class C>
void run(const char* name, const Layout& L, double* ws, int k, int reps, int band = 1) {
  if (set_smem<C, true, SyrkMap>() != cudaSuccess) {
    printf("%-40s smem attr failed\n", name);
    return;
  }
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.k = k;
  map.Mb = (int)((L.N - (int64_t)(k + 1) * L.nb) / 128);
  map.cb_lo = 0;
  map.cb_hi = map.Mb;
  map.band = band;
  const double flops = (double)map.blocks(C::BM, C::BN) * 2.0 * C::BM * C::BN * L.nb;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch<C, true>(map, nullptr, 0);
  cudaDeviceSynchronize();
  float best = 1e30f, tot = 0.f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch<C, true>(map, nullptr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
    tot += ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("%-44s band=%2d k=%d blocks=%8lld best %8.3f ms  %6.2f TF  (avg %6.2f TF) %s\n", name, band, k,
         (long long)map.blocks(C::BM, C::BN), best, flops / best / 1e9, flops / (tot / reps) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 40000;
  Layout L;
  L.n = n;
  L.nb = 512;
  L.T = (int)((n + 511) / 512);
  L.N = (int64_t)L.T * 512;
  double* ws;
  const size_t bytes = (size_t)L.total() * 8 + 4096;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  fill<<<1024, 256>>>(ws, (int64_t)(bytes / 8));
  cudaDeviceSynchronize();
  printf("n=%lld T=%d workspace %.2f GB\n", (long long)n, L.T, bytes / 1e9);
  for (int k : {0}) {
    run<Cfg<64, 64, 8, 2, 2, 4, 4>>("64x64x8 w2x2 st4 minb4 (32x32)", L, ws, k, 3, 8);
    run<Cfg<64, 64, 8, 2, 2, 5, 4>>("64x64x8 w2x2 st5 minb4 (32x32)", L, ws, k, 3, 8);
    run<Cfg<64, 64, 8, 2, 2, 6, 4>>("64x64x8 w2x2 st6 minb4 (32x32)", L, ws, k, 3, 8);
    run<Cfg<64, 64, 4, 2, 2, 8, 4>>("64x64x4 w2x2 st8 minb4 (32x32)", L, ws, k, 3, 8);
    run<Cfg<64, 64, 4, 2, 2, 12, 4>>("64x64x4 w2x2 st12 minb4 (32x32)", L, ws, k, 3, 8);
    run<Cfg<64, 64, 8, 2, 2, 3, 4>>("64x64x8 w2x2 st3 minb4 (32x32)", L, ws, k, 3, 8);
  }
  return 0;
}
