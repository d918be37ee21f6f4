// gemm_tune.cu -- timing harness for DMMA contraction configurations (development tool).
// Times the step-k bulk trailing update U2(k) (SyrkMap over panels k+2 .. T-1) on a
// synthetic panel workspace for several tile configurations of the product kernel.
// Reports algorithmic TFLOP/s (the true lower triangle incl. the z row). (A bulk-copy +
// mbarrier variant and cross-stage fragment pipelining were measured in earlier revisions
// of gemm_dmma.cuh: 29.7 and 31.7-32.5 TF.)
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

template <class C, int BULK>
void run(const char* name, const Layout& L, double* ws, int k, int reps, int group = 1) {
  if (set_smem<C, true, SyrkMap>() != cudaSuccess) {
    printf("%-40s smem attr failed\n", name);
    return;
  }
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.Pk = ws + L.off(k);
  map.k = k;
  map.J0 = k + 2;
  map.npan = L.T - k - 2;
  map.row_end = L.N;
  map.group = group;
  const double m = (double)(L.n - (int64_t)(k + 2) * L.nb);
  const double flops = 2.0 * L.nb * (m * (m + 1) / 2 + m);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto go = [&]() {
    if (BULK == 2) launch<C, true, SyrkMap, true>(map, nullptr, 0);
    else launch<C, true>(map, nullptr, 0);
  };
  go();
  cudaDeviceSynchronize();
  float best = 1e30f, tot = 0.f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    go();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
    tot += ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("%-44s %s k=%3d blocks=%8lld best %8.3f ms  %6.2f TF  (avg %6.2f TF) %s\n", name, BULK == 2 ? "preC " : "cpasy",
         k, (long long)map.blocks(C::BM, C::BN), best, flops / best / 1e9, flops / (tot / reps) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 40000;
  const int nb = argc > 2 ? atoi(argv[2]) : 512;
  Layout L;
  L.n = n;
  L.nb = nb;
  L.T = (int)((n + nb - 1) / nb);
  L.N = (int64_t)L.T * nb;
  double* ws;
  const size_t bytes = (size_t)L.total() * 8 + 4096;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  fill<<<1024, 256>>>(ws, (int64_t)(bytes / 8));
  cudaDeviceSynchronize();
  printf("n=%lld T=%d workspace %.2f GB\n", (long long)n, L.T, bytes / 1e9);
  const int group = [&] {  // the product's super-panel size (gemm_dmma.cu syrk_group)
    const int64_t g = ((int64_t)2 << 20) / ((int64_t)nb * nb);
    return (int)(g < 1 ? 1 : (g > 8 ? 8 : g));
  }();
  const int which = argc > 3 ? atoi(argv[3]) : 0;  // 0: all steps below; 1: k = 0 only
  for (int k : {0, L.T / 2, (3 * L.T) / 4}) {
    if (which == 1 && k != 0) break;
    run<Cfg<64, 64, 16, 2, 2, 2, 4>, 2>("64x64x16 st2 preC (product)", L, ws, k, 3, group);
    // the cuBLAS DGEMM kernel on this B200 (ncu: cutlass_80_tensorop_d884gemm_64x128_16x3,
    // 128 threads, 220 registers, 2 CTAs/SM, DMMA pipe 96.5%): warp tiles 32x64 / 64x32
    run<Cfg<64, 128, 16, 2, 2, 3, 2>, 2>("64x128x16 st3 preC 2 CTA (warp 32x64)", L, ws, k, 3, group);
    run<Cfg<128, 64, 16, 2, 2, 3, 2>, 2>("128x64x16 st3 preC 2 CTA (warp 64x32)", L, ws, k, 3, group);
    run<Cfg<64, 128, 16, 2, 2, 2, 2>, 2>("64x128x16 st2 preC 2 CTA", L, ws, k, 3, group);
    run<Cfg<64, 128, 16, 2, 2, 4, 2>, 2>("64x128x16 st4 preC 2 CTA", L, ws, k, 3, group);
    run<Cfg<128, 128, 16, 2, 4, 3, 1>, 2>("128x128x16 st3 preC 8 warps 1 CTA (warp 64x32)", L, ws, k, 3, group);
  }
  return 0;
}
