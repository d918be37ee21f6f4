// Probe: do DMMA (tensor pipe) and DFMA (FP64 pipe) run concurrently on sm_100a?
// Warps 0..W-1 issue DMMA, warps W..2W-1 issue DFMA; report combined TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__device__ void dmma_body(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <int NACC>
__device__ void dfma_body(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC];
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}
// mode 0: all DMMA, 1: all DFMA, 2: half warps DMMA + half DFMA
__global__ void mix(double* out, int it_mma, int it_fma, int mode) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && warp < nw / 2);
  if (do_mma) dmma_body<8>(out, it_mma, 1.0);
  else dfma_body<16>(out, it_fma, 1.0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int warps = 16, grid = sms * 2;
  // iterations chosen so each mode runs ~similar time
  const int it_mma = 20000, it_fma = 20000 * 16 * 8 * 4 * 2 / (2 * 16 * 32) / 1;  // equal flops per warp
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<grid, 32 * warps>>>(out, 100, 100, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    mix<<<grid, 32 * warps>>>(out, it_mma, it_fma, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double f_mma_warp = 2.0 * 8 * 8 * 4 * 8 * it_mma;   // per warp
    const double f_fma_warp = 2.0 * 16 * 32 * (double)it_fma;  // per warp
    double flops;
    if (mode == 0) flops = f_mma_warp * warps * grid;
    else if (mode == 1) flops = f_fma_warp * warps * grid;
    else flops = (f_mma_warp + f_fma_warp) * (warps / 2) * grid;
    printf("mode %d (%s): %.2f TFLOP/s  (%.2f ms)  %s\n", mode, mode == 0 ? "DMMA" : mode == 1 ? "DFMA" : "mixed",
           flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
