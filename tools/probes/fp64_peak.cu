// Probe: sustained FP64 throughput on sm_100a for DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used to derive the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC][2];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dmma_loop<8><<<grid, block>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
    printf("DMMA warps/CTA=%d  2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<16><<<grid, block>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<16><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)grid.x * block.x;
    printf("DFMA warps/CTA=%d 2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  // sustained DMMA for ~4 s
  {
    int warps = 8, iters = 400000;
    dim3 grid(sms * 2), block(32 * warps);
    cudaEventRecord(e0);
    dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
    printf("DMMA sustained: %.2f TFLOP/s (%.1f ms)\n", flops / ms / 1e9, ms);
  }
  return 0;
}
