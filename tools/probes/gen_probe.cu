// Probe: cost of generating one 64 x 64 Matern tile (nu = 1/2) on one CTA of 256 threads, the
// executor's GEN task body, timed with clock64 (tools/probes; not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1708_02835_b200/csrc/matern_eval.cuh"
using namespace exageo;
__global__ void probe(const double* x, const double* y, MaternConsts mc, double* T, long long* cyc, int variant) {
  __shared__ double xc[64], yc[64];
  const int r = threadIdx.x & 63, cb = 16 * (threadIdx.x >> 6);
  if (threadIdx.x < 64) { xc[threadIdx.x] = x[threadIdx.x]; yc[threadIdx.x] = y[threadIdx.x]; }
  const double xr = x[64 + r], yr = y[64 + r];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
#pragma unroll 4
    for (int cc = 0; cc < 16; ++cc) {
      double v;
      if (variant == 0) v = mat::matern_eval_k<1>(mat::dist2d(xr, yr, xc[cb + cc], yc[cb + cc], mc), mc, nullptr);
      else if (variant == 1) { double dx = xr - xc[cb + cc], dy = yr - yc[cb + cc]; v = sqrt(dx * dx + dy * dy); }
      else { double dx = xr - xc[cb + cc], dy = yr - yc[cb + cc]; v = exp(-(dx * dx + dy * dy)); }
      T[(cb + cc) * 64 + r] = v + rep;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[variant] = (t1 - t0) / 10;
}
int main() {
  double *x, *y, *T; long long* cyc;
  cudaMalloc(&x, 128 * 8); cudaMalloc(&y, 128 * 8); cudaMalloc(&T, 4096 * 8); cudaMallocManaged(&cyc, 64);
  double hx[128]; for (int i = 0; i < 128; ++i) hx[i] = 0.01 * i;
  cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice); cudaMemcpy(y, hx, sizeof hx, cudaMemcpyHostToDevice);
  MaternConsts mc{}; mc.theta1 = 1; mc.inv_theta2 = 10; mc.nu = 0.5; mc.kind = 1; mc.metric = 0;
  for (int v = 0; v < 3; ++v) { probe<<<1, 256>>>(x, y, mc, T, cyc, v); cudaDeviceSynchronize(); }
  for (int v = 0; v < 3; ++v) { probe<<<1, 256>>>(x, y, mc, T, cyc, v); cudaDeviceSynchronize(); }
  printf("cycles per 64x64 tile: matern(nu=1/2) %lld  sqrt only %lld  exp only %lld  (%s)\n", cyc[0], cyc[1], cyc[2],
         cudaGetErrorString(cudaGetLastError()));
}
