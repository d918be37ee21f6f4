// potrf_bench.cu -- latency of the 64x64 diagonal-block POTRF (+inverse) kernel and of the
// panel GEMMs at a few sizes (development tool). Links potrf_reduce.cu / gemm_dmma.cu.
#include <cmath>
#include <cstdio>
#include <vector>

#include "internal.h"

using namespace exageo;
#ifdef EXAGEO_POTRF_TRACE
namespace exageo {
cudaError_t potrf_trace_read(long long* out);
}
#endif

__global__ void make_spd(double* a, int64_t lda, int n) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int r = idx % n, c = idx / n;
    a[(int64_t)c * lda + r] = (r == c) ? (double)n : 1.0 / (1.0 + r + c);
  }
}

int main() {
  potrf_init();
  gemm_init();
  const int64_t lda = 4096;
  double *a, *W, *slot;
  int* info;
  cudaMalloc(&a, sizeof(double) * lda * 64);
  cudaMalloc(&W, sizeof(double) * 64 * 64);
  cudaMalloc(&slot, sizeof(double));
  cudaMalloc(&info, sizeof(int));
  cudaMemset(info, 0, sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    make_spd<<<64, 256>>>(a, lda, 64);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) {
      make_spd<<<64, 256>>>(a, lda, 64);
      launch_potrf_block(a, lda, W, slot, info, 0, 0);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("potrf_block+make_spd: %.2f us per call\n", 1000.f * ms / 20);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) make_spd<<<64, 256>>>(a, lda, 64);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("make_spd alone: %.2f us per call\n", 1000.f * ms / 20);
  }
#ifdef EXAGEO_POTRF_TRACE
  {
    long long tr[64];
    make_spd<<<64, 256>>>(a, lda, 64);
    launch_potrf_block(a, lda, W, slot, info, 0, 0);
    cudaDeviceSynchronize();
    potrf_trace_read(tr);
    printf("trace (cycles from kernel start): load %lld strips %lld %lld %lld %lld  W done %lld  end %lld\n",
           tr[1] - tr[0], tr[2] - tr[0], tr[3] - tr[0], tr[4] - tr[0], tr[5] - tr[0], tr[6] - tr[0], tr[7] - tr[0]);
    printf("K0 cycles per pivot:");
    for (int j = 0; j < 16; ++j) printf(" %lld", tr[32 + j]);
    printf("\n");
  }
#endif
  int h;
  cudaMemcpy(&h, info, sizeof(int), cudaMemcpyDeviceToHost);
  printf("info=%d err=%s\n", h, cudaGetErrorString(cudaGetLastError()));
  {  // correctness: L L^T = A, W L = I, upper parts zero, slot = sum log L_jj
    make_spd<<<64, 256>>>(a, lda, 64);
    launch_potrf_block(a, lda, W, slot, info, 0, 0);
    std::vector<double> hL(64 * 64), hW(64 * 64);
    double hs;
    cudaMemcpy2D(hL.data(), 64 * sizeof(double), a, lda * sizeof(double), 64 * sizeof(double), 64,
                 cudaMemcpyDeviceToHost);
    cudaMemcpy(hW.data(), W, sizeof(double) * 64 * 64, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hs, slot, sizeof(double), cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0, up = 0, ls = 0;
    for (int i = 0; i < 64; ++i) {
      ls += std::log(hL[i * 64 + i]);
      for (int j = 0; j < 64; ++j) {
        if (j > i) up = std::fmax(up, std::fabs(hL[j * 64 + i]) + std::fabs(hW[j * 64 + i]));
        double s1 = 0, s2 = 0;
        for (int k = 0; k < 64; ++k) {
          s1 += hL[k * 64 + i] * hL[k * 64 + j];
          s2 += hW[k * 64 + i] * hL[j * 64 + k];
        }
        const double aij = (i == j) ? 64.0 : 1.0 / (1.0 + i + j);
        e1 = std::fmax(e1, std::fabs(s1 - aij));
        e2 = std::fmax(e2, std::fabs(s2 - (i == j ? 1.0 : 0.0)));
      }
    }
    printf("check: max|LL^T-A|=%.3e max|WL-I|=%.3e upper=%.3e slot-err=%.3e\n", e1, e2, up, hs - ls);
  }
  // panel GEMMs
  for (int64_t M : {1024, 16384, 100000}) {
    double *A, *B, *C;
    cudaMalloc(&A, sizeof(double) * M * 512);
    cudaMalloc(&C, sizeof(double) * M * 64);
    cudaMalloc(&B, sizeof(double) * 64 * 512);
    cudaMemset(A, 0, sizeof(double) * M * 512);
    cudaMemset(B, 0, sizeof(double) * 64 * 512);
    cudaMemset(C, 0, sizeof(double) * M * 64);
    for (int K : {64, 256, 448}) {
      launch_gemm_panel(M, 64, K, A, M, B, 64, C, M, true, info, 0);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch_gemm_panel(M, 64, K, A, M, B, 64, C, M, true, info, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1000.0 * ms / 10;
      printf("gemm_panel M=%lld K=%d: %.2f us  (%.2f TF)\n", (long long)M, K, us, 2.0 * M * 64 * K / us / 1e6);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}
