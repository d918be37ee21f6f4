// bar_lat.cu -- cost of one step "STS; __syncthreads(); LDS (neighbour); DFMA" vs CTA size
// (the POTRF64 step skeleton), and of an 8-DFMA dependent update per step.
#include <cstdio>

template <int WORK>
__global__ void step_loop(double* out, long long* cyc, int iters) {
  __shared__ double sh[1024];
  const int t = threadIdx.x, n = blockDim.x;
  double x = 1.0 + t * 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sh[t] = x;
    __syncthreads();
    const double v = sh[(t + 33) % n];
#pragma unroll
    for (int k = 0; k < WORK; ++k) x = fma(x, 0.999999, v * 1e-3);
  }
  const long long t1 = clock64();
  if (t == 0) *cyc = t1 - t0;
  out[t] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 2000;
  for (int threads : {32, 64, 128, 256, 512, 1024}) {
    for (int w = 0; w < 2; ++w) {
      long long h[2];
      for (int rep = 0; rep < 2; ++rep) {
        if (w == 0) step_loop<1><<<1, threads>>>(out, cyc, iters);
        else step_loop<8><<<1, threads>>>(out, cyc, iters);
        cudaMemcpy(&h[rep], cyc, sizeof(long long), cudaMemcpyDeviceToHost);
      }
      printf("threads=%4d work=%d DFMA: %7.1f cycles/step\n", threads, w ? 8 : 1, (double)h[1] / iters);
    }
  }
  return 0;
}
