// fp64_lat.cu -- dependent-chain latencies of FP64 ops on one warp (clock64 cycles per op).
#include <cstdio>

template <int OP>
__global__ void chain(double* out, double x0, long long* cyc, int iters) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = x;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = fma(x, y, 1e-300);
    if (OP == 1) x = x * y;
    if (OP == 2) x = x + y;
    if (OP == 3) x = __drcp_rn(x);
    if (OP == 4) x = sqrt(x);
    if (OP == 5) x = 1.0 / x;
    if (OP == 6) x = __dsqrt_rn(x) + 0.0;
    if (OP == 7) { x = sh[((int)x) & 63] + 1e-300; }
    if (OP == 8) x = log(x) + 2.0;
    if (OP == 9) { float f = (float)x; x = (double)f * y; }
    if (OP == 10) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * y;
    if (OP == 11) {  // DMMA m8n8k4 accumulator chain
      double c0 = x, c1 = y;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(1e-3), "d"(1e-3));
      x = c0;
      y = c1;
    }
    if (OP == 12) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
      for (int it = 0; it < 3; ++it) r = fma(r, fma(-x, r, 1.0), r);
      x = r;
    }
    if (OP == 13) x = rsqrt(x);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"DFMA", "DMUL", "DADD", "drcp_rn", "sqrt", "1/x", "dsqrt_rn", "LDS(dep)", "log", "F2F+DMUL",
                         "SHFL.f64*y", "DMMA acc", "rcp+3NR", "rsqrt"};
  const int iters = 4096;
  for (int op = 0; op < 14; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 1: chain<1><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 2: chain<2><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 3: chain<3><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 4: chain<4><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 5: chain<5><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 6: chain<6><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 7: chain<7><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 8: chain<8><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 9: chain<9><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 10: chain<10><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 11: chain<11><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 12: chain<12><<<1, 32>>>(out, 1.5, cyc, iters); break;
        case 13: chain<13><<<1, 32>>>(out, 1.5, cyc, iters); break;
      }
      long long h;
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep) printf("%-10s %7.1f cycles/op\n", names[op], (double)h / iters);
    }
  }
  return 0;
}
