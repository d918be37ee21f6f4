// potrf_skeleton2.cu -- cycles per step of the 2-D register-tile POTRF64 step, built up one
// ingredient at a time (256 threads, 16 x 16 thread grid, 4 x 4 entries per thread).
#include <cstdio>

constexpr int NT = 256, STEPS = 64, LDS_P = 65, WOFF = 64 * 65;

template <int V>
__global__ void skel(double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* colA = sm;
  double* rowW = sm + WOFF;
  double* dummy = sm + 2 * WOFF;
  const int t = threadIdx.x, tr = t >> 4, tc = t & 15;
  for (int i = t; i < 2 * WOFF + 1024; i += NT) sm[i] = 1.0 + 1e-3 * (i % 97);  // positive pivots
  double v[4][4];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) v[i][k] = 2.0 + 1e-3 * (i + k + t);
  __syncthreads();
  const long long t0 = clock64();
  int bad = -1;
  for (int j = 0; j < STEPS; ++j) {
    const int jk = j >> 4, jt = j & 15;
    if (V >= 5) {  // row j of W (branch-free)
      const bool mine = tr == jt;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = tc + 16 * k;
        double wv = v[0][k];
#pragma unroll
        for (int ii = 1; ii < 4; ++ii) wv = (ii == jk) ? v[ii][k] : wv;
        wv = (c < j) ? wv : (c == j ? 1.0 : 0.0);
        double* dst = mine ? &rowW[j * LDS_P + c] : &dummy[k * 256 + t];
        *dst = wv;
      }
    }
    __syncthreads();
    const double* cj = colA + j * LDS_P;
    const double d = cj[j];
    if (V >= 6 && !(d > 0.0)) {
      bad = j;
      break;
    }
    const double rd = __drcp_rn(d);
    double f[4], src[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = (V >= 7 && !(tr + 16 * i > j)) ? 0.0 : cj[tr + 16 * i] * rd;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = tc + 16 * k;
      src[k] = (V >= 7 && c <= j) ? rowW[j * LDS_P + c] : cj[c];
    }
    const bool rst = V >= 4 && tc == jt;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) v[i][k] = fma(-1e-6 * f[i], src[k], (rst && k == jk) ? 1.5 : v[i][k]);  // stays positive
    const int j1 = (j + 1) & 63;
    if (V >= 3) {
      const int k1 = j1 >> 4;
      const bool pub = tc == (j1 & 15);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double cv = v[i][0];
#pragma unroll
        for (int kk = 1; kk < 4; ++kk) cv = (kk == k1) ? v[i][kk] : cv;
        double* dst = pub ? &colA[j1 * LDS_P + tr + 16 * i] : &dummy[i * 256 + t];
        *dst = cv;
      }
    } else {
      if (tc == (j1 & 15)) colA[j1 * LDS_P + tr] = v[0][0];
    }
  }
  const long long t1 = clock64();
  if (t == 0) *cyc = t1 - t0;
  double s = bad;
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) s += v[i][k];
  out[t] = s;
}

template <int V>
void run(const char* name, double* out, long long* cyc) {
  const int smem = (2 * WOFF + 1024) * 8;
  cudaFuncSetAttribute(skel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    skel<V><<<1, NT, smem>>>(out, cyc);
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  }
  printf("%-58s %7.1f cycles/step\n", name, (double)h / STEPS);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, NT * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  run<2>("S2 barrier, LDS d, rcp, 8 LDS, 16 DFMA, 1 STS", out, cyc);
  run<3>("S3 + branch-free column publication", out, cyc);
  run<4>("S4 + column reset selects", out, cyc);
  run<5>("S5 + branch-free W row publication", out, cyc);
  run<6>("S6 + pivot check (break)", out, cyc);
  run<7>("S7 + row mask on f, source select W/A", out, cyc);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
