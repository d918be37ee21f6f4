// potrf_skeleton.cu -- cycles per elimination step of POTRF64-like skeletons (256 threads),
// adding one ingredient at a time: barrier + dependent shared load/store; + reciprocal;
// + 4 row loads and 16 FMAs; + divergent publication of one column; the real pivot chain.
#include <cstdio>

constexpr int NT = 256, STEPS = 64;

template <int V>
__global__ void skel(double* out, long long* cyc) {
  __shared__ double col[STEPS + 1][80];
  __shared__ double row[80];
  const int t = threadIdx.x, tr = t >> 4, tc = t & 15;
  for (int i = t; i < (STEPS + 1) * 80; i += NT) (&col[0][0])[i] = 1.0 + 1e-3 * (i % 97);
  double v[4][4];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) v[i][k] = 1.0 + 1e-3 * (i + k + t);
  __syncthreads();
  const long long t0 = clock64();
  for (int j = 0; j < STEPS; ++j) {
    __syncthreads();
    const double d = col[j][j & 63];
    double rd = d;
    if (V >= 1) rd = __drcp_rn(d);
    if (V == 0) {
      v[0][0] = fma(v[0][0], rd, 1e-9);
      if (t == ((j + 1) & 63)) col[j + 1][(j + 1) & 63] = v[0][0];
    } else if (V == 1) {
      v[0][0] = fma(v[0][0], rd, 1e-9);
      if (t == ((j + 1) & 63)) col[j + 1][(j + 1) & 63] = v[0][0];
    } else {
      double f[4], src[4];
      for (int i = 0; i < 4; ++i) f[i] = col[j][tr + 16 * i] * rd;
      for (int k = 0; k < 4; ++k) src[k] = (V >= 3 && tc + 16 * k <= j) ? row[tc + 16 * k] : col[j][tc + 16 * k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) v[i][k] = fma(-f[i], src[k], v[i][k]);
      if (V >= 3) {
        const int j1 = j + 1;
        if (tc == (j1 & 15)) {
          const int k1 = (j1 >> 4) & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            double cv = v[i][0];
#pragma unroll
            for (int kk = 1; kk < 4; ++kk) cv = (kk == k1) ? v[i][kk] : cv;
            col[j1][tr + 16 * i] = cv;
          }
        }
        if (tr == (j & 15) && tc < 4) row[tc] = v[0][tc & 3];
      } else {
        if (tc == ((j + 1) & 15)) col[j + 1][tr] = v[0][0];
      }
    }
  }
  const long long t1 = clock64();
  if (t == 0) *cyc = t1 - t0;
  double s = 0;
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) s += v[i][k];
  out[t] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, NT * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"barrier + LDS + FMA + STS", "+ __drcp_rn on the chain", "+ 4 LDS f, 4 LDS src, 16 DFMA",
                         "+ W/column publication (divergent)"};
  for (int v = 0; v < 4; ++v) {
    long long h = 0;
    for (int rep = 0; rep < 3; ++rep) {
      if (v == 0) skel<0><<<1, NT>>>(out, cyc);
      if (v == 1) skel<1><<<1, NT>>>(out, cyc);
      if (v == 2) skel<2><<<1, NT>>>(out, cyc);
      if (v == 3) skel<3><<<1, NT>>>(out, cyc);
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    }
    printf("%-45s %7.1f cycles/step\n", names[v], (double)h / STEPS);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
