// potrf_trace.cu -- per-step clock64 trace of a copy of the 16-threads-per-row POTRF64
// kernel (development tool; the product kernel is potrf_reduce.cu). Records, for every
// step j, the SM clock at: A = after the barrier (thread of row j+1, slot owner of column
// j+1), B = after its f = a_rj / d_j, C = after its slot loop, and D = thread 0 after the
// barrier.
#include <cstdio>
#include <vector>

constexpr int PB = 64, LDS_P = PB + 1, TPR = 16;
__device__ long long g_tr[PB][4];
#ifdef NOTRACE
#define TRACE_ON false
#else
#define TRACE_ON true
#endif

__global__ void make_spd(double* a, int64_t lda, int n) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int r = idx % n, c = idx / n;
    a[(int64_t)c * lda + r] = (r == c) ? (double)n : 1.0 / (1.0 + r + c);
  }
}

template <int VARIANT>
__global__ void __launch_bounds__(64 * TPR) potrf_traced(double* __restrict__ a, int64_t lda) {
  constexpr int NS = PB / TPR, RPW = 32 / TPR, WOFF = PB * LDS_P;
  extern __shared__ double smem_p[];
  double* colA = smem_p;
  double* rowW = smem_p + WOFF;
  __shared__ double rdj[PB];
  const int tid = threadIdx.x, r = tid / TPR, q = tid % TPR;
  double v[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int c = q + TPR * s;
    v[s] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
  }
  if (q == 0) colA[r] = v[0];
  if (VARIANT == 1 && tid == 0) rdj[0] = __drcp_rn(v[0]);
  for (int j = 0; j < PB; ++j) {
    if (r == j) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int c = q + TPR * s;
        rowW[j * LDS_P + c] = (c < j) ? v[s] : (c == j ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    const bool tr = (r == j + 1) && (q == (j + 1) % TPR);
    if (TRACE_ON && tr) g_tr[j][0] = clock64();
    if (TRACE_ON && tid == 0) g_tr[j][3] = clock64();
    const double d = colA[j * LDS_P + j];
    if (!(d > 0.0)) break;
    if ((tid >> 5) * RPW + RPW - 1 > j) {
      const bool row_active = r > j;
      const double rd = VARIANT == 1 ? rdj[j] : __drcp_rn(d);
      const double f = colA[j * LDS_P + r] * rd;
      if (TRACE_ON && tr) g_tr[j][1] = clock64() + (long long)(f * 0.0);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int c = q + TPR * s;
        const bool isw = c <= j;
        const double src = smem_p[j * LDS_P + c + (isw ? WOFF : 0)];
        const double base = (c == j) ? 0.0 : v[s];
        const double nv = base - f * src;
        const bool act = row_active && (isw || c <= r);
        v[s] = act ? nv : v[s];
        if (act && c == j + 1) {
          colA[(j + 1) * LDS_P + r] = nv;
          if (VARIANT == 1 && r == j + 1) rdj[j + 1] = __drcp_rn(nv);
        }
      }
      if (TRACE_ON && tr) g_tr[j][2] = clock64() + (long long)(v[0] * 0.0);
    }
  }
  __syncthreads();
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx % PB, c = idx / PB;
    if (rr >= c) a[(int64_t)c * lda + rr] = colA[c * LDS_P + rr];
  }
}


// 2-D register tiles: 256 threads as a 16 x 16 grid; thread (tr, tc) owns rows
// r = tr + 16 i and columns c = tc + 16 k (i, k < 4): per step 1 + 4 + 4 shared loads and
// 16 FMAs per thread (the 16-threads-per-row kernel needs 6 loads per 4 FMAs, and its
// shared-memory wavefronts bound each step).
__global__ void __launch_bounds__(256) potrf_2d(double* __restrict__ a, int64_t lda) {
  constexpr int WOFF = PB * LDS_P;
  extern __shared__ double smem_p[];
  double* colA = smem_p;
  double* rowW = smem_p + WOFF;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = tr + 16 * i, c = tc + 16 * k;
      v[i][k] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
    }
  if (tc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) colA[tr + 16 * i] = v[i][0];  // column 0
  }
  for (int j = 0; j < PB; ++j) {
    if (tr == (j & 15)) {  // row j of W
      const int i = j >> 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = tc + 16 * k;
        double wv = 0.0;
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) wv = (ii == i) ? v[ii][k] : wv;
        rowW[j * LDS_P + c] = (c < j) ? wv : (c == j ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    if (TRACE_ON && tid == 16 * ((j + 1) & 15) + ((j + 1) & 15)) g_tr[j][0] = clock64();
    if (TRACE_ON && tid == 0) g_tr[j][3] = clock64();
    const double d = colA[j * LDS_P + j];
    if (!(d > 0.0)) break;
    const double rd = __drcp_rn(d);
    double f[4], src[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = colA[j * LDS_P + tr + 16 * i] * rd;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = tc + 16 * k;
      src[k] = smem_p[j * LDS_P + c + (c <= j ? WOFF : 0)];
    }
    if (TRACE_ON && tid == 16 * ((j + 1) & 15) + ((j + 1) & 15)) g_tr[j][1] = clock64() + (long long)(f[0] * 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = tr + 16 * i;
      const bool row_active = r > j;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = tc + 16 * k;
        const bool isw = c <= j;
        const double base = (c == j) ? 0.0 : v[i][k];
        const double nv = base - f[i] * src[k];
        const bool act = row_active && (isw || c <= r);
        v[i][k] = act ? nv : v[i][k];
        if (act && c == j + 1) colA[(j + 1) * LDS_P + r] = nv;
      }
    }
    if (TRACE_ON && tid == 16 * ((j + 1) & 15) + ((j + 1) & 15)) g_tr[j][2] = clock64() + (long long)(v[0][0] * 0.0);
  }
  __syncthreads();
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx % PB, c = idx / PB;
    if (rr >= c) a[(int64_t)c * lda + rr] = colA[c * LDS_P + rr];
  }
}


// 2-D register tiles without per-entry predication: rows at or above the pivot get f = 0,
// upper-triangle entries of a tile take harmless garbage (never read), the column-j
// reset and the column-(j+1) publication touch one tile column of 2 lanes per warp.
__global__ void __launch_bounds__(256) potrf_2d2(double* __restrict__ a, int64_t lda) {
  constexpr int WOFF = PB * LDS_P;
  extern __shared__ double smem_p[];
  double* colA = smem_p;
  double* rowW = smem_p + WOFF;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = tr + 16 * i, c = tc + 16 * k;
      v[i][k] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
    }
  if (tc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) colA[tr + 16 * i] = v[i][0];
  }
  for (int j = 0; j < PB; ++j) {
    const int jk = j >> 4, jt = j & 15;
    if (tr == jt) {  // row j of W
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = tc + 16 * k;
        double wv = v[0][k];
#pragma unroll
        for (int ii = 1; ii < 4; ++ii) wv = (ii == jk) ? v[ii][k] : wv;
        rowW[j * LDS_P + c] = (c < j) ? wv : (c == j ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    const bool trc = tid == 16 * ((j + 1) & 15) + ((j + 1) & 15);
    if (TRACE_ON && trc) g_tr[j][0] = clock64();
    if (TRACE_ON && tid == 0) g_tr[j][3] = clock64();
    const double* cj = colA + j * LDS_P;
    const double d = cj[j];
    if (!(d > 0.0)) break;
    const double rd = __drcp_rn(d);
    double f[4], src[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = (tr + 16 * i > j) ? cj[tr + 16 * i] * rd : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = tc + 16 * k;
      src[k] = (c <= j) ? rowW[j * LDS_P + c] : cj[c];
    }
    if (TRACE_ON && trc) g_tr[j][1] = clock64() + (long long)(f[0] * 0.0);
    if (tc == jt) {  // column j turns from a_rj into w_rj = 0 - f_r
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) v[i][k] = (k == jk) ? 0.0 : v[i][k];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) v[i][k] -= f[i] * src[k];
    if (TRACE_ON && trc) g_tr[j][2] = clock64() + (long long)(v[0][0] * 0.0);
    const int j1 = j + 1;
    if (tc == (j1 & 15) && j1 < PB) {  // publish column j+1
      const int k1 = j1 >> 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double cv = v[i][0];
#pragma unroll
        for (int kk = 1; kk < 4; ++kk) cv = (kk == k1) ? v[i][kk] : cv;
        colA[j1 * LDS_P + tr + 16 * i] = cv;
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx % PB, c = idx / PB;
    if (rr >= c) a[(int64_t)c * lda + rr] = colA[c * LDS_P + rr];
  }
}


// 2-D register tiles, branch-free publication: every thread stores every step, to the real
// location or to a private dummy slot (address select), so no divergent branch and no
// reconvergence sits on the pivot chain (a probe measured ~320 cycles per step for the
// divergent publication of one column).
__global__ void __launch_bounds__(256) potrf_2d3(double* __restrict__ a, int64_t lda) {
  constexpr int WOFF = PB * LDS_P;
  extern __shared__ double smem_p[];
  double* colA = smem_p;
  double* rowW = smem_p + WOFF;
  double* dummy = smem_p + 2 * WOFF;  // 256 x 4 private slots
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = tr + 16 * i, c = tc + 16 * k;
      v[i][k] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
    }
  if (tc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) colA[tr + 16 * i] = v[i][0];
  }
  for (int j = 0; j < PB; ++j) {
    const int jk = j >> 4, jt = j & 15;
    {  // row j of W: threads with tr == jt store for real
      const bool mine = tr == jt;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = tc + 16 * k;
        double wv = v[0][k];
#pragma unroll
        for (int ii = 1; ii < 4; ++ii) wv = (ii == jk) ? v[ii][k] : wv;
        wv = (c < j) ? wv : (c == j ? 1.0 : 0.0);
        double* dst = mine ? &rowW[j * LDS_P + c] : &dummy[k * 256 + tid];
        *dst = wv;
      }
    }
    __syncthreads();
    const double* cj = colA + j * LDS_P;
    const double d = cj[j];
    if (!(d > 0.0)) break;
    const double rd = __drcp_rn(d);
    double f[4], src[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = (tr + 16 * i > j) ? cj[tr + 16 * i] * rd : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = tc + 16 * k;
      src[k] = (c <= j) ? rowW[j * LDS_P + c] : cj[c];
    }
    const bool rst = tc == jt;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) v[i][k] = fma(-f[i], src[k], (rst && k == jk) ? 0.0 : v[i][k]);
    const int j1 = j + 1;
    if (j1 < PB) {
      const int k1 = j1 >> 4;
      const bool pub = tc == (j1 & 15);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double cv = v[i][0];
#pragma unroll
        for (int kk = 1; kk < 4; ++kk) cv = (kk == k1) ? v[i][kk] : cv;
        double* dst = pub ? &colA[j1 * LDS_P + tr + 16 * i] : &dummy[i * 256 + tid];
        *dst = cv;
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx % PB, c = idx / PB;
    if (rr >= c) a[(int64_t)c * lda + rr] = colA[c * LDS_P + rr];
  }
}

template <int V>
void run(const char* name, double* a, int64_t lda) {
  const int smem = 2 * PB * LDS_P * sizeof(double);
  cudaFuncSetAttribute(potrf_traced<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(potrf_2d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(potrf_2d2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(potrf_2d3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 256 * 4 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 20; ++rep) {
    make_spd<<<64, 256>>>(a, lda, 64);
    cudaEventRecord(e0);
    if (V == 4) potrf_2d3<<<1, 256, smem + 256 * 4 * 8>>>(a, lda);
    else if (V == 3) potrf_2d2<<<1, 256, smem>>>(a, lda);
    else if (V == 2) potrf_2d<<<1, 256, smem>>>(a, lda);
    else potrf_traced<V><<<1, 64 * TPR, smem>>>(a, lda);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  long long t[PB][4];
  cudaMemcpyFromSymbol(t, g_tr, sizeof(t));
  printf("%s: best %.2f us, steps (cycles) A->B (rcp/f)  B->C (slots)  C->A' (to next barrier exit)  D->D'\n", name,
         1000.f * best);
  double sab = 0, sbc = 0, sca = 0, sdd = 0;
  for (int j = 0; j + 1 < PB - 1; ++j) {
    sab += t[j][1] - t[j][0];
    sbc += t[j][2] - t[j][1];
    sca += t[j + 1][0] - t[j][2];
    sdd += t[j + 1][3] - t[j][3];
    if (j % 8 == 0)
      printf("  j=%2d  %5lld %5lld %5lld  | %5lld\n", j, t[j][1] - t[j][0], t[j][2] - t[j][1], t[j + 1][0] - t[j][2],
             t[j + 1][3] - t[j][3]);
  }
  const int m = PB - 2;
  printf("  mean  %5.0f %5.0f %5.0f  | %5.0f\n", sab / m, sbc / m, sca / m, sdd / m);
}

int main() {
  const int64_t lda = 4096;
  double* a;
  cudaMalloc(&a, sizeof(double) * lda * 64);
  std::vector<double> h0(64 * 64), h2(64 * 64);
  run<0>("baseline (rcp after the barrier)", a, lda);
  cudaMemcpy2D(h0.data(), 64 * 8, a, lda * 8, 64 * 8, 64, cudaMemcpyDeviceToHost);
  run<1>("rcp by the producer before the barrier", a, lda);
  run<2>("2-D register tiles, 256 threads", a, lda);
  cudaMemcpy2D(h2.data(), 64 * 8, a, lda * 8, 64 * 8, 64, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int c = 0; c < 64; ++c)
    for (int r = c; r < 64; ++r) diff += h0[c * 64 + r] != h2[c * 64 + r];
  printf("2-D vs baseline: %d lower entries differ (bitwise)\n", diff);
  run<3>("2-D register tiles, predication-free", a, lda);
  cudaMemcpy2D(h2.data(), 64 * 8, a, lda * 8, 64 * 8, 64, cudaMemcpyDeviceToHost);
  diff = 0;
  for (int c = 0; c < 64; ++c)
    for (int r = c; r < 64; ++r) diff += h0[c * 64 + r] != h2[c * 64 + r];
  printf("2-D predication-free vs baseline: %d lower entries differ (bitwise)\n", diff);
  run<4>("2-D register tiles, branch-free publication", a, lda);
  cudaMemcpy2D(h2.data(), 64 * 8, a, lda * 8, 64 * 8, 64, cudaMemcpyDeviceToHost);
  diff = 0;
  for (int c = 0; c < 64; ++c)
    for (int r = c; r < 64; ++r) diff += h0[c * 64 + r] != h2[c * 64 + r];
  printf("2-D branch-free vs baseline: %d lower entries differ (bitwise)\n", diff);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
