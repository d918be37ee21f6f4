// potrf64.cuh -- K2 device code: the PB x PB (PB = 64) diagonal-block Cholesky with
// W = L^{-1} and the log-det partial (the paper's dpotrf at tile granularity, Alg. 2 l.3,
// P:682), shared by the stream-launched potrf_block_kernel (potrf_reduce.cu) and the
// persistent tile-task kernel (dag.cu). Included inside namespace exageo::{anonymous}.
#pragma once

// c (8 x 8, two per lane) += a (8 x 4 row fragment) * b (4 x 8 column fragment), FP64 DMMA;
// lane l holds a = A[l/4][l%4], b = B[l%4][l/4], c = C[l/4][2(l%4) + {0, 1}]
__device__ __forceinline__ void dmma64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---- K2: 64 x 64 diagonal block: one warp factors 16-column strips, seven warps form W ------
// Shared memory: the block A (col-major, ld LDA2 = 68 = 4 mod 16 doubles: the 64-bit fragment
// loads of a half warp -- 4 rows x 4 columns -- hit 32 distinct banks), W = L^{-1} (same
// layout), the inverses T_K = L_KK^{-1} of the four 16 x 16 diagonal blocks (ld LDT), the
// pivots d_j and 1/sqrt(d_j).
constexpr int LDA2 = PB + 4;
constexpr int LDT = 20;
constexpr int kPotrfSmemDoubles = 2 * PB * LDA2 + 4 * 16 * LDT + 2 * PB;

#ifdef EXAGEO_POTRF_TRACE  // development: clock64 stamps of thread 0 (tools/potrf_bench.cu)
__device__ long long g_potrf_trace[64];
#define PTRACE(i)                                       \
  do {                                                  \
    if ((threadIdx.x & 31) == 0) g_potrf_trace[i] = clock64(); \
  } while (0)
#else
#define PTRACE(i) \
  do {            \
  } while (0)
#endif

// 1 / d and 1 / sqrt(d) for normal positive d without a slow path: MUFU seed + Newton steps
// (quadratic convergence from ~2^-22: two steps for 1/d, whose last one is the usual correctly
// rounding update r += r (1 - d r); three for 1/sqrt(d)).
// d <= 0 or NaN gives garbage that the pivot check discards.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
#pragma unroll
  for (int it = 0; it < 2; ++it) r = fma(r, fma(-d, r, 1.0), r);
  return r;
}
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = fma(y, fma(-hd * y, y, 0.5), y);  // y (3/2 - d y^2 / 2)
  return y;
}

__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// 16 x 16 x 16 product on one warp: acc (2 x 2 tiles of 8 x 8) += A B, with A(m, k) and
// B(k, n) read through accessors (shared memory).
template <class FA, class FB>
__device__ __forceinline__ void mm16(double (&acc)[2][2][2], FA A, FB B) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 16; kk += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      af[t] = A(8 * t + fr, kk + fk);
      bf[t] = B(kk + fk, 8 * t + fr);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma64(acc[mt][nt], af[mt], bf[nt]);
  }
}
template <class F>
__device__ __forceinline__ void acc_store(const double (&acc)[2][2][2], F C) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) C(8 * mt + fr, 8 * nt + 2 * fk + e, acc[mt][nt][e]);
}

// Strip K of the block (columns c0 = 16K .. c0+15, rows c0 .. 63, H = 64 - c0 rows) on the
// factor warps w = 0 .. NFW-1, in place in As. Left-looking: first A_strip -= L[c0:, :c0]
// L[c0:c0+16, :c0]^T as m8n8k4 DMMA (warp w: strip rows 16w .. 16w+15; accumulators preloaded
// with A, negated A fragments). Then the unblocked factorization in registers: in every factor
// warp lanes 0..15 hold the 16 rows of the diagonal block (replicated: each warp repeats the
// same operations, bitwise identical) and lanes 16..31 the off-diagonal rows 16 + 16w + l - 16.
// Pivot j: d = a_jj (lane j), f_r = a_rj / d, a_rc -= f_r a_cj (c > j). The next pivot's own
// update is lane-local (chain per pivot: shuffle -> reciprocal -> multiply -> FMA); the column
// a_.j+1 of the diagonal block goes through a per-warp shared buffer, off that chain. Deferred
// scaling as the paper's dpotrf with a reciprocal: identical rows give f = 1 and an exact zero
// pivot. Returns the first bad pivot (strip-local) or -1 (same in every factor warp).
constexpr int NFW = 3;  // factor warps

// One instantiation for the four strips (runtime K): the unrolled pivot loop exists once in the
// binary -- four copies pushed the persistent tile-task kernel's K2 out of the instruction cache.
__device__ __forceinline__ int factor_strip(const int K, double* As, double* dv, double* rs, double* colbuf) {
  const int c0 = 16 * K, H = PB - c0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int NW = H > 32 ? (H - 16) / 16 : 1;  // factor warps with rows in this strip
  if (c0 > 0) {
    if (16 * w < H) {  // this warp's 16 strip rows of the update
      const int fr = lane >> 2, fk = lane & 3;
      const int rb = c0 + 16 * w;
      double acc[2][2][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[mt][nt][e] = As[(c0 + 8 * nt + 2 * fk + e) * LDA2 + rb + 8 * mt + fr];
#pragma unroll 4
      for (int kk = 0; kk < c0; kk += 4) {
        const double* col = As + (kk + fk) * LDA2 + fr;
        double af[2], bf[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          af[t] = -col[rb + 8 * t];
          bf[t] = col[c0 + 8 * t];
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma64(acc[mt][nt], af[mt], bf[nt]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) As[(c0 + 8 * nt + 2 * fk + e) * LDA2 + rb + 8 * mt + fr] = acc[mt][nt][e];
    }
    named_sync(6, 32 * NFW);
  }
  int bad = -1;
  if (w < NW) {
    // strip-local row of this lane: diagonal rows 0..15, then this warp's off-diagonal rows
    const int r = (lane < 16) ? lane : 16 + 16 * w + (lane - 16);
    const bool valid = r < H;
    double v[16], dd[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = (valid && c <= r) ? As[(c0 + c) * LDA2 + c0 + r] : 0.0;
    double* cb = colbuf + w * 32;  // 16 doubles per pivot, double buffered
    if (lane < 16) cb[lane] = v[0];
    __syncwarp();
    double dn = v[0];  // lane j: its own updated diagonal a_jj, ready before the broadcast
#ifdef EXAGEO_POTRF_TRACE
    long long tj[17];
    tj[0] = clock64();
#endif
    // software-pipelined: the broadcast and reciprocal of pivot j+1 are issued as soon as its
    // diagonal is known, ahead of pivot j's remaining row updates (which fill their latency)
    double d = __shfl_sync(0xffffffffu, dn, 0);
    double rd = rcp_nr(d);
    double dm = 1.0;  // lane j < 16: its own pivot d_j
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      dd[j] = d;
      dm = (lane == j) ? d : dm;
      bad = (bad < 0 && !(d > 0.0)) ? j : bad;
      const double f = (r > j) ? v[j] * rd : 0.0;
      const double* cj = cb + 16 * (j & 1);  // a_cj, c = 0..15, of the diagonal block
      double d_next = 0.0, rd_next = 0.0;
      if (j + 1 < 16) {
        dn = fma(-f, v[j], v[j + 1]);  // lane j+1: a_{j+1,j+1} - f a_{j+1,j}, lane-local
        d_next = __shfl_sync(0xffffffffu, dn, j + 1);
        rd_next = rcp_nr(d_next);
        v[j + 1] = fma(-f, cj[j + 1], v[j + 1]);
        if (lane < 16) cb[16 * ((j + 1) & 1) + lane] = v[j + 1];  // column j+1 for the next pivot
      }
#pragma unroll
      for (int c = j + 2; c < 16; ++c) v[c] = fma(-f, cj[c], v[c]);
      __syncwarp();
      d = d_next;
      rd = rd_next;
#ifdef EXAGEO_POTRF_TRACE
      tj[j + 1] = clock64();
#endif
    }
#ifdef EXAGEO_POTRF_TRACE
    if (c0 == 0 && lane == 0 && w == 0)
      for (int j = 0; j < 16; ++j) g_potrf_trace[32 + j] = tj[j + 1] - tj[j];
#endif
    // 1/sqrt(d_j) by lane j (own pivot), shared within the warp by shuffles (warp 0 also
    // publishes d_j and 1/sqrt(d_j) for the helper warps); then L_rc = a_rc / sqrt(d_c) below
    // the diagonal, L_cc = d_c / sqrt(d_c), zeros above -- into As (helper warp 7 copies the strip
    // to global memory: no global stores queue up in front of the factor warps' loads)
    const double ism = rsqrt_nr(dm);
    if (lane < 16 && w == 0) {
      dv[c0 + lane] = dm;
      rs[c0 + lane] = ism;
    }
    double isv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) isv[c] = __shfl_sync(0xffffffffu, ism, c);
    if (valid && (lane >= 16 || w == 0)) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double l = (r > c) ? v[c] * isv[c] : ((r == c) ? dd[c] * isv[c] : 0.0);
        As[(c0 + c) * LDA2 + c0 + r] = l;
      }
    }
  }
  named_sync(6, 32 * NFW);
  return bad;
}

// The paper's dpotrf at tile granularity (Alg. 2 l.3) for the PB x PB diagonal block
// of the current panel, with W = L^{-1} for the panel TRSM as a DMMA product, the partial
// log-determinant sum_j log L_jj = sum_j log(d_j) / 2 (R5), and the first
// non-positive (or NaN) pivot as a global index (R14; every later kernel reads info and exits).
//   warps 0..2: the four strips in order (factor_strip), announcing strip K on named barrier 1+K;
//   warps 3..7: after strip K, T_K = L_KK^{-1} (warp 3, per-lane column substitution) and the
//               W row block K: W_KC = -T_K G_KC, G_KC = sum_{M=C}^{K-1} L_KM W_MC (warp 5, 6, 4
//               for C = 0, 1, 2);
//               they trail the factor warps by about one strip, off their critical path.
// Called by all 256 threads of a CTA with kPotrfSmemDoubles of shared memory at smem_p.
// Loads the block with L1-bypassing loads (ld.global.cg): in the tile-task kernel (dag.cu)
// other SMs wrote it moments ago.
// kFromSmem: the block is already in As (smem_p, ld LDA2; lower triangle and the diagonal 16 x 16
// blocks are read) -- the tile-task chain CTA hands the SYRK result over in shared memory.
// hook(K), K = 0..4, runs on warp 7 (a helper warp without block work) at the start of strip
// K's helper phase (K = 4: after the last one), hook.after_strips() on the factor warps after
// their last strip (idle until the W tail ends): the chain CTA polls and prefetches the next
// step's tiles there and computes its tile pointers. Returns false
// (uniformly) when a pivot failed (info written). nstrips (1..4): 16-column strips holding
// columns < n; the others are identity padding (R12): not factored, L stays the generated
// identity, W gets identity rows, log L_ii = 0 -- the ragged last block of a matrix costs
// only its real strips.
struct NoHook {
  __device__ __forceinline__ void operator()(int) const {}
  __device__ __forceinline__ void after_strips() const {}  // factor warps, after their last strip
};

template <bool kFromSmem = false, class Hook = NoHook>
__device__ __forceinline__ bool potrf64_body(double* __restrict__ a, int64_t lda, double* __restrict__ W,
                                             double* __restrict__ slot, int* __restrict__ info, int64_t pivot_base,
                                             double* smem_p, Hook hook = Hook(), int nstrips = 4) {
  PTRACE(0);
  double* As = smem_p;             // As[c * LDA2 + r]
  double* Ws = As + PB * LDA2;     // Ws[c * LDA2 + r]
  double* Ts = Ws + PB * LDA2;     // Ts[K * 16 * LDT + c * LDT + r]
  double* dv = Ts + 4 * 16 * LDT;  // d_j
  double* rs = dv + PB;            // 1 / sqrt(d_j)
  __shared__ __align__(16) double colbuf[NFW * 32];
  __shared__ int badj;
  __shared__ double lred[2], lgv[PB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!kFromSmem) {  // the lower triangle (and the diagonal blocks' upper halves, never read), 16-byte loads
    double2 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 256 * u, r2 = idx & 31, c = idx >> 5;  // 32 double2 per column
      t[u] = (2 * r2 + 1 >= (c & ~15)) ? __ldcg(reinterpret_cast<const double2*>(a + (int64_t)c * lda + 2 * r2))
                                      : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 256 * u, r2 = idx & 31, c = idx >> 5;
      *reinterpret_cast<double2*>(As + c * LDA2 + 2 * r2) = t[u];
    }
  }
  if (tid == 0) badj = PB;
  __syncthreads();
  PTRACE(1);
  if (warp < NFW) {
    int first = -1;
#pragma unroll 1
    for (int K = 0; K < nstrips; ++K) {
      const int b = factor_strip(K, As, dv, rs, colbuf);
      if (first < 0 && b >= 0) first = 16 * K + b;
      PTRACE(2 + K);
      named_arrive(1 + K, 256);
    }
    if (tid == 0 && first >= 0) badj = first;
    hook.after_strips();
  } else {
    constexpr int NH = 256 - 32 * NFW;  // helper threads
#pragma unroll 1
    for (int K = 0; K < 4; ++K) {
      const int k0 = 16 * K;
      if (warp == 7) hook(K);
      if (K >= nstrips) {  // identity padding: W row block K = identity rows, log L_ii = 0
        for (int idx = tid - 32 * NFW; idx < 16 * PB; idx += NH) {
          const int r = idx & 15, c = idx >> 4;
          W[c * PB + k0 + r] = (c == k0 + r) ? 1.0 : 0.0;
        }
        if (warp == NFW && lane < 16) lgv[k0 + lane] = 0.0;
        continue;
      }
      named_sync(1 + K, 256);  // strip K is in As
      // log-det terms of strip K on warp 4, beside T_K (warp 3) and the G products (warps 5, 6):
      // off the tail after the last strip
      if (warp == 4 && lane < 16) lgv[k0 + lane] = 0.5 * log(dv[k0 + lane]);
      if (warp == 7) {  // L strip K (columns k0..k0+15; zeros above row k0, as a dpotrf leaves them) to global memory
#pragma unroll 4
        for (int c = k0; c < k0 + 16; ++c)
          *reinterpret_cast<double2*>(a + (int64_t)c * lda + 2 * lane) =
              2 * lane >= k0 ? *reinterpret_cast<const double2*>(As + c * LDA2 + 2 * lane) : make_double2(0.0, 0.0);
      }
      if (warp == NFW && lane < 16) {  // column c = lane of T_K: t_r = (delta_rc - sum_{m<r} L_rm t_m) / L_rr
        const int c = lane;
        double acc[16], t[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = 0.0;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          t[m] = (m < c) ? 0.0 : ((m == c ? 1.0 : 0.0) - acc[m]) * rs[k0 + m];
#pragma unroll
          for (int r = m + 1; r < 16; ++r) acc[r] = fma(As[(k0 + m) * LDA2 + k0 + r], t[m], acc[r]);
        }
        double* T = Ts + K * 16 * LDT;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          T[c * LDT + r] = t[r];
          Ws[(k0 + c) * LDA2 + k0 + r] = t[r];
        }
      }
      double g[2][2][2] = {};
      // column block C of W row block K on warps 5, 6, 4 (C = 0, 1, 2): the heavy C = 0 and 1 off
      // SMSP 0, which runs factor warp 0 -- the only factor warp of strips 2 and 3
      const int C = warp == 5 ? 0 : (warp == 6 ? 1 : (warp == 4 ? 2 : -1));
      if (C >= 0 && C < K) {  // G_KC = sum_{M=C}^{K-1} L_KM W_MC
#pragma unroll 1
        for (int M = C; M < K; ++M)
          mm16(g, [=](int m, int k) { return As[(16 * M + k) * LDA2 + k0 + m]; },
               [=](int k, int n) { return Ws[(16 * C + n) * LDA2 + 16 * M + k]; });
      }
      named_sync(5, NH);  // T_K is in shared memory
      if (C >= 0 && C < K) {  // W_KC = -T_K G_KC
        const double* T = Ts + K * 16 * LDT;
        // G to shared memory first: its accumulator layout is not the B fragment layout
        acc_store(g, [=](int m, int n, double v) { Ws[(16 * C + n) * LDA2 + k0 + m] = v; });
        __syncwarp();
        double w[2][2][2] = {};
        mm16(w, [=](int m, int k) { return -T[k * LDT + m]; },
             [=](int k, int n) { return Ws[(16 * C + n) * LDA2 + k0 + k]; });
        __syncwarp();
        acc_store(w, [=](int m, int n, double v) { Ws[(16 * C + n) * LDA2 + k0 + m] = v; });
      }
      named_sync(5, NH);  // W row block K complete before the next G reads it
      // W row block K to global memory (zeros right of the diagonal block); log-det terms
      for (int idx = tid - 32 * NFW; idx < 16 * PB; idx += NH) {
        const int r = idx & 15, c = idx >> 4;
        W[c * PB + k0 + r] = (c < k0 + 16) ? Ws[c * LDA2 + k0 + r] : 0.0;
      }
    }
    if (warp == 7) hook(4);
  }
  __syncthreads();
  PTRACE(6);
  if (badj < PB) {
    if (tid == 0) *info = (int)(pivot_base + badj + 1);
    return false;
  }
  // sum log L_jj = sum log(d_j) / 2, fixed two-level tree (L and W are already stored)
  if (tid < PB) {
    double lg = lgv[tid];
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_down_sync(0xffffffffu, lg, o);
    if ((tid & 31) == 0) lred[tid >> 5] = lg;
  }
  __syncthreads();
  if (tid == 0) *slot = lred[0] + lred[1];
  PTRACE(7);
  return true;
}

