// potrf_reduce.cu -- K2 (diagonal-block POTRF + inverse + log-det partial),
// K6 (deterministic log-det / dot reductions and l(theta)), read-back and TRMV.
//
//  * potrf_block: the PB x PB (PB = 64) diagonal block of the current panel is
//    factored in shared memory by the right-looking unblocked algorithm
//    (L_jj = sqrt(a_jj); l_ij = a_ij / L_jj; a_ic -= l_ij l_cj), the paper's
//    dpotrf at tile granularity (Alg. 2 l.3). The same CTA forms
//    W = L^{-1} so that the panel TRSM becomes a DMMA multiplication, and the
//    partial log-determinant sum_i log L_ii (R5). The first
//    non-positive pivot is recorded as a global index (R14); every later
//    kernel reads the info word and exits.
//  * reductions: per rank, logdet/2 = sum of its panels' partials and quad = sum y_c^2
//    over its columns of the z row (y = L^{-1} z, Alg. 2 l.4-6, R6-R7); the ranks'
//    pairs are combined (after an all-reduce when multi-GPU) into
//    l = -quad/2 - logdet/2 - n/2 log 2 pi (Alg. 2 l.7). Fixed-order trees:
//    bitwise reproducible for a fixed rank count.
#include <cmath>

#include "internal.h"

namespace exageo {

namespace {

constexpr int LDS_P = PB + 1;

// 64 TPR threads: thread t owns row r = t / TPR and the NS = 64 / TPR slots
// c = (t % TPR) + TPR s of it, in registers. Slot c holds a_rc (the Schur complement,
// unscaled) while c > j and, from step c on, w_rc of W = L^{-1} (unscaled). Step j: the
// owners of row j publish W's row j to shared memory (column j of A was published at step
// j-1), one barrier, then every row r > j applies, with d_j = a_jj and f = a_rj / d_j,
//   c >  j: a_rc -= f a_cj        (right-looking Cholesky; L_jj = sqrt d_j, L_rj = a_rj / L_jj)
//   c <= j: w_rc -= f w_jc        (right-looking L W = I;  W_jc = w_jc / L_jj, w_jj = 1)
// and the owner of column j+1 publishes a_r,j+1. Scaling is deferred to the write-out.
// colA and rowW share one array (rowW at offset PB * LDS_P) so the per-slot source is an
// index select, not a pointer select.
template <int TPR>
__global__ void __launch_bounds__(64 * TPR) potrf_block_kernel(double* __restrict__ a, int64_t lda,
                                                               double* __restrict__ W, double* __restrict__ slot,
                                                               int* __restrict__ info, int64_t pivot_base) {
  constexpr int NS = PB / TPR;
  constexpr int RPW = 32 / TPR;  // rows per warp
  constexpr int WOFF = PB * LDS_P;
  if (*(volatile int*)info != 0) return;
  extern __shared__ double smem_p[];
  double* colA = smem_p;         // colA[j * LDS_P + r] = a_rj at step j (unscaled)
  double* rowW = smem_p + WOFF;  // rowW[j * LDS_P + c] = w_jc at step j (unscaled)
  const int tid = threadIdx.x;
  const int r = tid / TPR, q = tid % TPR;
  double v[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int c = q + TPR * s;
    v[s] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
  }
  if (q == 0) colA[r] = v[0];  // column 0
  int bad = -1;
  for (int j = 0; j < PB; ++j) {
    if (r == j) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int c = q + TPR * s;
        rowW[j * LDS_P + c] = (c < j) ? v[s] : (c == j ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    const double d = colA[j * LDS_P + j];
    if (!(d > 0.0)) {
      bad = j;
      break;
    }
    if ((tid >> 5) * RPW + RPW - 1 > j) {  // warp-uniform: this warp holds rows > j
      // Branch-free over the slots (the lanes of a row own different columns, so any
      // per-slot branch would diverge): select the source row/column, predicate the update.
      const bool row_active = r > j;
      const double f = colA[j * LDS_P + r] * __drcp_rn(d);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int c = q + TPR * s;
        const bool isw = c <= j;  // W part (c == j: reset a_rj to w_rj = 0 - f w_jj, w_jj = 1)
        const double src = smem_p[j * LDS_P + c + (isw ? WOFF : 0)];
        const double base = (c == j) ? 0.0 : v[s];
        const double nv = base - f * src;
        const bool act = row_active && (isw || c <= r);
        v[s] = act ? nv : v[s];
        if (act && c == j + 1) colA[(j + 1) * LDS_P + r] = nv;
      }
    }
  }
  if (bad >= 0) {
    if (tid == 0) *info = (int)(pivot_base + bad + 1);
    return;
  }
  __syncthreads();
  // L_jj = sqrt(d_j) and 1 / L_jj once per column; sum log L_jj = sum log(d_j) / 2 by a
  // fixed two-level tree (warps 0-1, then lane 0 of warp 0)
  __shared__ double lj[PB], ilj[PB], lred[2];
  if (tid < PB) {
    const double dj = colA[tid * LDS_P + tid];
    lj[tid] = sqrt(dj);
    ilj[tid] = 1.0 / lj[tid];
    double lg = 0.5 * log(dj);
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_down_sync(0xffffffffu, lg, o);
    if ((tid & 31) == 0) lred[tid >> 5] = lg;
  }
  __syncthreads();
  if (tid == 0) *slot = lred[0] + lred[1];
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx % PB, c = idx / PB;
    a[(int64_t)c * lda + rr] = (rr > c) ? colA[c * LDS_P + rr] * ilj[c] : (rr == c ? lj[c] : 0.0);
    W[c * PB + rr] = (rr >= c) ? rowW[rr * LDS_P + c] * ilj[rr] : 0.0;
  }
}

// Fixed-shape block sum (blockDim.x a multiple of 32): deterministic tree.
__device__ double block_sum(double v, double* red) {
  const int tid = threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (tid < 32) {
    r = (tid < (int)(blockDim.x >> 5)) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// y_c of owned column c (z row of its panel)
__device__ __forceinline__ double zrow_value(const Layout& L, const double* ws, int64_t c) {
  const int j = (int)(c / L.nb);
  const int64_t jb = (int64_t)j * L.nb;
  return ws[L.off(j) + (c - jb) * L.ld(j) + (L.N - jb)];
}

// Stage 1: kQuadBlocks CTAs; CTA b sums y_c^2 over a contiguous range of this rank's
// columns (the owned panels' columns, in order, restricted to c < n).
__global__ void __launch_bounds__(512) quad_partial_kernel(Layout L, const double* __restrict__ ws,
                                                           double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t cols = (int64_t)L.owned() * L.nb;
  const int64_t per = (cols + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = (lo + per) < cols ? (lo + per) : cols;
  double v = 0.0;
  for (int64_t idx = lo + threadIdx.x; idx < hi; idx += blockDim.x) {
    const int64_t c = (int64_t)L.owned_panel((int)(idx / L.nb)) * L.nb + idx % L.nb;
    if (c < L.n) {
      const double yv = zrow_value(L, ws, c);
      v += yv * yv;
    }
  }
  const double s = block_sum(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Stage 2 (one CTA): out2 = {sum of log-det slots, sum of the quad partials}, fixed order.
__global__ void __launch_bounds__(1024) local_partials_kernel(const double* __restrict__ slots, int nslots,
                                                              const double* __restrict__ part, int nparts,
                                                              double* __restrict__ out2) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) a += slots[i];
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) b += part[i];
  const double sa = block_sum(a, red);
  const double sb = block_sum(b, red);
  if (threadIdx.x == 0) {
    out2[0] = sa;
    out2[1] = sb;
  }
}

// Combine the ranks' pairs in rank order: logdet = 2 sum(slots), quad = sum(y^2),
// l = -quad/2 - logdet/2 - (n/2) log 2 pi (Alg. 2 l.7).
__global__ void combine_kernel(const double* __restrict__ parts, int nparts, int64_t n, double* __restrict__ out3) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nparts; ++i) {
    a += parts[2 * i];
    b += parts[2 * i + 1];
  }
  const double logdet = 2.0 * a;
  const double log2pi = 1.8378770664093454835606594728112;
  out3[0] = -0.5 * b - 0.5 * logdet - 0.5 * (double)n * log2pi;
  out3[1] = logdet;
  out3[2] = b;
}

// One CTA per owned column.
__global__ void read_lower_kernel(Layout L, const double* __restrict__ ws, double* __restrict__ dst, int64_t ld) {
  const int64_t c = (int64_t)L.owned_panel((int)(blockIdx.x / L.nb)) * L.nb + blockIdx.x % L.nb;
  if (c >= L.n) return;
  const int j = (int)(c / L.nb);
  const int64_t jb = (int64_t)j * L.nb;
  const double* col = ws + L.off(j) + (c - jb) * L.ld(j) - jb;  // index by global row
  for (int64_t r = c + threadIdx.x; r < L.n; r += blockDim.x) dst[c * ld + r] = col[r];
}

__global__ void read_zrow_kernel(Layout L, const double* __restrict__ ws, double* __restrict__ dst) {
  const int64_t cols = (int64_t)L.owned() * L.nb;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (int64_t)L.owned_panel((int)(idx / L.nb)) * L.nb + idx % L.nb;
    if (c < L.n) dst[c] = zrow_value(L, ws, c);
  }
}

__global__ void read_entries_kernel(Layout L, const double* __restrict__ ws, int64_t count,
                                    const int64_t* __restrict__ rc, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rc[i], c = rc[count + i];
    const int j = (int)(c / L.nb);
    if (!L.owns(j)) continue;
    const int64_t jb = (int64_t)j * L.nb;
    out[i] = ws[L.off(j) + (c - jb) * L.ld(j) + (r - jb)];
  }
}

// TRMV stage 1: part[m][r] = sum_{c in owned panel m, c <= r, c < n} L_rc e_c  (grid: row blocks x owned panels).
__global__ void __launch_bounds__(256) trmv_partial_kernel(Layout L, const double* __restrict__ ws,
                                                           const double* __restrict__ e, double* __restrict__ part) {
  const int m = blockIdx.y;
  const int j = L.owned_panel(m);
  const int64_t jb = (int64_t)j * L.nb;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= L.N) return;
  double acc = 0.0;
  if (r >= jb) {
    const double* P = ws + L.off(j) + (r - jb);
    const int64_t ld = L.ld(j);
    const int64_t cend = (r - jb + 1) < L.nb ? (r - jb + 1) : L.nb;
    for (int64_t cc = 0; cc < cend; ++cc) {
      const int64_t c = jb + cc;
      if (c < L.n) acc += P[cc * ld] * e[c];
    }
  }
  part[(int64_t)m * L.N + r] = acc;
}

__global__ void trmv_sum_kernel(int64_t n, int64_t N, const double* __restrict__ part, int nparts,
                                double* __restrict__ z) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double acc = 0.0;
  for (int j = 0; j < nparts; ++j) acc += part[(int64_t)j * N + r];
  z[r] = acc;
}

}  // namespace

constexpr int kPotrfSmem = 2 * PB * LDS_P * (int)sizeof(double);
#ifndef EXAGEO_POTRF_TPR
#define EXAGEO_POTRF_TPR 16
#endif
constexpr int kPotrfTpr = EXAGEO_POTRF_TPR;  // threads per row of the 64 x 64 block

cudaError_t potrf_init() {
  return cudaFuncSetAttribute(potrf_block_kernel<kPotrfTpr>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kPotrfSmem);
}

// (Measured alternatives on B200: a 4 x 4-blocked variant with a warp-serial 16 x 16
// diagonal factorization, 68 us; a pair-step variant eliminating two columns per barrier
// with a 2 x 2 pivot block, 27 us but it loses exact-zero pivot detection for duplicate
// sites; this kernel: 31 us.)
void launch_potrf_block(double* a, int64_t lda, double* W, double* slot, int* info, int64_t pivot_base,
                        cudaStream_t s) {
  potrf_block_kernel<kPotrfTpr><<<1, 64 * kPotrfTpr, kPotrfSmem, s>>>(a, lda, W, slot, info, pivot_base);
}

void launch_local_partials(const Layout& L, const double* ws, const double* slots, int nslots, double* scratch,
                           double* out2, cudaStream_t s) {
  quad_partial_kernel<<<kQuadBlocks, 512, 0, s>>>(L, ws, scratch);
  local_partials_kernel<<<1, 1024, 0, s>>>(slots, nslots, scratch, kQuadBlocks, out2);
}

void launch_combine(const double* parts, int nparts, int64_t n, double* out3, cudaStream_t s) {
  combine_kernel<<<1, 32, 0, s>>>(parts, nparts, n, out3);
}

void launch_read_lower(const Layout& L, const double* ws, double* dst, int64_t ld, cudaStream_t s) {
  if (L.owned() == 0) return;
  read_lower_kernel<<<(unsigned)(L.owned() * L.nb), 256, 0, s>>>(L, ws, dst, ld);
}

void launch_read_zrow(const Layout& L, const double* ws, double* dst, cudaStream_t s) {
  read_zrow_kernel<<<128, 256, 0, s>>>(L, ws, dst);
}

void launch_read_entries(const Layout& L, const double* ws, int64_t count, const int64_t* rc, double* out,
                         cudaStream_t s) {
  int g = (int)((count + 255) / 256);
  if (g > 1024) g = 1024;
  if (g < 1) g = 1;
  read_entries_kernel<<<g, 256, 0, s>>>(L, ws, count, rc, out);
}

void launch_trmv_partial(const Layout& L, const double* ws, const double* e, double* part, cudaStream_t s) {
  if (L.owned() == 0) return;
  dim3 g1((unsigned)((L.N + 255) / 256), (unsigned)L.owned());
  trmv_partial_kernel<<<g1, 256, 0, s>>>(L, ws, e, part);
}

void launch_trmv_sum(int64_t n, int64_t N, const double* part, int nparts, double* z, cudaStream_t s) {
  trmv_sum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, N, part, nparts, z);
}

}  // namespace exageo
