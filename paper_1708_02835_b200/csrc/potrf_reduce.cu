// potrf_reduce.cu -- K2 (diagonal-block POTRF + inverse + log-det partial),
// K6 (deterministic log-det / dot reductions and l(theta)), read-back and TRMV.
//
//  * potrf_block: the PB x PB (PB = 64) diagonal block of the current panel is
//    factored by the right-looking unblocked algorithm with the entries in
//    registers (L_jj = sqrt(a_jj); l_ij = a_ij / L_jj; a_ic -= l_ij l_cj), the
//    paper's dpotrf at tile granularity (Alg. 2 l.3). The same CTA then
//    forms W = L^{-1} so that the panel TRSM becomes a DMMA multiplication, and
//    the partial log-determinant sum_i log L_ii (R5). The first
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

constexpr int LDS_P = PB + 1;  // odd stride: conflict-free column access

// c (8 x 8, two per lane) += a (8 x 4 row fragment) * b (4 x 8 column fragment), FP64 DMMA
__device__ __forceinline__ void dmma64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
constexpr int LDS_A = PB + 2;  // even stride: 16-byte aligned double2 rows of colA

// 256 threads as a 16 x 16 grid: thread (tr, tc) holds a_rc for rows r = tr + 16 i and
// columns c = 4 tc + k (i, k < 4) in registers. Step j (right-looking, deferred scaling):
// d_j = a_jj, f_r = a_rj / d_j (reciprocal-multiply, as the paper's dpotrf), a_rc -= f_r a_cj
// for every held entry (rows r <= j get f = 0; entries above the diagonal take finite garbage
// that is never read), then the owner of column j+1 publishes it to shared memory -- one
// barrier per pivot. The j loop is unrolled by 4 so the register slot of column j+1 is a
// compile-time index (no select chains on the pivot chain). W = L^{-1} is formed after the
// factorization: 16 x 16 diagonal blocks by per-lane substitution, the off-diagonal blocks
// W_IJ = -W_II sum_K L~_IK W_KJ by distance (tools/potrf_trace.cu: 24.6 us vs 32.7 us for
// the previous 16-threads-per-row kernel that carried W through the pivot loop; the factor
// L is bitwise the same).
constexpr int kPotrfSmemDoubles = PB * LDS_A + PB * LDS_P + 3 * 256 + PB * LDS_P;

__global__ void __launch_bounds__(256) potrf_block_kernel(double* __restrict__ a, int64_t lda,
                                                          double* __restrict__ W, double* __restrict__ slot,
                                                          int* __restrict__ info, int64_t pivot_base) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // programmatic dependent launch
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (*(volatile int*)info != 0) return;
  extern __shared__ double smem_p[];
  double* colA = smem_p;             // colA[c * LDS_A + r] = a_rc at step c (unscaled)
  double* Wt = colA + PB * LDS_A;    // Wt[c * LDS_P + r] = w~_rc, w~ = L~^{-1} (unit lower)
  double* Xs = Wt + PB * LDS_P;      // 3 x 16 x 16 off-diagonal products
  double* Ls = Xs + 3 * 256;         // Ls[c * LDS_P + r] = L~_rc = a_rc / d_c (r > c)
  __shared__ double rdv[PB], ilj[PB], lj[PB], lred[2];
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = tr + 16 * i, c = 4 * tc + k;
      v[i][k] = (c <= r) ? a[(int64_t)c * lda + r] : 0.0;
    }
  if (tc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) colA[tr + 16 * i] = v[i][0];  // column 0
  }
  for (int m = 0; m < PB / 4; ++m) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 4 * m + u;
      __syncthreads();
      const double* cj = colA + j * LDS_A;
      const double rd = __drcp_rn(cj[j]);  // a bad pivot is found by the scan after the loop
      double f[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = (tr + 16 * i > j) ? cj[tr + 16 * i] * rd : 0.0;
      const double2 s01 = *reinterpret_cast<const double2*>(cj + 4 * tc);
      const double2 s23 = *reinterpret_cast<const double2*>(cj + 4 * tc + 2);
      const double src[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) v[i][k] = fma(-f[i], src[k], v[i][k]);
      const int k1 = (u + 1) & 3;  // register slot of column j + 1 (constant after unrolling)
      const int j1 = j + 1;
      if (j1 < PB && tc == (j1 >> 2)) {
#pragma unroll
        for (int i = 0; i < 4; ++i) colA[j1 * LDS_A + tr + 16 * i] = v[i][k1];
      }
    }
  }
  __syncthreads();
  // first non-positive (or NaN) pivot: d_j as used at step j; later pivots may be garbage
  __shared__ int badj;
  if (tid == 0) badj = PB;
  __syncthreads();
  if (tid < PB && !(colA[tid * LDS_A + tid] > 0.0)) atomicMin(&badj, tid);
  __syncthreads();
  if (badj < PB) {
    if (tid == 0) *info = (int)(pivot_base + badj + 1);
    return;
  }
  // L_jj = sqrt(d_j), 1 / L_jj; sum log L_jj = sum log(d_j) / 2 by a fixed two-level tree
  if (tid < PB) {
    const double dj = colA[tid * LDS_A + tid];
    rdv[tid] = __drcp_rn(dj);
    lj[tid] = sqrt(dj);
    ilj[tid] = 1.0 / lj[tid];
    double lg = 0.5 * log(dj);
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_down_sync(0xffffffffu, lg, o);
    if ((tid & 31) == 0) lred[tid >> 5] = lg;
  }
  __syncthreads();
  if (tid == 0) *slot = lred[0] + lred[1];
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx & (PB - 1), c = idx / PB;
    Ls[c * LDS_P + rr] = (rr > c) ? colA[c * LDS_A + rr] * rdv[c] : 0.0;
  }
  __syncthreads();
  {  // diagonal 16 x 16 blocks of w~ = L~^{-1}: warp I, lane c computes column c
    const int I = tid >> 5, c = tid & 31;
    if (I < 4 && c < 16) {
      const int b = 16 * I;
      double w[16];
#pragma unroll
      for (int mm = 0; mm < 16; ++mm) w[mm] = (mm == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int r = k + 1; r < 16; ++r) w[r] = fma(-Ls[(b + k) * LDS_P + b + r], w[k], w[r]);
#pragma unroll
      for (int r = 0; r < 16; ++r) Wt[(b + c) * LDS_P + b + r] = (r >= c) ? w[r] : 0.0;
    }
  }
  __syncthreads();
  {  // off-diagonal blocks by distance on the FP64 tensor cores: warp blk owns block
    // (I, J) = (blk + dist, blk): X = sum_K L~_IK w~_KJ, then w~_IJ = -w~_II X, each a
    // 16 x 16 product of 2 x 2 m8n8k4 tiles (A row fragments, B column fragments)
    const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
    double* Xw = Xs + warp * 256;  // this warp's X, column-major 16 x 16 (ld 16)
#pragma unroll 1
    for (int dist = 1; dist < 4; ++dist) {
      if (warp < 4 - dist) {
        const int bI = warp + dist, bJ = warp;
        double acc[2][2][2] = {};
#pragma unroll 1
        for (int K = bJ; K < bI; ++K) {
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            double af[2], bf[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              af[t] = Ls[(16 * K + kk + fk) * LDS_P + 16 * bI + 8 * t + fr];   // L~[m][k]
              bf[t] = Wt[(16 * bJ + 8 * t + fr) * LDS_P + 16 * K + kk + fk];   // w~[k][n]
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) dmma64(acc[mt][nt], af[mt], bf[nt]);
          }
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) Xw[(8 * nt + 2 * fk + e) * 16 + 8 * mt + fr] = acc[mt][nt][e];
        __syncwarp();
        double acc2[2][2][2] = {};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          double af[2], bf[2];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            af[t] = Wt[(16 * bI + kk + fk) * LDS_P + 16 * bI + 8 * t + fr];  // w~_II[m][k]
            bf[t] = Xw[(8 * t + fr) * 16 + kk + fk];                           // X[k][n]
          }
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) dmma64(acc2[mt][nt], af[mt], bf[nt]);
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              Wt[(16 * bJ + 8 * nt + 2 * fk + e) * LDS_P + 16 * bI + 8 * mt + fr] = -acc2[mt][nt][e];
      }
      __syncthreads();
    }
  }
  for (int idx = tid; idx < PB * PB; idx += blockDim.x) {
    const int rr = idx & (PB - 1), c = idx / PB;
    a[(int64_t)c * lda + rr] = (rr > c) ? colA[c * LDS_A + rr] * ilj[c] : (rr == c ? lj[c] : 0.0);
    W[c * PB + rr] = (rr >= c) ? Wt[c * LDS_P + rr] * ilj[rr] : 0.0;
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

constexpr int kPotrfSmem = kPotrfSmemDoubles * (int)sizeof(double);

cudaError_t potrf_init() {
  return cudaFuncSetAttribute(potrf_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotrfSmem);
}

void launch_potrf_block(double* a, int64_t lda, double* W, double* slot, int* info, int64_t pivot_base,
                        cudaStream_t s, bool pdl) {
  if (!pdl) {
    potrf_block_kernel<<<1, 256, kPotrfSmem, s>>>(a, lda, W, slot, info, pivot_base);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kPotrfSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, potrf_block_kernel, a, lda, W, slot, info, pivot_base);
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
