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

#include "potrf64.cuh"

__global__ void __launch_bounds__(256) potrf_block_kernel(double* __restrict__ a, int64_t lda,
                                                          double* __restrict__ W, double* __restrict__ slot,
                                                          int* __restrict__ info, int64_t pivot_base, int nstrips) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // programmatic dependent launch
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (*(volatile int*)info != 0) return;
  extern __shared__ double smem_p[];
  potrf64_body(a, lda, W, slot, info, pivot_base, smem_p, NoHook(), nstrips);
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

// y_c of owned column c (z row of its local panel; only ranks whose process row holds the z
// row block call this)
__device__ __forceinline__ double zrow_value(const Layout& L, const double* ws, int64_t c) {
  const int j = (int)(c / L.nb);
  const int64_t jb = (int64_t)j * L.nb;
  return ws[L.off(j) + (c - jb) * L.ld(j) + L.lrows(j)];
}

// Stage 1: kQuadBlocks CTAs; CTA b sums y_c^2 over a contiguous range of this rank's
// columns (the owned panels' columns, in order, restricted to c < n); zero on ranks without
// the z row block.
__global__ void __launch_bounds__(512) quad_partial_kernel(Layout L, const double* __restrict__ ws,
                                                           double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t cols = L.has_z() ? (int64_t)L.owned() * L.nb : 0;
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

// NCCL + CUDA graphs: this rank's first failing pivot as an all-reduce(min) key (INT64_MAX: none).
__global__ void pivot_key_kernel(const int* __restrict__ info, int64_t* __restrict__ key) {
  const int v = *info;
  *key = v > 0 ? (int64_t)v - 1 : (int64_t)0x7fffffffffffffffLL;
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

// One CTA per owned column: its stored rows (global r >= c, r < n) into dense dst.
__global__ void read_lower_kernel(Layout L, const double* __restrict__ ws, double* __restrict__ dst, int64_t ld) {
  const int64_t c = (int64_t)L.owned_panel((int)(blockIdx.x / L.nb)) * L.nb + blockIdx.x % L.nb;
  if (c >= L.n) return;
  const int j = (int)(c / L.nb);
  const int64_t jb = (int64_t)j * L.nb;
  const double* col = ws + L.off(j) + (c - jb) * L.ld(j);
  const int64_t R = L.lrows(j);
  for (int64_t lr = threadIdx.x; lr < R; lr += blockDim.x) {
    const int64_t r = L.grow(j, lr);
    if (r >= c && r < L.n) dst[c * ld + r] = col[lr];
  }
}

__global__ void read_zrow_kernel(Layout L, const double* __restrict__ ws, double* __restrict__ dst) {
  if (!L.has_z()) return;
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
    const int64_t lr = L.lrow(j, r);
    if (lr < 0) continue;
    const int64_t jb = (int64_t)j * L.nb;
    out[i] = ws[L.off(j) + (c - jb) * L.ld(j) + lr];
  }
}

// TRMV stage 1: part[m][r] = sum_{c in owned panel m, c <= r, c < n} L_rc e_c for the global
// rows r stored here (grid: local row blocks x owned panels); the other rows of part stay as
// the caller zeroed them.
__global__ void __launch_bounds__(256) trmv_partial_kernel(Layout L, const double* __restrict__ ws,
                                                           const double* __restrict__ e, double* __restrict__ part) {
  const int m = blockIdx.y;
  const int j = L.owned_panel(m);
  const int64_t jb = (int64_t)j * L.nb;
  const int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= L.lrows(j)) return;
  const int64_t r = L.grow(j, lr);
  const double* Pp = ws + L.off(j) + lr;
  const int64_t ld = L.ld(j);
  const int64_t cend = (r - jb + 1) < L.nb ? (r - jb + 1) : L.nb;
  double acc = 0.0;
  for (int64_t cc = 0; cc < cend; ++cc) {
    const int64_t c = jb + cc;
    if (c < L.n) acc += Pp[cc * ld] * e[c];
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

#ifdef EXAGEO_POTRF_TRACE
cudaError_t potrf_trace_read(long long* out) { return cudaMemcpyFromSymbol(out, g_potrf_trace, 64 * sizeof(long long)); }
#endif

cudaError_t potrf_init() {
  return cudaFuncSetAttribute(potrf_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotrfSmem);
}

void launch_potrf_block(double* a, int64_t lda, double* W, double* slot, int* info, int64_t pivot_base,
                        cudaStream_t s, bool pdl, int ncols) {
  const int nstrips = ncols >= PB ? 4 : (ncols + 15) / 16;
  if (!pdl) {
    potrf_block_kernel<<<1, 256, kPotrfSmem, s>>>(a, lda, W, slot, info, pivot_base, nstrips);
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
  cudaLaunchKernelEx(&cfg, potrf_block_kernel, a, lda, W, slot, info, pivot_base, nstrips);
}

void launch_local_partials(const Layout& L, const double* ws, const double* slots, int nslots, double* scratch,
                           double* out2, cudaStream_t s) {
  quad_partial_kernel<<<kQuadBlocks, 512, 0, s>>>(L, ws, scratch);
  local_partials_kernel<<<1, 1024, 0, s>>>(slots, nslots, scratch, kQuadBlocks, out2);
}

void launch_pivot_key(const int* info, int64_t* key, cudaStream_t s) { pivot_key_kernel<<<1, 1, 0, s>>>(info, key); }

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
  cudaMemsetAsync(part, 0, sizeof(double) * (size_t)L.owned() * (size_t)L.N, s);
  dim3 g1((unsigned)((L.lrows(L.owned_panel(0)) + 255) / 256), (unsigned)L.owned());
  trmv_partial_kernel<<<g1, 256, 0, s>>>(L, ws, e, part);
}

void launch_trmv_sum(int64_t n, int64_t N, const double* part, int nparts, double* z, cudaStream_t s) {
  trmv_sum_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, N, part, nparts, z);
}

}  // namespace exageo
