// trsv.cu -- K5^T: blocked backward triangular solve L^T w = y over the lower panels
// (the second half of Alg. 3's dposv, P:720-721 / P:738, R19). The forward half
// y = L^{-1} z2 is already in the z row of every panel (fused into the factorization).
//
// Panel by panel from the last (j = T-1 .. 0), in two launches per panel:
//   gemv_t:     part[s][c] = sum over rows r in chunk s of the panel's sub-diagonal rows
//               (global rows (j+1) nb .. N-1) of L_rc w_r         (reads the panel once,
//               coalesced down columns; HBM-bound)
//   tile_solve: rhs_c = y_c - sum_s part[s][c];  L_jj^T w_j = rhs  (one CTA, 64-column
//               blocks from the last: shared-memory substitution with the 64 x 64 diagonal
//               block, then the rank-64 update of the remaining right-hand side)
// Fixed chunking and summation order: bitwise reproducible.
#include "internal.h"

namespace exageo {

namespace {

constexpr int kColsPerCta = 8;  // columns of the panel per CTA in gemv_t
constexpr int kRowChunk = 4096;

__global__ void __launch_bounds__(256) gemv_t_kernel(Layout L, int j, const double* __restrict__ P, int64_t ld,
                                                     int64_t lr0, int64_t rows, const double* __restrict__ w,
                                                     double* __restrict__ part) {
  // P: local panel j (column-major, ld); local rows lr0 .. lr0 + rows - 1 (square rows below
  // the diagonal tile), the local row lr being global row L.grow(j, lr); w is indexed by
  // global row.
  __shared__ double red[8][kColsPerCta];
  const int nb = L.nb;
  const int c0 = blockIdx.x * kColsPerCta;
  const int64_t r_lo = (int64_t)blockIdx.y * kRowChunk;
  const int64_t r_hi = (r_lo + kRowChunk) < rows ? (r_lo + kRowChunk) : rows;
  double acc[kColsPerCta];
#pragma unroll
  for (int q = 0; q < kColsPerCta; ++q) acc[q] = 0.0;
#pragma unroll 4  // several rows' loads in flight per thread (the loop is HBM-latency bound)
  for (int64_t r = r_lo + threadIdx.x; r < r_hi; r += blockDim.x) {
    const double wr = w[L.grow(j, lr0 + r)];
#pragma unroll
    for (int q = 0; q < kColsPerCta; ++q) acc[q] += P[(int64_t)(c0 + q) * ld + lr0 + r] * wr;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kColsPerCta; ++q) {
    double v = acc[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < kColsPerCta) {
    double v = 0.0;
    for (int wq = 0; wq < 8; ++wq) v += red[wq][threadIdx.x];
    part[(int64_t)blockIdx.y * nb + c0 + threadIdx.x] = v;
  }
}

// out[c] = sum_s part[s][c], fixed order (one partial vector per rank for the 2-D solve).
__global__ void sum_parts_kernel(const double* __restrict__ part, int nparts, int nb, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nb) return;
  double v = 0.0;
  for (int s = 0; s < nparts; ++s) v += part[(int64_t)s * nb + c];
  out[c] = v;
}

// One CTA of min(nb, 1024) threads: thread c owns columns c, c + blockDim.x, ... of the
// diagonal tile. rhs_c = y_c - sum_s part[s][c]; y from yv (nb entries) when given, else
// from the panel's z row (local row zrow).
__global__ void tile_solve_kernel(const double* __restrict__ P, int64_t ld, int nb, int64_t zrow,
                                  const double* __restrict__ yv, const double* __restrict__ part, int nparts,
                                  double* __restrict__ wj) {
  extern __shared__ double sh[];
  double* rhs = sh;            // nb
  double* blk = sh + nb;       // 64 x 65 diagonal block (column-major)
  const int nt = blockDim.x;
  for (int c = threadIdx.x; c < nb; c += nt) {
    double v = yv ? yv[c] : P[(int64_t)c * ld + zrow];  // y_c
    for (int s = 0; s < nparts; ++s) v -= part[(int64_t)s * nb + c];
    rhs[c] = v;
  }
  __syncthreads();
  for (int b = nb / 64 - 1; b >= 0; --b) {
    const int b0 = b * 64;
    // load the 64 x 64 diagonal block L[b0.., b0..]
    for (int idx = threadIdx.x; idx < 64 * 64; idx += nt) {
      const int r = idx % 64, cc = idx / 64;
      blk[cc * 65 + r] = P[(int64_t)(b0 + cc) * ld + b0 + r];
    }
    __syncthreads();
    // backward substitution: w_k = (rhs_k - sum_{r > k} L_rk w_r) / L_kk, right-looking
    for (int k = 63; k >= 0; --k) {
      if (threadIdx.x == 0) rhs[b0 + k] /= blk[k * 65 + k];
      __syncthreads();
      const double wk = rhs[b0 + k];
      const int c = threadIdx.x;
      if (c < k) rhs[b0 + c] -= blk[c * 65 + k] * wk;  // L_{k, c} = row k of column c
      __syncthreads();
    }
    // rhs_c -= sum_{r in block b} L_rc w_r for the columns c < b0 (rows of block b, column c)
    for (int c = threadIdx.x; c < b0; c += nt) {
      double acc = 0.0;
      const double* col = P + (int64_t)c * ld + b0;
      for (int r = 0; r < 64; ++r) acc += col[r] * rhs[b0 + r];
      rhs[c] -= acc;
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < nb; c += nt) wj[c] = rhs[c];
}

// ---- multi-right-hand-side forward solve L V = S for the kriging variance (exageo_predict_var)
// Diagonal block: one CTA per kRhs right-hand sides (columns of S, nb threads: thread r owns
// row r of each), right-looking substitution with the panel's nb x nb diagonal tile (lower
// part only; its upper part holds unused covariance values). Each loaded L_rk serves kRhs
// columns; the next column's entry is loaded one step ahead (L2 latency off the chain).
constexpr int kRhs = 4;
__global__ void diag_solve_cols_kernel(const double* __restrict__ P, int64_t ld, int nb, double* __restrict__ S,
                                       int64_t lds, int cols) {
  extern __shared__ double sv[];  // [kRhs][nb]
  const int r = threadIdx.x, c0 = blockIdx.x * kRhs;
  double v[kRhs];
#pragma unroll
  for (int q = 0; q < kRhs; ++q) v[q] = (c0 + q < cols) ? S[(int64_t)(c0 + q) * lds + r] : 0.0;
  double lk = P[r];
  for (int k = 0; k < nb; ++k) {
    const double lnext = (k + 1 < nb) ? P[(int64_t)(k + 1) * ld + r] : 0.0;
    if (r == k) {
#pragma unroll
      for (int q = 0; q < kRhs; ++q) {
        v[q] = v[q] / lk;
        sv[q * nb + k] = v[q];
      }
    }
    __syncthreads();
    if (r > k) {
#pragma unroll
      for (int q = 0; q < kRhs; ++q) v[q] -= lk * sv[q * nb + k];
    }
    lk = lnext;
  }
#pragma unroll
  for (int q = 0; q < kRhs; ++q)
    if (c0 + q < cols) S[(int64_t)(c0 + q) * lds + r] = v[q];
}

// Bt (cols x rows, ld cols) = S (rows x cols, ld lds)^T, 32 x 32 tiles through shared memory.
__global__ void transpose_kernel(const double* __restrict__ S, int64_t lds, int rows, int cols,
                                 double* __restrict__ Bt) {
  __shared__ double t[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + threadIdx.x, c = c0 + i;
    t[i][threadIdx.x] = (r < rows && c < cols) ? S[(int64_t)c * lds + r] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + threadIdx.x, r = r0 + i;
    if (r < rows && c < cols) Bt[(int64_t)r * cols + c] = t[threadIdx.x][i];
  }
}

// var_c = theta1 - sum_{k < n} V_kc^2 (fixed-order block tree per column).
__global__ void __launch_bounds__(256) column_var_kernel(const double* __restrict__ V, int64_t ldv, int64_t n,
                                                         double theta1, double* __restrict__ var) {
  __shared__ double red[8];
  const double* col = V + (int64_t)blockIdx.x * ldv;
  double a = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) a += col[k] * col[k];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int q = 0; q < 8; ++q) s2 += red[q];
    var[blockIdx.x] = theta1 - s2;
  }
}

// dst (rows x cols, ld ldd) += src (rows x cols, ld lds)
__global__ void add_block_kernel(double* __restrict__ dst, int64_t ldd, const double* __restrict__ src, int64_t lds,
                                 int rows, int cols) {
  const int c = blockIdx.y;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    dst[(int64_t)c * ldd + r] += src[(int64_t)c * lds + r];
}

// acc[c] += sum_{r < rows} V_rc^2 (one CTA per column, fixed-order tree)
__global__ void __launch_bounds__(256) colsq_accum_kernel(const double* __restrict__ V, int64_t ldv, int rows,
                                                          double* __restrict__ acc) {
  __shared__ double red[8];
  const double* col = V + (int64_t)blockIdx.x * ldv;
  double a = 0.0;
  for (int k = threadIdx.x; k < rows; k += blockDim.x) a += col[k] * col[k];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int q = 0; q < 8; ++q) s2 += red[q];
    acc[blockIdx.x] += s2;
  }
}

__global__ void var_from_acc_kernel(const double* __restrict__ acc, int cols, double theta1, double* __restrict__ var) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < cols) var[c] = theta1 - acc[c];
}

}  // namespace

// tile_solve_kernel keeps the nb-entry right-hand side and a 64 x 65 block in shared memory:
// above 48 KB (nb > 1984, e.g. the automatic nb = 2048 of n >= 56k) it needs the opt-in limit
// (200 KB: nb up to 21k).
cudaError_t trsv_init() {
  cudaError_t e = cudaFuncSetAttribute(tile_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(diag_solve_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kRhs * 1024 * sizeof(double)));
}

void launch_add_block(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  add_block_kernel<<<dim3((rows + 255) / 256, cols), 256, 0, s>>>(dst, ldd, src, lds, rows, cols);
}

void launch_colsq_accum(const double* V, int64_t ldv, int rows, int cols, double* acc, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  colsq_accum_kernel<<<cols, 256, 0, s>>>(V, ldv, rows, acc);
}

void launch_var_from_acc(const double* acc, int cols, double theta1, double* var, cudaStream_t s) {
  var_from_acc_kernel<<<(cols + 255) / 256, 256, 0, s>>>(acc, cols, theta1, var);
}

void launch_diag_solve_cols(const double* P, int64_t ld, int nb, double* S, int64_t lds, int cols, cudaStream_t s) {
  diag_solve_cols_kernel<<<(cols + kRhs - 1) / kRhs, nb, kRhs * nb * sizeof(double), s>>>(P, ld, nb, S, lds, cols);
}

void launch_transpose(const double* S, int64_t lds, int rows, int cols, double* Bt, cudaStream_t s) {
  dim3 grid((rows + 31) / 32, (cols + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(S, lds, rows, cols, Bt);
}

void launch_column_var(const double* V, int64_t ldv, int64_t n, int cols, double theta1, double* var,
                       cudaStream_t s) {
  column_var_kernel<<<cols, 256, 0, s>>>(V, ldv, n, theta1, var);
}

int trsv_chunks(int64_t rows) { return rows > 0 ? (int)((rows + kRowChunk - 1) / kRowChunk) : 0; }

void launch_backsolve_panel(const double* P, int64_t ld, int nb, int64_t row_after, int64_t rows,
                            const double* w, double* wj, double* part, cudaStream_t s) {
  Layout L;  // 1-D panel: local row lr of panel j = row_after / nb - 1 is global row j nb + lr
  L.nb = nb;
  const int j = (int)(row_after / nb) - 1;
  const int nparts = trsv_chunks(rows);
  if (nparts > 0) {
    dim3 grid(nb / kColsPerCta, nparts);
    gemv_t_kernel<<<grid, 256, 0, s>>>(L, j, P, ld, nb, rows, w, part);
  }
  const int64_t zrow = ld - ZR;  // local row of the z row
  const int nt = nb < 1024 ? nb : 1024;
  tile_solve_kernel<<<1, nt, (nb + 64 * 65) * sizeof(double), s>>>(P, ld, nb, zrow, nullptr, part, nparts, wj);
}

void launch_backsolve_partial(const Layout& L, int j, const double* P, int64_t ld, int64_t lr0, int64_t rows,
                              const double* w, double* part, double* out, cudaStream_t s) {
  const int nparts = trsv_chunks(rows);
  if (nparts > 0) {
    dim3 grid(L.nb / kColsPerCta, nparts);
    gemv_t_kernel<<<grid, 256, 0, s>>>(L, j, P, ld, lr0, rows, w, part);
    sum_parts_kernel<<<(L.nb + 255) / 256, 256, 0, s>>>(part, nparts, L.nb, out);
  } else {
    cudaMemsetAsync(out, 0, sizeof(double) * L.nb, s);
  }
}

void launch_tile_solve(const double* P, int64_t ld, int nb, const double* yj, const double* parts, int nparts,
                       double* wj, cudaStream_t s) {
  const int nt = nb < 1024 ? nb : 1024;
  tile_solve_kernel<<<1, nt, (nb + 64 * 65) * sizeof(double), s>>>(P, ld, nb, 0, yj, parts, nparts, wj);
}

}  // namespace exageo
