// matern.cu -- K1: Matern covariance generation (Eq. (2); Alg. 2 l.2).
//
// Device evaluator of C(r; theta) = theta1 / (2^(nu-1) Gamma(nu)) x^nu K_nu(x),
// x = r / theta2, with an in-house modified Bessel function of the second kind:
//   * nu in {1/2, 3/2, 5/2}: closed forms (P:260-262 for nu = 1/2);
//   * otherwise Temme's method: write nu = mu + nl, |mu| <= 1/2, evaluate
//     K_mu and K_mu+1 by Temme's power series (x <= 2) or by Steed's
//     continued fraction CF2 (x > 2, scaled by e^x), then recur upward
//     K_{a+1} = K_{a-1} + (2a/x) K_a, which is stable for K.
//     Sources: N. M. Temme, "On the numerical evaluation of the modified Bessel function of
//     the third kind", J. Comput. Phys. 19 (1975) 324-337 (series and CF2); the same
//     algorithm as Numerical Recipes 3rd ed. Sec. 6.6 (bessik), whose variable names
//     (gam1/gam2, p, q, delh, a1) the two routines below keep.
// Per-theta constants (prefactor, Temme's gamma_1/gamma_2, 1/Gamma(1 +- mu))
// are computed once on the host in long double (exageo::matern_consts).
//
// The generator writes the lower block-column panels of the workspace
// (internal.h), one CTA per (panel, column), coalesced double2 stores down the
// column; identity padding for rows/cols >= n; z into the z row block.
#include <cmath>

#include "internal.h"
#include "matern_eval.cuh"

namespace exageo {

using namespace mat;

// K1T: per-theta Chebyshev table (see matern_eval.cuh)
__global__ void __launch_bounds__(kTabDeg) matern_table_kernel(MaternConsts mc, double* __restrict__ tab) {
  const int i = blockIdx.x, j = threadIdx.x;
  double a, b;
  if (i < kTabLog) {
    a = exp2(-6.0 + 0.25 * i);
    b = exp2(-6.0 + 0.25 * (i + 1));
  } else {
    a = kTabX1 + 0.5 * (i - kTabLog);
    b = a + 0.5;
  }
  const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
  __shared__ double fv[kTabDeg];
  fv[j] = matern_x(mid + half * cospi((j + 0.5) / kTabDeg), mc);  // Chebyshev nodes
  __syncthreads();
  double ck = 0.0;  // c_k = (2/N) sum_j f_j cos(pi k (j + 1/2) / N), c_0 halved
  for (int jj = 0; jj < kTabDeg; ++jj) ck += fv[jj] * cospi(j * (jj + 0.5) / kTabDeg);
  ck *= (j == 0 ? 1.0 : 2.0) / kTabDeg;
  double* p = tab + i * kTabStride;
  p[2 + j] = ck;
  if (j == 0) {
    p[0] = 1.0 / half;
    p[1] = mid / half;
  }
}

constexpr int kGenCols = 8;  // columns per CTA: one (x, y) row load and index test serve 8 entries

// One CTA per (owned panel j = q + Q * blockIdx.y, columns kGenCols * blockIdx.x ..) -> walks
// the local rows of those columns, two rows per thread and step, coalesced double2 stores
// down each column. Local rows of tile rows strictly below the diagonal tile inside n (the
// bulk) take the check-free path. Pairs of local rows (lr even) never straddle a tile, so
// they are consecutive global rows (2-D layouts: internal.h grow()).
template <int KIND>
__global__ void __launch_bounds__(256) gen_panels_kernel(Layout L, double* __restrict__ ws, MaternConsts mc,
                                                         const double* __restrict__ x, const double* __restrict__ y,
                                                         const double* __restrict__ z, const double* __restrict__ tab) {
  const int j = L.owned_panel(blockIdx.y);
  const int cc0 = blockIdx.x * kGenCols;
  const int64_t jb = (int64_t)j * L.nb;
  const int64_t ld = L.ld(j);
  const int64_t R = L.lrows(j);  // square rows of this local panel (the z row block follows)
  double* col0 = ws + L.off(j) + (int64_t)cc0 * ld;
  __shared__ double xc[kGenCols], yc[kGenCols];
  if (threadIdx.x < kGenCols) {
    const int64_t c = jb + cc0 + threadIdx.x;
    xc[threadIdx.x] = c < L.n ? x[c] : 0.0;
    yc[threadIdx.x] = c < L.n ? y[c] : 0.0;
  }
  __syncthreads();
  const bool cols_in = jb + cc0 + kGenCols <= L.n;
  for (int64_t rr = 2 * (int64_t)threadIdx.x; rr < ld; rr += 2 * blockDim.x) {
    const int64_t r0 = rr < R ? L.grow(j, rr) : L.N;  // global row of the pair (z block: N)
    if (cols_in && rr < R && r0 >= jb + L.nb && r0 + 1 < L.n && L.in_super_tile(r0, jb)) {
      const double x0 = x[r0], y0 = y[r0], x1 = x[r0 + 1], y1 = y[r0 + 1];
#pragma unroll 1
      for (int k = 0; k < kGenCols; ++k) {  // rolled: one inlined copy of the evaluator
        const double v0 = matern_eval_k<KIND>(dist2d(x0, y0, xc[k], yc[k], mc), mc, tab);
        const double v1 = matern_eval_k<KIND>(dist2d(x1, y1, xc[k], yc[k], mc), mc, tab);
        *reinterpret_cast<double2*>(col0 + k * ld + rr) = make_double2(v0, v1);
      }
    } else {
#pragma unroll 1
      for (int k = 0; k < kGenCols; ++k) {
        const int64_t c = jb + cc0 + k;
        const double xck = c < L.n ? x[c] : 0.0, yck = c < L.n ? y[c] : 0.0;
        double v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t lr = rr + e;
          if (lr < R) v[e] = gen_entry<KIND>(L, mc, x, y, r0 + e, c, xck, yck, tab);
          else v[e] = (lr == R && c < L.n && z != nullptr) ? z[c] : 0.0;  // z row block
        }
        *reinterpret_cast<double2*>(col0 + k * ld + rr) = make_double2(v[0], v[1]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) matern_dense_kernel(MaternConsts mc, int64_t m, const double* __restrict__ x1,
                                                           const double* __restrict__ y1, int64_t n,
                                                           const double* __restrict__ x2,
                                                           const double* __restrict__ y2, double* __restrict__ C,
                                                           int64_t ldc, const double* __restrict__ tab) {
  const int64_t j = blockIdx.y;
  const double xj = x2[j], yj = y2[j];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    C[i + j * ldc] = matern_eval(dist2d(x1[i], y1[i], xj, yj, mc), mc, tab);
}

constexpr int kKrigeChunk = 8192;

// K8: part[chunk][i] = sum over observed j in the chunk of C(||snew_i - s_j||) w_j.
__global__ void __launch_bounds__(256) krige_partial_kernel(MaternConsts mc, int64_t m, const double* __restrict__ xn,
                                                            const double* __restrict__ yn, int64_t n,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ y,
                                                            const double* __restrict__ w, double* __restrict__ part,
                                                            const double* __restrict__ tab) {
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * kKrigeChunk;
  const int64_t j1 = (j0 + kKrigeChunk) < n ? (j0 + kKrigeChunk) : n;
  const double xi = xn[i], yi = yn[i];
  double acc = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) acc += matern_eval(dist2d(xi, yi, x[j], y[j], mc), mc, tab) * w[j];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += red[q];
    part[(int64_t)blockIdx.y * m + i] = s;
  }
}

__global__ void krige_sum_kernel(int64_t m, const double* __restrict__ part, int nchunks, double* __restrict__ znew) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * m + i];
  znew[i] = s;
}

int krige_chunks(int64_t n) { return (int)((n + kKrigeChunk - 1) / kKrigeChunk); }

int matern_table_doubles() { return kTabN * kTabStride; }
const void* matern_table_kernel_fn() { return (const void*)matern_table_kernel; }

int launch_matern_table(const MaternConsts& mc, double* tab, cudaStream_t s) {
  if (mc.kind != 0 || tab == nullptr) return 0;
  matern_table_kernel<<<kTabN, kTabDeg, 0, s>>>(mc, tab);
  return 1;
}

void launch_krige(const MaternConsts& mc, int64_t m, const double* xn, const double* yn, int64_t n, const double* x,
                  const double* y, const double* w, double* part, double* znew, double* tab, cudaStream_t s) {
  const int nch = krige_chunks(n);  // <= 65535 chunks (n < 5.3e8)
  dim3 grid((unsigned)m, (unsigned)nch);
  const double* t = launch_matern_table(mc, tab, s) ? tab : nullptr;
  krige_partial_kernel<<<grid, 256, 0, s>>>(mc, m, xn, yn, n, x, y, w, part, t);
  krige_sum_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, part, nch, znew);
}

const void* gen_panels_kernel_fn(int kind) {
  switch (kind) {
    case 1: return (const void*)gen_panels_kernel<1>;
    case 2: return (const void*)gen_panels_kernel<2>;
    case 3: return (const void*)gen_panels_kernel<3>;
    default: return (const void*)gen_panels_kernel<0>;
  }
}

void launch_gen_panels(const Layout& L, double* ws, const MaternConsts& mc, const double* x, const double* y,
                       const double* z, const double* tab, cudaStream_t s) {
  if (L.owned() == 0) return;
  dim3 grid(L.nb / kGenCols, L.owned());
  switch (mc.kind) {
    case 1: gen_panels_kernel<1><<<grid, 256, 0, s>>>(L, ws, mc, x, y, z, nullptr); break;
    case 2: gen_panels_kernel<2><<<grid, 256, 0, s>>>(L, ws, mc, x, y, z, nullptr); break;
    case 3: gen_panels_kernel<3><<<grid, 256, 0, s>>>(L, ws, mc, x, y, z, nullptr); break;
    default: gen_panels_kernel<0><<<grid, 256, 0, s>>>(L, ws, mc, x, y, z, tab); break;
  }
}

void launch_matern_dense(const MaternConsts& mc, int64_t m, const double* x1, const double* y1, int64_t n,
                         const double* x2, const double* y2, double* C, int64_t ldc, double* tab, cudaStream_t s) {
  const double* t = launch_matern_table(mc, tab, s) ? tab : nullptr;
  for (int64_t j0 = 0; j0 < n; j0 += 65535) {
    const int64_t nj = (n - j0) < 65535 ? (n - j0) : 65535;
    int gx = (int)((m + 255) / 256);
    if (gx > 64) gx = 64;
    dim3 grid(gx, (unsigned)nj);
    matern_dense_kernel<<<grid, 256, 0, s>>>(mc, m, x1, y1, nj, x2 + j0, y2 + j0, C + j0 * ldc, ldc, t);
  }
}

}  // namespace exageo
