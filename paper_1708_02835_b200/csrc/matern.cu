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

namespace exageo {

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

// 1 / d: MUFU approximation + two Newton steps (within ~1 ulp, branch-free). The series
// and continued-fraction loops below divide 3-4 times per term; the IEEE-rounded
// division is a long branchy sequence and dominated the generator's instruction count.
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  return fma(y, fma(-d, y, 1.0), y);
}

// Temme series for K_mu(x), K_mu+1(x), 0 < x <= 2 (unscaled).
__device__ __forceinline__ void bessel_k_temme(double x, const MaternConsts& c, double& kmu, double& kmu1) {
  const double mu = c.mu;
  const double x2 = 0.5 * x;
  const double d = -log(x2);          // ln(2/x)
  const double e = mu * d;            // sigma = mu ln(2/x)
  const double sinh_e_over_e = (fabs(e) < 1e-4) ? (1.0 + e * e * (1.0 / 6.0 + e * e * (1.0 / 120.0))) : sinh(e) * rcp_nr(e);
  double f = c.pimu_sin * (c.gam1 * cosh(e) + c.gam2 * sinh_e_over_e * d);  // f_0
  const double ee = exp(e);           // (2/x)^mu
  double p = 0.5 * ee * rcp_nr(c.gampl);  // p_0 = (x/2)^-mu Gamma(1+mu) / 2
  double q = 0.5 * rcp_nr(ee * c.gammi);  // q_0 = (x/2)^mu  Gamma(1-mu) / 2
  double ck = 1.0;
  const double dd = x2 * x2;
  double sum = f, sum1 = p;
  const double mu2 = mu * mu;
  for (int i = 1; i < 200; ++i) {
    const double di = (double)i;
    f = (di * f + p + q) * rcp_nr(di * di - mu2);
    ck *= dd * rcp_nr(di);
    p *= rcp_nr(di - mu);
    q *= rcp_nr(di + mu);
    const double del = ck * f;
    sum += del;
    sum1 += ck * (p - di * f);
    if (fabs(del) < 1e-17 * fabs(sum)) break;
  }
  kmu = sum;
  kmu1 = sum1 * (2.0 * rcp_nr(x));
}

// Steed's algorithm (CF2, Temme 1975) for e^x K_mu(x), e^x K_mu+1(x), x > 2.
__device__ __forceinline__ void bessel_k_cf2_scaled(double x, double mu, double& kmu, double& kmu1) {
  const double a1 = 0.25 - mu * mu;
  double b = 2.0 * (1.0 + x);
  double d = rcp_nr(b);
  double h = d, delh = d;
  double q1 = 0.0, q2 = 1.0;
  double q = a1, c = a1, a = -a1;
  double s = 1.0 + q * delh;
  for (int i = 1; i < 500; ++i) {
    const double di = (double)i;
    a -= 2.0 * di;
    c = -a * c * rcp_nr(di + 1.0);
    const double qn = (q1 - b * q2) * rcp_nr(a);
    q1 = q2;
    q2 = qn;
    q += c * qn;
    b += 2.0;
    d = rcp_nr(b + a * d);
    delh = (b * d - 1.0) * delh;
    h += delh;
    const double dels = q * delh;
    s += dels;
    if (fabs(dels) < 1e-17 * fabs(s)) break;
  }
  h = a1 * h;
  const double rx = rcp_nr(x);
  kmu = sqrt(0.5 * kPi * rx) * rcp_nr(s);
  kmu1 = kmu * (mu + x + 0.5 - h) * rx;
}

}  // namespace

// theta1 / (2^(nu-1) Gamma(nu)) x^nu K_nu(x) for x > 0 (Eq. (2) at x = r / theta2).
__device__ __forceinline__ double matern_x(double x, const MaternConsts& c) {
  switch (c.kind) {
    case 1: return c.theta1 * exp(-x);
    case 2: return c.theta1 * (1.0 + x) * exp(-x);
    case 3: return c.theta1 * (1.0 + x + x * x * (1.0 / 3.0)) * exp(-x);
    default: break;
  }
  double k0, k1;
  const bool small = x <= 2.0;
  if (small) bessel_k_temme(x, c, k0, k1);
  else bessel_k_cf2_scaled(x, c.mu, k0, k1);
  double knu;
  if (c.nl == 0) {
    knu = k0;
  } else {
    double a = c.mu + 1.0;
    const double two_rx = 2.0 * rcp_nr(x);
    for (int i = 1; i < c.nl; ++i) {
      const double kn = k0 + (a * two_rx) * k1;
      k0 = k1;
      k1 = kn;
      a += 1.0;
    }
    knu = k1;
  }
  // x^nu K_nu(x) = exp(nu ln x) K (small x) or exp(nu ln x - x) [e^x K] (large x)
  const double lx = log(x);
  const double ex = small ? exp(c.nu * lx) : exp(c.nu * lx - x);
  return c.pref * ex * knu;
}

// ---- per-theta Chebyshev table of matern_x for general nu (K1T) -------------------------
// theta is fixed during one evaluation, so x -> C(x) is tabulated once per evaluation on
// 152 intervals -- [2^-6, 4) in quarter octaves (their width is proportional to the
// distance from the branch point x = 0 of x^nu K_nu, so the Chebyshev series converge at
// the same geometric rate on every interval) and [4, 64) in steps of 1/2 -- each by a
// degree-15 Chebyshev interpolant of the direct evaluator (coefficients decay below 1e-20
// of the value), evaluated by Clenshaw's recurrence: ~35 FP64 instructions per entry instead
// of the series/continued fraction's ~1500. Outside [2^-6, 64) the direct evaluator runs.
constexpr int kTabDeg = 16;     // Chebyshev coefficients per interval
constexpr int kTabStride = 18;  // {1 / half width, mid / half width, c_0 .. c_15}
constexpr int kTabLog = 32;     // [2^-6, 4): 8 octaves x 4
constexpr int kTabLin = 120;    // [4, 64): width 1/2
constexpr int kTabN = kTabLog + kTabLin;
constexpr double kTabX0 = 0.015625, kTabX1 = 4.0, kTabXMax = 64.0;

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

__device__ __forceinline__ double matern_tab(double x, const double* __restrict__ tab) {
  int i;
  if (x < kTabX1) {  // quarter octave of x: exponent bits + three mantissa thresholds
    const long long bits = __double_as_longlong(x);
    const int e = (int)((bits >> 52) & 0x7ff) - 1023;
    const double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
    i = 4 * (e + 6) + (m >= 1.1892071150027210667) + (m >= 1.4142135623730950488) + (m >= 1.6817928305074290861);
  } else {
    i = kTabLog + (int)((x - kTabX1) * 2.0);
  }
  const double* p = tab + i * kTabStride;
  const double t = fma(x, __ldg(p), -__ldg(p + 1));
  const double t2 = 2.0 * t;
  double b1 = 0.0, b2 = 0.0;
#pragma unroll
  for (int k = kTabDeg - 1; k >= 1; --k) {
    const double b0 = fma(t2, b1, __ldg(p + 2 + k) - b2);
    b2 = b1;
    b1 = b0;
  }
  return fma(t, b1, __ldg(p + 2) - b2);
}

// Matern covariance at distance r (Eq. (2)); C(0) = theta1 (R9). tab: the per-theta table
// (general nu) or nullptr.
__device__ __forceinline__ double matern_eval(double r, const MaternConsts& c, const double* __restrict__ tab) {
  if (r == 0.0) return c.theta1;
  const double x = r * c.inv_theta2;
  if (c.kind == 0 && tab != nullptr && x >= kTabX0 && x < kTabXMax) return matern_tab(x, tab);
  return matern_x(x, c);
}

// The same with the covariance family fixed at compile time (K1's bulk path: each
// instantiation carries only its own evaluator, so the closed forms keep a small register
// footprint and full occupancy).
template <int KIND>
__device__ __forceinline__ double matern_eval_k(double r, const MaternConsts& c, const double* __restrict__ tab) {
  if (r == 0.0) return c.theta1;
  const double x = r * c.inv_theta2;
  if constexpr (KIND == 1) return c.theta1 * exp(-x);
  if constexpr (KIND == 2) return c.theta1 * (1.0 + x) * exp(-x);
  if constexpr (KIND == 3) return c.theta1 * (1.0 + x + x * x * (1.0 / 3.0)) * exp(-x);
  if constexpr (KIND == 0) {
    if (tab != nullptr && x >= kTabX0 && x < kTabXMax) return matern_tab(x, tab);
    return matern_x(x, c);
  }
  return 0.0;
}

// Distance between s1 = (x1, y1) and s2 = (x2, y2): Euclidean (R15), or the great-circle
// distance by the haversine formula with x = longitude, y = latitude in
// degrees: d = 2 R asin(sqrt(hav(dphi) + cos(phi1) cos(phi2) hav(dlambda))), hav(a) = sin^2(a/2).
__device__ __forceinline__ double dist2d(double x1, double y1, double x2, double y2, const MaternConsts& c) {
  if (c.metric == 1) {
    constexpr double kDeg = 0.017453292519943295769;  // pi / 180
    const double p1 = y1 * kDeg, p2 = y2 * kDeg;
    const double sp = sin(0.5 * (p2 - p1)), sl = sin(0.5 * (x2 - x1) * kDeg);
    double h = sp * sp + cos(p1) * cos(p2) * sl * sl;
    h = h < 1.0 ? h : 1.0;
    return 2.0 * c.radius * asin(sqrt(h));
  }
  const double dx = x1 - x2, dy = y1 - y2;
  return sqrt(dx * dx + dy * dy);
}

// Entry (global row r, global column c) of the generated panel (slow path): identity
// padding outside n, IND-annihilated tiles, the diagonal theta1 (R9), else Eq. (2).
template <int KIND>
__device__ __forceinline__ double gen_entry(const Layout& L, const MaternConsts& mc, const double* __restrict__ x,
                                            const double* __restrict__ y, int64_t r, int64_t c, double xc,
                                            double yc, const double* __restrict__ tab) {
  if (r >= L.n || c >= L.n) return (r == c) ? 1.0 : 0.0;
  if (!L.in_super_tile(r, c)) return 0.0;  // IND: annihilated off-diagonal tile
  if (r == c) return mc.theta1;
  return matern_eval_k<KIND>(dist2d(x[r], y[r], xc, yc, mc), mc, tab);
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
