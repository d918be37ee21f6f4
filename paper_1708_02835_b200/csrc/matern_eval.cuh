// matern_eval.cuh -- the device Matern evaluator of Eq. (2): closed forms, the
// in-house K_nu (Temme series / Steed CF2, see matern.cu's header), the per-theta Chebyshev
// table lookup (K1T), the distance (Euclidean or great-circle) and the generated entry of
// the tile layout. Shared by the generator kernels (matern.cu) and the tile-task executor's
// fused generation (dag.cu); namespace exageo::mat.
#pragma once
#include <cmath>

#include "internal.h"

namespace exageo {
namespace mat {


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


}  // namespace mat
}  // namespace exageo
