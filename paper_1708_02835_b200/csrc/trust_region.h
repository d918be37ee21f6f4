// trust_region.h -- derivative-free bound-constrained minimisation by quadratic
// interpolation models in a trust region: the BOBYQA / UOBYQA class of methods the paper's
// optimizer belongs to (R16), simplified for the d <= 3 parameters of theta.
//
//  * The model m(s) = c + g^T s + s^T H s / 2 interpolates f at p = (d+1)(d+2)/2 points
//    (fully determined quadratic, as in UOBYQA), in coordinates s = (u - u_best) / Delta.
//  * Step: the exact minimiser of m over {|s_i| <= 1} intersected with the box (a box in
//    <= 3 dimensions: every face is enumerated, its stationary point solved, the best
//    feasible one taken -- this is exact also for indefinite H).
//  * Ratio test, radius update, and replacement of the point with the largest weighted
//    Lagrange-function value at the trial point (keeps the interpolation set poised);
//    points far outside the trust region are replaced by geometry steps.
//  * Failed evaluations (+inf, e.g. a non-positive-definite covariance) are never put in
//    the model: the radius halves.
// Host-only, no CUDA; tested on the CPU (tests/test_host_logic.py).
#pragma once
#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <vector>

namespace exageo {
namespace dfo {

inline int nbasis(int d) { return (d + 1) * (d + 2) / 2; }

// phi(s) = [1, s_1 .. s_d, s_i s_j (i <= j; squares halved)], so that the coefficients are
// [c, g, H_11, H_12, .., H_dd] of c + g^T s + s^T H s / 2.
inline void basis(int d, const double* s, double* out) {
  int k = 0;
  out[k++] = 1.0;
  for (int i = 0; i < d; ++i) out[k++] = s[i];
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) out[k++] = (i == j ? 0.5 : 1.0) * s[i] * s[j];
}

// Solve A x = b (n x n, row-major, copied) by Gaussian elimination with partial pivoting.
inline bool solve(int n, std::vector<double> A, std::vector<double>& b) {
  double scale = 0.0;
  for (double v : A) scale = std::max(scale, std::fabs(v));
  if (!(scale > 0.0)) return false;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (!(std::fabs(A[piv * n + c]) > 1e-13 * scale)) return false;
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[piv * n + k]);
      std::swap(b[c], b[piv]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      b[r] -= f * b[c];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    double v = b[c];
    for (int k = c + 1; k < n; ++k) v -= A[c * n + k] * b[k];
    b[c] = v / A[c * n + c];
  }
  return true;
}

struct Quad {
  int d = 0;
  double g[3] = {0, 0, 0};
  double H[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double value(const double* s) const {  // m(s) - c
    double v = 0.0;
    for (int i = 0; i < d; ++i) {
      v += g[i] * s[i];
      for (int j = 0; j < d; ++j) v += 0.5 * s[i] * H[i][j] * s[j];
    }
    return v;
  }
  void from_coeffs(int dd, const std::vector<double>& a) {
    d = dd;
    int k = 1;
    for (int i = 0; i < d; ++i) g[i] = a[k++];
    for (int i = 0; i < d; ++i)
      for (int j = i; j < d; ++j) H[i][j] = H[j][i] = a[k++];
  }
};

// Exact minimiser of the model over the box lo <= s <= hi (lo <= 0 <= hi), d <= 3: each
// coordinate free / at its lower / at its upper bound (3^d faces); on each face the
// stationary point of the reduced quadratic, if it is feasible.
inline void minimize_box(const Quad& m, const double* lo, const double* hi, double* best) {
  const int d = m.d;
  double bv = 0.0;  // s = 0
  for (int i = 0; i < d; ++i) best[i] = 0.0;
  int combos = 1;
  for (int i = 0; i < d; ++i) combos *= 3;
  for (int code = 0; code < combos; ++code) {
    int state[3], cc = code;
    for (int i = 0; i < d; ++i) {
      state[i] = cc % 3;
      cc /= 3;
    }
    double s[3] = {0, 0, 0};
    int fr[3], nf = 0;
    for (int i = 0; i < d; ++i) {
      if (state[i] == 1) s[i] = lo[i];
      else if (state[i] == 2) s[i] = hi[i];
      else fr[nf++] = i;
    }
    bool ok = true;
    if (nf > 0) {
      std::vector<double> A(nf * nf), r(nf);
      for (int a = 0; a < nf; ++a) {
        double v = -m.g[fr[a]];
        for (int i = 0; i < d; ++i)
          if (state[i] != 0) v -= m.H[fr[a]][i] * s[i];
        r[a] = v;
        for (int b = 0; b < nf; ++b) A[a * nf + b] = m.H[fr[a]][fr[b]];
      }
      ok = solve(nf, A, r);
      if (ok)
        for (int a = 0; a < nf; ++a) {
          s[fr[a]] = r[a];
          if (!(r[a] >= lo[fr[a]] - 1e-12 && r[a] <= hi[fr[a]] + 1e-12)) ok = false;
          s[fr[a]] = std::min(std::max(s[fr[a]], lo[fr[a]]), hi[fr[a]]);
        }
    }
    if (!ok) continue;
    const double v = m.value(s);
    if (v < bv) {
      bv = v;
      for (int i = 0; i < d; ++i) best[i] = s[i];
    }
  }
}

// Minimise fn over the box [lo, hi] (d = x0.size() <= 3) from x0, initial radius delta0,
// final radius delta_end; fn(v) evaluates (and may count / record) and returns +inf on
// failure. Returns false when the initial interpolation set could not be evaluated
// (caller falls back to another method). stop() is polled before every evaluation.
inline bool minimize(const std::function<double(std::vector<double>&)>& fn, const std::vector<double>& x0,
                     const std::vector<double>& lo, const std::vector<double>& hi, double delta0, double delta_end,
                     const std::function<bool()>& stop) {
  const int d = (int)x0.size();
  const int p = nbasis(d);
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<std::vector<double>> Y;
  std::vector<double> F;
  double delta = delta0;
  auto clampv = [&](std::vector<double> v) {
    for (int i = 0; i < d; ++i) v[i] = std::min(std::max(v[i], lo[i]), hi[i]);
    return v;
  };
  auto eval = [&](std::vector<double> v, double& fv) {
    v = clampv(v);
    if (stop()) return false;
    fv = fn(v);
    Y.push_back(v);
    F.push_back(fv);
    return true;
  };
  // ---- initial interpolation set: x0, x0 +- delta e_i, x0 + delta (sg_i e_i + sg_j e_j)
  double f0;
  if (!eval(x0, f0) || !std::isfinite(f0)) return false;
  std::vector<int> sg(d, 1);
  for (int i = 0; i < d; ++i) {
    double step[2] = {delta, -delta};
    if (x0[i] + delta > hi[i]) step[0] = -2 * delta;  // at the upper bound: go down twice
    if (x0[i] - delta < lo[i]) step[1] = 2 * delta;   // at the lower bound: go up twice
    double fv[2];
    for (int t = 0; t < 2; ++t) {
      std::vector<double> v = x0;
      double h = step[t];
      for (int tries = 0;; ++tries) {
        v = x0;
        v[i] += h;
        if (!eval(v, fv[t])) return false;
        if (std::isfinite(fv[t]) || tries >= 4) break;
        Y.pop_back();
        F.pop_back();
        h *= 0.5;
      }
      if (!std::isfinite(fv[t])) return false;
    }
    const double better = (fv[1] < fv[0]) ? step[1] : step[0];  // towards the lower value
    sg[i] = better > 0 ? 1 : -1;
    if (x0[i] + sg[i] * delta > hi[i] || x0[i] + sg[i] * delta < lo[i]) sg[i] = -sg[i];
  }
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      std::vector<double> v = x0;
      v[i] += sg[i] * delta;
      v[j] += sg[j] * delta;
      double fv;
      if (!eval(v, fv) || !std::isfinite(fv)) return false;
    }
  // ---- main loop
  const double delta_max = std::max(delta0, 1.0);
  int stalls = 0;
  double best_sig = inf;  // best value at the last significant decrease
  int since_progress = 0;
  while (!stop()) {
    int b = (int)(std::min_element(F.begin(), F.end()) - F.begin());
    const std::vector<double> xb = Y[b];
    const double fb = F[b];
    // interpolation system in s = (y - xb) / delta
    std::vector<double> M(p * p), phi(p);
    for (int r = 0; r < p; ++r) {
      double s[3];
      for (int i = 0; i < d; ++i) s[i] = (Y[r][i] - xb[i]) / delta;
      basis(d, s, &M[r * p]);
    }
    std::vector<double> a(p);
    for (int r = 0; r < p; ++r) a[r] = F[r] - fb;
    Quad m;
    const bool poised = solve(p, M, a);
    double farthest = 0.0;
    int jfar = -1;
    for (int r = 0; r < p; ++r) {
      double dist = 0.0;
      for (int i = 0; i < d; ++i) dist = std::max(dist, std::fabs(Y[r][i] - xb[i]));
      if (dist > farthest) {
        farthest = dist;
        jfar = r;
      }
    }
    // Lagrange function of point j at s: solve M^T l = phi(s), take l_j
    auto lagrange = [&](const double* s, std::vector<double>& l) {
      basis(d, s, phi.data());
      std::vector<double> MT(p * p);
      for (int r = 0; r < p; ++r)
        for (int c2 = 0; c2 < p; ++c2) MT[c2 * p + r] = M[r * p + c2];
      l = phi;
      return solve(p, MT, l);
    };
    auto geometry_step = [&](int j) {  // replace point j by the trust-region point maximising |l_j|
      std::vector<std::vector<double>> cand;
      for (int i = 0; i < d; ++i)
        for (int sgn : {-1, 1}) {
          std::vector<double> s(d, 0.0);
          s[i] = sgn;
          cand.push_back(s);
        }
      for (int i = 0; i < d; ++i)
        for (int k = i + 1; k < d; ++k)
          for (int s1 : {-1, 1})
            for (int s2 : {-1, 1}) {
              std::vector<double> s(d, 0.0);
              s[i] = s1 * 0.7071067811865476;
              s[k] = s2 * 0.7071067811865476;
              cand.push_back(s);
            }
      double bestl = -1.0;
      std::vector<double> bests;
      std::vector<double> l;
      for (auto& s : cand) {
        std::vector<double> v(d);
        for (int i = 0; i < d; ++i) v[i] = xb[i] + delta * s[i];
        v = clampv(v);
        double sc[3];
        for (int i = 0; i < d; ++i) sc[i] = (v[i] - xb[i]) / delta;
        double lj = 1.0;
        if (poised) {
          if (!lagrange(sc, l)) continue;
          lj = std::fabs(l[j]);
        }
        bool dup = false;  // never re-use an interpolation point
        for (auto& y : Y) {
          double dd = 0.0;
          for (int i = 0; i < d; ++i) dd = std::max(dd, std::fabs(y[i] - v[i]));
          if (dd < 1e-3 * delta) dup = true;
        }
        if (!dup && lj > bestl) {
          bestl = lj;
          bests = v;
        }
      }
      if (bests.empty()) return false;
      if (stop()) return false;
      const double fv = fn(bests);
      if (!std::isfinite(fv)) {
        delta *= 0.5;
        return true;
      }
      Y[j] = bests;
      F[j] = fv;
      return true;
    };
    if (!poised) {  // degenerate set: re-poise with a geometry step on the farthest point
      if (jfar < 0 || jfar == b || !geometry_step(jfar)) {
        if (delta <= delta_end) break;
        delta *= 0.5;
      }
      if (++stalls > 50) break;
      continue;
    }
    m.from_coeffs(d, a);
    double slo[3], shi[3], s[3];
    for (int i = 0; i < d; ++i) {
      slo[i] = std::max(-1.0, (lo[i] - xb[i]) / delta);
      shi[i] = std::min(1.0, (hi[i] - xb[i]) / delta);
    }
    minimize_box(m, slo, shi, s);
    const double pred = -m.value(s);
    double snorm = 0.0;
    for (int i = 0; i < d; ++i) snorm = std::max(snorm, std::fabs(s[i]));
    // reductions below the evaluation noise carry no information: they count as no progress
    // (a log-likelihood from an n x n Cholesky is reproducible but not smooth below ~n eps
    // relative; 1e-11 covers n <= 1e5 with margin)
    const double noise = 1e-11 * std::max(1.0, std::fabs(fb));
    if (fb < best_sig - noise) {  // significant progress since the last check
      best_sig = fb;
      since_progress = 0;
    } else if (++since_progress > 8 * p) {
      break;  // 8 p iterations without a significant decrease: converged to noise level
    }
    if (!(pred > noise) || snorm < 0.05) {
      // no useful step at this radius: fix the geometry if points are far, else shrink
      if (farthest > 2.0 * delta && jfar != b) {
        if (!geometry_step(jfar)) break;
        continue;
      }
      if (delta <= delta_end) break;
      delta = std::max(0.1 * delta, 0.5 * delta_end);
      continue;
    }
    std::vector<double> xn(d);
    for (int i = 0; i < d; ++i) xn[i] = xb[i] + delta * s[i];
    xn = clampv(xn);
    if (stop()) break;
    const double fn_new = fn(xn);
    if (!std::isfinite(fn_new)) {
      delta *= 0.5;
      if (delta < delta_end) break;
      continue;
    }
    const double ratio = (fb - fn_new > noise) ? (fb - fn_new) / pred : 0.0;
    // replacement: the point whose Lagrange function is largest at the trial point,
    // weighted by its distance (never the best point unless the trial point improves)
    std::vector<double> l;
    int jout = -1;
    if (lagrange(s, l)) {
      double bw = -1.0;
      for (int r = 0; r < p; ++r) {
        if (r == b && !(fn_new < fb)) continue;
        double dist = 0.0;
        for (int i = 0; i < d; ++i) dist = std::max(dist, std::fabs(Y[r][i] - xn[i]));
        const double w = std::fabs(l[r]) * std::max(1.0, (dist / delta) * (dist / delta));
        if (w > bw) {
          bw = w;
          jout = r;
        }
      }
    } else {
      jout = (jfar == b && !(fn_new < fb)) ? (b + 1) % p : jfar;
    }
    Y[jout] = xn;
    F[jout] = fn_new;
    if (ratio < 0.1) {
      delta = std::max(0.5 * delta * std::max(snorm, 0.2), 0.5 * delta_end);
      if (delta <= delta_end && farthest <= 2.0 * delta) break;
    } else if (ratio > 0.7 && snorm > 0.9) {
      delta = std::min(2.0 * delta, delta_max);
    }
    stalls = 0;
  }
  return true;
}

}  // namespace dfo
}  // namespace exageo
