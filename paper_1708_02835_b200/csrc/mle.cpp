// mle.cpp -- exageo_mle: maximum-likelihood estimation theta_hat = argmax l(theta)
// by a derivative-free, bound-constrained search driving the device
// log-likelihood (the paper's NLopt/BOBYQA loop; reading R16: any
// derivative-free box-constrained optimizer).
//
// Method: Nelder-Mead simplex on u = log(theta) (theta > 0 for free, relative
// tolerances become absolute ones), trial points projected onto the box
// [log lo, log hi]; parameters with lo == hi are held fixed. A non-positive-definite
// evaluation counts as l = -inf. Convergence: simplex diameter (max-norm in u)
// below xtol_rel; then one restart from the best vertex with a fresh simplex, kept only
// while it improves. Deterministic: on a distributed context every rank runs the same
// search on bitwise-identical l values (all-reduced), so no theta broadcast is needed.
//
// exageo_mle_profile: the same search over (theta2, theta3) only, with theta1 profiled out
// in closed form. Sigma(theta) = theta1 R(theta2, theta3) (Eq. 2 is linear in theta1), so one
// factorization of R gives l(s, theta2, theta3) = -q/(2s) - (n log s + log|R|)/2 - (n/2) log 2pi
// for every s, with q = z^T R^-1 z; it is unimodal in s with maximum at s = q/n, clamped to
// [lo1, hi1]. The maximiser over the box is the same as the full search's.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "context.h"
#include "trust_region.h"

namespace exageo {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct Objective {
  exageo_ctx* ctx;
  int64_t n;
  const double *x, *y, *z;
  double base[3];           // log theta of the fixed parameters / start
  std::vector<int> free_;   // indices of the free parameters
  double lo[3], hi[3];      // log bounds
  int evals = 0, max_evals = 0;
  double* trace = nullptr;
  double best_f = kInf;
  double best_u[3] = {0, 0, 0};
  exageo_status err = EXAGEO_OK;
  int fails = 0;
  double fixed[3] = {0, 0, 0};  // exact values of the fixed parameters
  bool is_free[3] = {false, false, false};
  bool profile = false;         // theta1 profiled out (exageo_mle_profile)
  double s_lo = 0, s_hi = 0;    // theta1 bounds (profile)
  exageo_theta best_theta{0, 0, 0};

  exageo_theta to_theta(const double u[3]) const {
    double v[3];
    for (int p = 0; p < 3; ++p) v[p] = is_free[p] ? std::exp(u[p]) : fixed[p];
    return exageo_theta{v[0], v[1], v[2]};
  }

  // project a free-parameter vector onto the box (in place) and evaluate -l
  double operator()(std::vector<double>& v) {
    double u[3];
    memcpy(u, base, sizeof(u));
    for (size_t i = 0; i < free_.size(); ++i) {
      const int p = free_[i];
      v[i] = std::min(std::max(v[i], lo[p]), hi[p]);
      u[p] = v[i];
    }
    if (evals >= max_evals || err != EXAGEO_OK) return kInf;
    exageo_theta t = to_theta(u);
    double ll = -kInf;
    exageo_status st;
    if (profile) {
      t.sigma2 = 1.0;
      double logdet = 0.0, quad = 0.0;
      st = eval_loglik(ctx, &t, n, x, y, z, &ll, &logdet, &quad);
      if (st == EXAGEO_OK) {
        const double nn = (double)n;
        t.sigma2 = std::min(std::max(quad / nn, s_lo), s_hi);
        const double log2pi = 1.8378770664093454835606594728112;
        ll = -0.5 * quad / t.sigma2 - 0.5 * (nn * std::log(t.sigma2) + logdet) - 0.5 * nn * log2pi;
      }
    } else {
      st = eval_loglik(ctx, &t, n, x, y, z, &ll);
    }
    if (st != EXAGEO_OK && st != EXAGEO_ENOTPD) {
      err = st;
      return kInf;
    }
    if (st == EXAGEO_ENOTPD || !std::isfinite(ll)) {
      ll = -kInf;
      ++fails;
    }
    if (trace) {
      double* r = trace + 4 * evals;
      r[0] = t.sigma2;
      r[1] = t.beta;
      r[2] = t.nu;
      r[3] = ll;
    }
    ++evals;
    const double f = -ll;
    if (f < best_f) {
      best_f = f;
      memcpy(best_u, u, sizeof(u));
      best_theta = t;
    }
    return f;
  }
};

// Nelder-Mead from simplex around v0 with steps h; returns when the simplex diameter
// drops below xtol or the evaluation budget is spent.
void nelder_mead(Objective& f, std::vector<double> v0, const std::vector<double>& h, double xtol) {
  const int d = (int)v0.size();
  std::vector<std::vector<double>> S(d + 1, v0);
  std::vector<double> F(d + 1);
  F[0] = f(S[0]);
  for (int i = 0; i < d; ++i) {
    S[i + 1][i] += h[i];
    F[i + 1] = f(S[i + 1]);
    if (S[i + 1][i] == S[0][i]) {  // clamped onto the start: step the other way
      S[i + 1][i] -= h[i];
      F[i + 1] = f(S[i + 1]);
    }
  }
  const double alpha = 1.0, gamma = 2.0, rho = 0.5, sigma = 0.5;
  std::vector<int> idx(d + 1);
  while (f.evals < f.max_evals && f.err == EXAGEO_OK) {
    for (int i = 0; i <= d; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return F[a] < F[b]; });
    {
      std::vector<std::vector<double>> S2(d + 1);
      std::vector<double> F2(d + 1);
      for (int i = 0; i <= d; ++i) {
        S2[i] = S[idx[i]];
        F2[i] = F[idx[i]];
      }
      S.swap(S2);
      F.swap(F2);
    }
    double diam = 0.0;
    for (int i = 1; i <= d; ++i)
      for (int j = 0; j < d; ++j) diam = std::max(diam, std::fabs(S[i][j] - S[0][j]));
    if (diam <= xtol) break;
    std::vector<double> c(d, 0.0);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) c[j] += S[i][j] / d;
    auto along = [&](double t, const std::vector<double>& p) {
      std::vector<double> q(d);
      for (int j = 0; j < d; ++j) q[j] = c[j] + t * (p[j] - c[j]);
      return q;
    };
    std::vector<double> r = along(-alpha, S[d]);
    const double fr = f(r);
    if (fr < F[0]) {
      std::vector<double> e = along(-gamma, S[d]);
      const double fe = f(e);
      if (fe < fr) {
        S[d] = e;
        F[d] = fe;
      } else {
        S[d] = r;
        F[d] = fr;
      }
      continue;
    }
    if (fr < F[d - 1]) {
      S[d] = r;
      F[d] = fr;
      continue;
    }
    bool shrink = false;
    if (fr < F[d]) {
      std::vector<double> oc = along(-rho, S[d]);
      const double foc = f(oc);
      if (foc <= fr) {
        S[d] = oc;
        F[d] = foc;
      } else {
        shrink = true;
      }
    } else {
      std::vector<double> ic = along(rho, S[d]);
      const double fic = f(ic);
      if (fic < F[d]) {
        S[d] = ic;
        F[d] = fic;
      } else {
        shrink = true;
      }
    }
    if (shrink) {
      for (int i = 1; i <= d; ++i) {
        for (int j = 0; j < d; ++j) S[i][j] = S[0][j] + sigma * (S[i][j] - S[0][j]);
        F[i] = f(S[i]);
      }
    }
  }
}

}  // namespace
}  // namespace exageo

using namespace exageo;

namespace {

exageo_status run_mle(exageo_ctx* c, int64_t n, const double* x, const double* y, const double* z,
                      const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start, double xtol_rel,
                      int max_evals, exageo_theta* theta_hat, double* loglik, int* nevals, double* trace,
                      bool profile, int method) {
  if (!c) return EXAGEO_EINVAL;
  if (n < 1 || !x || !y || !z || !lo || !hi || !start || !theta_hat || max_evals < 1 || !(xtol_rel > 0))
    return set_error(c, EXAGEO_EINVAL, "bad arguments to exageo_mle");
  const double l3[3] = {lo->sigma2, lo->beta, lo->nu}, h3[3] = {hi->sigma2, hi->beta, hi->nu};
  const double s3[3] = {start->sigma2, start->beta, start->nu};
  for (int p = 0; p < 3; ++p)
    if (!(l3[p] > 0) || !std::isfinite(h3[p]) || h3[p] < l3[p] || s3[p] < l3[p] || s3[p] > h3[p])
      return set_error(c, EXAGEO_EINVAL, "bounds must satisfy 0 < lo <= start <= hi");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return set_error(c, EXAGEO_ECUDA, cudaGetErrorString(e));
  double* buf = nullptr;
  exageo_status st = staging(c, n, &buf);
  if (st != EXAGEO_OK) return st;
  double *dx = buf, *dy = buf + n, *dz = buf + 2 * n;
  for (auto [dst, src] : {std::pair<double*, const double*>{dx, x}, {dy, y}, {dz, z}}) {
    e = cudaMemcpyAsync(dst, src, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) return set_error(c, EXAGEO_ECUDA, cudaGetErrorString(e));
  }

  Objective f;
  f.ctx = c;
  f.n = n;
  f.x = dx;
  f.y = dy;
  f.z = dz;
  f.max_evals = max_evals;
  f.trace = trace;
  f.profile = profile;
  f.s_lo = l3[0];
  f.s_hi = h3[0];
  std::vector<double> v0, h;
  for (int p = 0; p < 3; ++p) {
    f.lo[p] = std::log(l3[p]);
    f.hi[p] = std::log(h3[p]);
    f.base[p] = std::log(s3[p]);
    f.fixed[p] = s3[p];
    f.is_free[p] = h3[p] > l3[p] && !(profile && p == 0);
    if (f.is_free[p]) {
      f.free_.push_back(p);
      v0.push_back(f.base[p]);
      h.push_back(0.1 * (f.hi[p] - f.lo[p]));
    }
  }
  if (f.free_.empty()) {
    std::vector<double> none;
    f(none);
  } else if (method == 1) {
    // quadratic-model trust region (trust_region.h) on the free log-parameters
    std::vector<double> lo_f, hi_f;
    double span = 1.0;
    for (int p : f.free_) {
      lo_f.push_back(f.lo[p]);
      hi_f.push_back(f.hi[p]);
      span = std::min(span, f.hi[p] - f.lo[p]);
    }
    const double delta0 = std::max(0.1 * span, 10.0 * xtol_rel);
    const bool ok = dfo::minimize([&](std::vector<double>& v) { return f(v); }, v0, lo_f, hi_f, delta0, xtol_rel,
                                  [&]() { return f.evals >= f.max_evals || f.err != EXAGEO_OK; });
    if (!ok && f.err == EXAGEO_OK && f.evals < f.max_evals) nelder_mead(f, v0, h, xtol_rel);  // fallback
  } else {
    nelder_mead(f, v0, h, xtol_rel);
    // restarts from the best vertex with a small fresh simplex while they improve
    for (int rs = 0; rs < 3 && f.evals < f.max_evals && f.err == EXAGEO_OK; ++rs) {
      const double before = f.best_f;
      std::vector<double> vb, hb;
      for (size_t i = 0; i < f.free_.size(); ++i) {
        const int p = f.free_[i];
        vb.push_back(f.best_u[p]);
        hb.push_back(std::max(100.0 * xtol_rel, 0.01 * (f.hi[p] - f.lo[p])));
      }
      nelder_mead(f, vb, hb, xtol_rel);
      if (!(f.best_f < before - 1e-12 * std::fabs(before))) break;
    }
  }
  if (f.err != EXAGEO_OK) return f.err;
  if (nevals) *nevals = f.evals;
  if (!std::isfinite(f.best_f)) return set_error(c, EXAGEO_EFIT, "every likelihood evaluation failed");
  *theta_hat = f.best_theta;
  if (loglik) *loglik = -f.best_f;
  return EXAGEO_OK;
}

}  // namespace

extern "C" exageo_status exageo_mle(exageo_ctx* c, int64_t n, const double* x, const double* y, const double* z,
                                    const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start,
                                    double xtol_rel, int max_evals, exageo_theta* theta_hat, double* loglik,
                                    int* nevals, double* trace) {
  return run_mle(c, n, x, y, z, lo, hi, start, xtol_rel, max_evals, theta_hat, loglik, nevals, trace, false, 0);
}

extern "C" exageo_status exageo_mle_profile(exageo_ctx* c, int64_t n, const double* x, const double* y,
                                            const double* z, const exageo_theta* lo, const exageo_theta* hi,
                                            const exageo_theta* start, double xtol_rel, int max_evals,
                                            exageo_theta* theta_hat, double* loglik, int* nevals, double* trace) {
  return run_mle(c, n, x, y, z, lo, hi, start, xtol_rel, max_evals, theta_hat, loglik, nevals, trace, true, 0);
}

extern "C" exageo_status exageo_mle_ex(exageo_ctx* c, int64_t n, const double* x, const double* y, const double* z,
                                       const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start,
                                       const exageo_mle_opts* o, exageo_theta* theta_hat, double* loglik,
                                       int* nevals, double* trace) {
  if (!c) return EXAGEO_EINVAL;
  if (!o || o->method < 0 || o->method > 1) return set_error(c, EXAGEO_EINVAL, "bad exageo_mle_opts");
  return run_mle(c, n, x, y, z, lo, hi, start, o->xtol_rel, o->max_evals, theta_hat, loglik, nevals, trace,
                 o->profile != 0, o->method);
}
