// test_trust_region.cpp -- CPU checks of the quadratic-model trust-region minimiser
// (paper_1708_02835_b200/csrc/trust_region.h) on functions with known minimisers.
// Prints one line per case: name evals error ok; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_1708_02835_b200/csrc/trust_region.h"

using exageo::dfo::minimize;

struct Case {
  const char* name;
  std::function<double(const std::vector<double>&)> f;
  std::vector<double> x0, lo, hi, xstar;
  double tol;
  int max_evals;
};

int main() {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<Case> cases = {
      {"1d quadratic", [](const std::vector<double>& x) { return (x[0] - 0.3) * (x[0] - 0.3) + 1.0; },
       {2.0}, {-5.0}, {5.0}, {0.3}, 1e-6, 60},
      {"2d ill-conditioned quadratic",
       [](const std::vector<double>& x) {
         const double a = x[0] - 1.0, b = x[1] + 0.5;
         return 10.0 * a * a + 0.1 * b * b + 1.5 * a * b;
       },
       {0.0, 0.0}, {-3.0, -3.0}, {3.0, 3.0}, {1.0, -0.5}, 1e-5, 80},
      {"2d rosenbrock",
       [](const std::vector<double>& x) {
         return 100.0 * (x[1] - x[0] * x[0]) * (x[1] - x[0] * x[0]) + (1 - x[0]) * (1 - x[0]);
       },
       {-1.2, 1.0}, {-2.0, -2.0}, {2.0, 2.0}, {1.0, 1.0}, 1e-4, 400},
      {"3d quadratic, minimiser outside the box (projected)",
       [](const std::vector<double>& x) {
         return (x[0] - 3) * (x[0] - 3) + 2 * (x[1] + 0.2) * (x[1] + 0.2) + (x[2] - 0.5) * (x[2] - 0.5) +
                0.5 * x[0] * x[2];
       },
       {0.0, 0.0, 0.0}, {-1.0, -1.0, -1.0}, {1.0, 1.0, 1.0}, {1.0, -0.2, 0.25}, 1e-5, 150},
      {"2d smooth with a failed (+inf) region next to the minimiser",
       [inf](const std::vector<double>& x) {
         if (x[0] + x[1] > 1.6) return inf;
         return std::pow(x[0] - 0.7, 2) + std::pow(x[1] - 0.7, 2) + 0.3 * std::pow(x[0] - x[1], 4);
       },
       {-1.0, -1.0}, {-2.0, -2.0}, {2.0, 2.0}, {0.7, 0.7}, 1e-5, 200},
      {"3d quadratic + 1e-14 relative evaluation noise (must terminate)",
       [](const std::vector<double>& x) {
         static unsigned long long st = 88172645463325252ull;
         st ^= st << 13;
         st ^= st >> 7;
         st ^= st << 17;
         const double u = (double)(st >> 11) * 0x1.0p-53 - 0.5;
         const double f = 1000.0 + 800.0 * ((x[0] - 0.2) * (x[0] - 0.2) + 2 * (x[1] + 0.1) * (x[1] + 0.1) +
                                           (x[2] - 0.3) * (x[2] - 0.3) + 0.4 * (x[0] - 0.2) * (x[2] - 0.3));
         return f * (1.0 + 1e-14 * u);
       },
       {0.5, 0.5, 0.5}, {-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {0.2, -0.1, 0.3}, 1e-5, 300},
      {"3d quadratic + 1e-10 relative noise, above the noise floor (must terminate)",
       [](const std::vector<double>& x) {
         static unsigned long long st = 1234567891011ull;
         st ^= st << 13;
         st ^= st >> 7;
         st ^= st << 17;
         const double u = (double)(st >> 11) * 0x1.0p-53 - 0.5;
         const double f = 300.0 + 800.0 * ((x[0] - 0.2) * (x[0] - 0.2) + 2 * (x[1] + 0.1) * (x[1] + 0.1) +
                                          (x[2] - 0.3) * (x[2] - 0.3));
         return f * (1.0 + 1e-10 * u);
       },
       {0.5, 0.5, 0.5}, {-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {0.2, -0.1, 0.3}, 1e-4, 400},
      {"3d log-likelihood-like (exp terms)",
       [](const std::vector<double>& x) {
         return std::exp(x[0]) - x[0] + std::exp(0.5 * x[1]) - 0.5 * x[1] + std::cosh(x[2] - 0.4) + 0.2 * x[0] * x[1];
       },
       {1.0, 1.5, -1.0}, {-4.0, -4.0, -4.0}, {4.0, 4.0, 4.0}, {0.0, 0.0, 0.4}, 2e-3, 200},
  };
  // the 3-d exp case: solve its stationarity numerically for the reference
  {
    // grad: e^x0 - 1 + 0.2 x1 = 0 ; 0.5 e^{x1/2} - 0.5 + 0.2 x0 = 0 ; sinh(x2 - .4) = 0
    double a = 0, b = 0;
    for (int it = 0; it < 200; ++it) {
      a = std::log(1 - 0.2 * b);
      b = 2 * std::log(1 - 0.4 * a);
    }
    cases[7].xstar = {a, b, 0.4};
    cases[7].tol = 1e-5;
  }
  int fails = 0;
  for (auto& c : cases) {
    int evals = 0;
    double bestf = inf;
    std::vector<double> bestx = c.x0;
    auto fn = [&](std::vector<double>& v) {
      ++evals;
      const double fv = c.f(v);
      if (fv < bestf) {
        bestf = fv;
        bestx = v;
      }
      return fv;
    };
    const bool ok0 = minimize(fn, c.x0, c.lo, c.hi, 0.3, 1e-8, [&]() { return evals >= c.max_evals; });
    double err = 0.0;
    for (size_t i = 0; i < bestx.size(); ++i) err = std::max(err, std::fabs(bestx[i] - c.xstar[i]));
    const bool ok = ok0 && err <= c.tol && evals < c.max_evals;
    fails += !ok;
    printf("%-60s evals %4d  err %.2e  %s\n", c.name, evals, err, ok ? "ok" : "FAIL");
  }
  return fails;
}
