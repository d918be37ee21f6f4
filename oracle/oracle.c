/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the exact Gaussian
 * log-likelihood of ExaGeoStat (arXiv 1708.02835). It exists so that the CUDA
 * path can be checked against something written directly from the paper.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it. It shares no code with paper_1708_02835_b200/ (no common
 * headers, helpers, tables or constants) and the product never calls it.
 *
 * Citations "P:<line>" refer to PAPER.md of arXiv 1708.02835 (the LaTeX text);
 * "DESIGN R<k>" to the numbered readings in DESIGN.md (where the paper is
 * silent or garbled).
 *
 * Arithmetic is IEEE double unless noted; special functions and the final
 * reductions are carried in long double (x87 80-bit) so that the oracle's own
 * rounding stays well below the 1e-10 parity tolerance.
 *
 * Build (done by oracle/__init__.py::build):
 *   gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared oracle.c -o liboracle.so -lm
 * -ffp-contract=off matters for the location generator (bit-exact, DESIGN R3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* 1. Location generator: jittered grid, P:842-845 (Sec. 7.1), DESIGN R1-R3. */
/* ------------------------------------------------------------------------ */

/* SplitMix64 finaliser (Steele, Lea, Flood 2014), written out from its
 * published definition: add the golden gamma, then two xor-shift-multiply
 * rounds and a final xor-shift. */
static uint64_t orc_splitmix64(uint64_t v) {
  v = v + 0x9E3779B97F4A7C15ULL;
  v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ULL;
  v = (v ^ (v >> 27)) * 0x94D049BB133111EBULL;
  return v ^ (v >> 31);
}

uint64_t oracle_splitmix64(uint64_t v) { return orc_splitmix64(v); }

/* Counter-based draw number i of stream `stream` (DESIGN R3):
 *   draw(seed, stream, i) = splitmix64(splitmix64(seed XOR stream) + i). */
uint64_t oracle_draw(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t base = orc_splitmix64(seed ^ stream);
  return orc_splitmix64(base + i);
}

#define ORC_STREAM_SUBSET 0x4C4F43535542534BULL /* grid subset keys (R2) */
#define ORC_STREAM_JITTER 0x4C4F434A49545452ULL /* jitter X_rl, Y_rl (R3) */

/* u = (bits >> 11) * 2^-53 in [0,1), exact. */
static double orc_unit(uint64_t bits) { return (double)(bits >> 11) * (1.0 / 9007199254740992.0); }

static int orc_cmp_key(const void* a, const void* b) {
  const uint64_t* x = (const uint64_t*)a;
  const uint64_t* y = (const uint64_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}
static int orc_cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Locations (x_q, y_q) = ((r - 0.5 + X_rl)/g, (l - 0.5 + Y_rl)/g), r,l in 1..g,
 * X,Y ~ U(-0.4, 0.4) (reading R1: divide by g = ceil(sqrt n)).
 * Non-square n (R2): grid index q = (r-1)*g + (l-1) gets key
 * draw(seed, SUBSET, q); the n smallest (key, q) pairs are kept and emitted
 * in increasing q. Jitter (R3): X = 0.8*u(draw(seed,JITTER,2q)) - 0.4,
 * Y = 0.8*u(draw(seed,JITTER,2q+1)) - 0.4, evaluated in exactly this order
 * with round-to-nearest and no contraction. Returns 0, or -1 if n < 1. */
int oracle_gen_locations(int64_t n, uint64_t seed, double* x, double* y) {
  if (n < 1) return -1;
  int64_t g = (int64_t)ceil(sqrt((double)n));
  while (g * g < n) ++g;
  while ((g - 1) * (g - 1) >= n) --g;
  int64_t G = g * g;
  uint64_t* kq = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)G);
  if (!kq) return -3;
  for (int64_t q = 0; q < G; ++q) {
    kq[2 * q] = oracle_draw(seed, ORC_STREAM_SUBSET, (uint64_t)q);
    kq[2 * q + 1] = (uint64_t)q;
  }
  qsort(kq, (size_t)G, 2 * sizeof(uint64_t), orc_cmp_key);
  uint64_t* sel = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  if (!sel) { free(kq); return -3; }
  for (int64_t i = 0; i < n; ++i) sel[i] = kq[2 * i + 1];
  free(kq);
  qsort(sel, (size_t)n, sizeof(uint64_t), orc_cmp_u64);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t q = sel[i];
    int64_t r = (int64_t)(q / (uint64_t)g) + 1;
    int64_t l = (int64_t)(q % (uint64_t)g) + 1;
    double X = 0.8 * orc_unit(oracle_draw(seed, ORC_STREAM_JITTER, 2 * q)) - 0.4;
    double Y = 0.8 * orc_unit(oracle_draw(seed, ORC_STREAM_JITTER, 2 * q + 1)) - 0.4;
    double tx = (double)r - 0.5;
    double ty = (double)l - 0.5;
    tx = tx + X;
    ty = ty + Y;
    x[i] = tx / (double)g;
    y[i] = ty / (double)g;
  }
  free(sel);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* 2. Special functions for Eq. (2): Gamma and modified Bessel K_nu.         */
/* ------------------------------------------------------------------------ */

/* log Gamma(z) for z > 0 in long double: shift z up to >= 24 with the
 * recurrence Gamma(z+1) = z Gamma(z), then Stirling's series
 *   ln G(w) = (w-1/2) ln w - w + ln(2 pi)/2 + sum_k B_2k / (2k(2k-1) w^(2k-1)).
 * Eight terms at w >= 24 leave a truncation error below 1e-30. */
long double oracle_lgammal(long double z) {
  long double shift = 0.0L;
  while (z < 24.0L) { shift += logl(z); z += 1.0L; }
  static const long double B[8] = {1.0L / 6, -1.0L / 30, 1.0L / 42, -1.0L / 30,
                                   5.0L / 66, -691.0L / 2730, 7.0L / 6, -3617.0L / 510};
  long double s = (z - 0.5L) * logl(z) - z + 0.5L * logl(2.0L * 3.14159265358979323846264338327950288L);
  long double zp = z;
  for (int k = 1; k <= 8; ++k) {
    s += B[k - 1] / ((long double)(2 * k) * (long double)(2 * k - 1) * zp);
    zp *= z * z;
  }
  return s - shift;
}

double oracle_gamma(double z) { return (double)expl(oracle_lgammal((long double)z)); }

/* K_nu(x) from the integral representation
 *   K_nu(x) = int_0^inf exp(-x cosh t) cosh(nu t) dt      (x > 0),
 * by the trapezoid rule on [0, inf) with step h = min(1/8, 1/(4 sqrt x)),
 * summed in long double until the terms fall below 1e-22 of the sum.
 * The integrand is analytic and decays doubly exponentially, so the
 * trapezoid error is far below double precision at this step. Returns the
 * SCALED value e^x K_nu(x) (exp(-x cosh t) = e^-x exp(-2x sinh^2(t/2))),
 * which stays representable for large x. */
long double oracle_bessel_k_scaled_l(long double nu, long double x) {
  long double h = 0.125L;
  long double hx = 0.25L / sqrtl(x);
  if (hx < h) h = hx;
  long double sum = 0.5L; /* t = 0 term: exp(0) * cosh(0) / 2 */
  for (long k = 1; k < 100000; ++k) {
    long double t = h * (long double)k;
    long double sh = sinhl(0.5L * t);
    long double term = expl(-2.0L * x * sh * sh) * coshl(nu * t);
    sum += term;
    if (term < 1e-22L * sum && x * sh * sh > 1.0L) break;
  }
  return h * sum;
}

double oracle_bessel_k(double nu, double x) {
  if (!(x > 0.0)) return NAN;
  return (double)(expl(-(long double)x) * oracle_bessel_k_scaled_l((long double)nu, (long double)x));
}

/* Matern covariance, Eq. (2):
 *   C(r; theta) = theta1 / (2^(theta3-1) Gamma(theta3)) (r/theta2)^theta3 K_theta3(r/theta2)
 * with C(0) = theta1, the r -> 0 limit (DESIGN R9). Evaluated in long double:
 * C = theta1 * exp( theta3 ln x - x - (theta3-1) ln 2 - lnGamma(theta3) ) * [e^x K(x)]. */
long double oracle_matern_l(long double r, long double t1, long double t2, long double t3) {
  if (r == 0.0L) return t1;
  long double x = r / t2;
  long double lg = oracle_lgammal(t3);
  long double ks = oracle_bessel_k_scaled_l(t3, x);
  long double e = t3 * logl(x) - x - (t3 - 1.0L) * logl(2.0L) - lg;
  return t1 * expl(e) * ks;
}

double oracle_matern(double r, double t1, double t2, double t3) {
  return (double)oracle_matern_l((long double)r, (long double)t1, (long double)t2, (long double)t3);
}

/* Distance metric of all oracle routines: 0 = Euclidean, 1 = great-circle. */
static int orc_metric = 0;
static double orc_radius = 6371.0;

void oracle_set_distance(int metric, double radius) {
  orc_metric = metric;
  orc_radius = radius;
}

/* Euclidean distance r = sqrt(dx*dx + dy*dy) (DESIGN R15), or the great-circle
 * distance by the haversine formula, x = longitude and y = latitude in
 * degrees, computed in long double:
 *   hav(d/R) = hav(phi2 - phi1) + cos(phi1) cos(phi2) hav(lambda2 - lambda1),
 *   hav(a) = sin^2(a/2),  d = 2 R asin(sqrt(hav(d/R))). */
static double orc_dist(double x1, double y1, double x2, double y2) {
  if (orc_metric == 1) {
    const long double deg = 3.14159265358979323846264338327950288L / 180.0L;
    long double p1 = (long double)y1 * deg, p2 = (long double)y2 * deg;
    long double l1 = (long double)x1 * deg, l2 = (long double)x2 * deg;
    long double s1 = sinl(0.5L * (p2 - p1)), s2 = sinl(0.5L * (l2 - l1));
    long double h = s1 * s1 + cosl(p1) * cosl(p2) * s2 * s2;
    if (h > 1.0L) h = 1.0L;
    return (double)(2.0L * (long double)orc_radius * asinl(sqrtl(h)));
  }
  double dx = x1 - x2, dy = y1 - y2;
  return sqrt(dx * dx + dy * dy);
}

double oracle_distance(double x1, double y1, double x2, double y2) { return orc_dist(x1, y1, x2, y2); }

/* Dense covariance block C[i + j*ldc] = C(||s1_i - s2_j||; theta), i < m, j < n
 * (Alg. 1 l.3-4, Alg. 3 l.3-6: genDistanceMatrix + genCovMatrix, P:639-642,
 * P:734-737). Column-major. */
void oracle_cov(int64_t m, const double* x1, const double* y1, int64_t n, const double* x2,
                const double* y2, double t1, double t2, double t3, double* C, int64_t ldc) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      C[i + j * ldc] = oracle_matern(orc_dist(x1[i], y1[i], x2[j], y2[j]), t1, t2, t3);
}

/* ------------------------------------------------------------------------ */
/* 3. Linear algebra: unblocked Cholesky, forward substitution, L*e.         */
/* ------------------------------------------------------------------------ */

/* Unblocked Cholesky (Cholesky-Crout, column by column) of the n x n SPD
 * matrix A stored ROW-major (A[i*n+j]); only the lower triangle is read and
 * overwritten by L (Sigma = L L^T, Alg. 2 l.3):
 *   L_jj = sqrt(A_jj - sum_{k<j} L_jk^2)
 *   L_ij = (A_ij - sum_{k<j} L_ik L_jk) / L_jj,   i > j.
 * Returns -1 on success, else the first column j whose pivot is not > 0
 * (not positive definite; DESIGN R14). */
int64_t oracle_cholesky(int64_t n, double* A) {
  for (int64_t j = 0; j < n; ++j) {
    double* Lj = A + j * n;
    double d = Lj[j];
    for (int64_t k = 0; k < j; ++k) d -= Lj[k] * Lj[k];
    if (!(d > 0.0)) return j;
    double ljj = sqrt(d);
    Lj[j] = ljj;
#pragma omp parallel for schedule(static)
    for (int64_t i = j + 1; i < n; ++i) {
      double* Li = A + i * n;
      double s = Li[j];
      for (int64_t k = 0; k < j; ++k) s -= Li[k] * Lj[k];
      Li[j] = s / ljj;
    }
  }
  return -1;
}

/* Forward substitution L y = z (Alg. 2 l.4, P:666-667 / P:683, DESIGN R6):
 * y_i = (z_i - sum_{k<i} L_ik y_k) / L_ii, L row-major lower. */
void oracle_forward(int64_t n, const double* L, const double* z, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    const double* Li = L + i * n;
    double s = z[i];
    for (int64_t k = 0; k < i; ++k) s -= Li[k] * y[k];
    y[i] = s / Li[i];
  }
}

/* Backward substitution L^T x = y (for Alg. 3's dposv, DESIGN R19). */
void oracle_backward(int64_t n, const double* L, const double* y, double* x) {
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
    x[i] = s / L[i * n + i];
  }
}

/* ------------------------------------------------------------------------ */
/* 4. Algorithms 1-3.                                                        */
/* ------------------------------------------------------------------------ */

/* Row-major full covariance of n locations (both triangles). */
static double* orc_build_sigma(int64_t n, const double* x, const double* y, double t1, double t2,
                               double t3) {
  double* S = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!S) return NULL;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double c = (i == j) ? t1 : oracle_matern(orc_dist(x[i], y[i], x[j], y[j]), t1, t2, t3);
      S[i * n + j] = c;
      S[j * n + i] = c;
    }
  return S;
}

/* Algorithm 2 / Eq. (1):
 *   Sigma = genCovMatrix(D, theta); L L^T = dpotrf(Sigma); y = L^{-1} z;
 *   logdet = 2 sum log L_ii (R5); dot = y^T y (R7);
 *   l = -0.5 dot - 0.5 logdet - (n/2) log(2 pi).
 * Outputs are written through out[3] = {loglik, logdet, quad}.
 * Returns 0, -2 (not PD, *pivot set), -3 (out of memory). */
int oracle_loglik(int64_t n, const double* x, const double* y, const double* z, double t1,
                  double t2, double t3, double* out, int64_t* pivot) {
  double* S = orc_build_sigma(n, x, y, t1, t2, t3);
  if (!S) return -3;
  int64_t p = oracle_cholesky(n, S);
  if (pivot) *pivot = p;
  if (p >= 0) { free(S); return -2; }
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  if (!w) { free(S); return -3; }
  oracle_forward(n, S, z, w);
  long double logdet = 0.0L, quad = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    logdet += 2.0L * logl((long double)S[i * n + i]);
    quad += (long double)w[i] * (long double)w[i];
  }
  long double l2pi = logl(2.0L * 3.14159265358979323846264338327950288L);
  long double ll = -0.5L * quad - 0.5L * logdet - 0.5L * (long double)n * l2pi;
  out[0] = (double)ll;
  out[1] = (double)logdet;
  out[2] = (double)quad;
  free(w);
  free(S);
  return 0;
}

/* Algorithm 1 l.4-7 (R18): z = L e with Sigma(theta) = L L^T.
 * e (the normal variates) is an input. Returns 0 / -2 / -3 like above. */
int oracle_simulate(int64_t n, const double* x, const double* y, double t1, double t2, double t3,
                    const double* e, double* z, int64_t* pivot) {
  double* S = orc_build_sigma(n, x, y, t1, t2, t3);
  if (!S) return -3;
  int64_t p = oracle_cholesky(n, S);
  if (pivot) *pivot = p;
  if (p >= 0) { free(S); return -2; }
  for (int64_t i = 0; i < n; ++i) {
    long double s = 0.0L;
    for (int64_t k = 0; k <= i; ++k) s += (long double)S[i * n + k] * (long double)e[k];
    z[i] = (double)s;
  }
  free(S);
  return 0;
}

/* Algorithm 3 / Eq. (5): Z1 = Sigma12 Sigma22^{-1} Z2,
 * with dposv = Cholesky + forward + backward substitution (R19). */
int oracle_predict(int64_t n, const double* x, const double* y, const double* z, int64_t m,
                   const double* xn, const double* yn, double t1, double t2, double t3,
                   double* znew, int64_t* pivot) {
  double* S = orc_build_sigma(n, x, y, t1, t2, t3);
  if (!S) return -3;
  int64_t p = oracle_cholesky(n, S);
  if (pivot) *pivot = p;
  if (p >= 0) { free(S); return -2; }
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  oracle_forward(n, S, z, w);
  oracle_backward(n, S, w, v);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    long double s = 0.0L;
    for (int64_t j = 0; j < n; ++j)
      s += (long double)oracle_matern(orc_dist(xn[i], yn[i], x[j], y[j]), t1, t2, t3) * (long double)v[j];
    znew[i] = (double)s;
  }
  free(w);
  free(v);
  free(S);
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
