// api.cu -- the C ABI (include/exageo.h) and the device-side schedule of one
// log-likelihood evaluation (Alg. 2):
//
//   K1 gen_panels                       Sigma(theta) lower panels + z row   (l.2)
//   for k = 0 .. T-1                    right-looking tile Cholesky          (l.3)
//     for s = 0 .. nb/64 - 1            left-looking factorization of panel k
//       gemm_panel  (s > 0)             P[c0:, c0:c0+64] -= P[c0:, :c0] P[c0:c0+64, :c0]^T
//       potrf_block                     L_ss, W = L_ss^{-1}, sum log L_ii, pivot check
//       gemm_panel  (TRSM)              P[c0+64:, c0:c0+64] = P[c0+64:, c0:c0+64] W^T
//     syrk_trailing(k)                  A_ij -= L_ik L_jk^T, i >= j > k (incl. z row -> forward solve, l.4)
//   finish                              logdet, dot, l                        (l.5-7)
//
// All launches are stream-ordered on the context stream.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/exageo.h"
#include "internal.h"

namespace exageo {
int gen_locations_host(int64_t n, uint64_t seed, double* x, double* y);
}

using namespace exageo;

struct exageo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nb_opt = 0;
  // tile workspace
  double* ws = nullptr;
  size_t ws_bytes = 0;
  bool ws_external = false;
  // small device buffers
  double* W = nullptr;      // PB x PB inverse of the current diagonal block
  double* slots = nullptr;  // log-det partials, one per potrf block
  int64_t slots_cap = 0;
  double* out = nullptr;    // kOutDoubles
  int* info = nullptr;      // 0 or first bad pivot + 1
  double* vec = nullptr;    // 4 * n staging for host-pointer entry points
  int64_t vec_cap = 0;
  double* part = nullptr;   // TRMV scratch
  size_t part_cap = 0;
  Layout L;
  bool have_matrix = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // lookahead schedule: two prioritised internal streams and their events
  cudaStream_t s_la = nullptr, s_main = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_F = nullptr, ev_U2 = nullptr, ev_join[2] = {nullptr, nullptr};
  // timing of the dominant kernel (bulk trailing update U2): one event pair per launch
  std::vector<cudaEvent_t> ev_u2_beg, ev_u2_end;
  int n_u2 = 0;
  double u2_flops = 0.0;
  int64_t kernels = 0;
  std::string err;
};

namespace {

std::string g_create_err = "no error";

exageo_status fail(exageo_ctx* c, exageo_status s, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_err = msg;
  return s;
}

#define CUDA_TRY(ctx, call)                                                                          \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      return fail((ctx), EXAGEO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

bool theta_ok(const exageo_theta* t) {
  return t && std::isfinite(t->sigma2) && std::isfinite(t->beta) && std::isfinite(t->nu) && t->sigma2 > 0 &&
         t->beta > 0 && t->nu > 0;
}

int auto_nb(int64_t n) {
  if (n >= 10000) return 512;
  if (n >= 2000) return 256;
  return 128;
}

Layout make_layout(int64_t n, int nb) {
  Layout L;
  L.n = n;
  L.nb = nb;
  L.T = (int)((n + nb - 1) / nb);
  L.N = (int64_t)L.T * nb;
  return L;
}

// Per-theta constants of Eq. (2), long double on the host.
MaternConsts make_consts(const exageo_theta& t) {
  MaternConsts c{};
  const long double nu = t.nu;
  c.theta1 = t.sigma2;
  c.inv_theta2 = 1.0 / t.beta;
  c.nu = t.nu;
  c.kind = (t.nu == 0.5) ? 1 : (t.nu == 1.5) ? 2 : (t.nu == 2.5) ? 3 : 0;
  c.nl = (int)std::floor(t.nu + 0.5);
  const long double mu = nu - (long double)c.nl;
  c.mu = (double)mu;
  c.pref = (double)expl(logl((long double)t.sigma2) - (nu - 1.0L) * logl(2.0L) - lgammal(nu));
  const long double gampl = 1.0L / tgammal(1.0L + mu);
  const long double gammi = 1.0L / tgammal(1.0L - mu);
  c.gampl = (double)gampl;
  c.gammi = (double)gammi;
  c.gam2 = (double)(0.5L * (gammi + gampl));
  if (fabsl(mu) < 1e-4L) {
    // gamma_1(mu) = (1/Gamma(1-mu) - 1/Gamma(1+mu)) / (2 mu) = -(g + c4 mu^2 + O(mu^4)),
    // g = Euler's constant, c4 = -0.0420026350340952 (Taylor series of 1/Gamma).
    c.gam1 = (double)(-(0.57721566490153286060651209L - 0.04200263503409523553L * mu * mu));
  } else {
    c.gam1 = (double)((gammi - gampl) / (2.0L * mu));
  }
  const long double pimu = 3.14159265358979323846264338327950288L * mu;
  c.pimu_sin = (mu == 0.0L) ? 1.0 : (double)(pimu / sinl(pimu));
  return c;
}

exageo_status ensure_vec(exageo_ctx* c, int64_t n) {
  if (c->vec_cap >= n) return EXAGEO_OK;
  if (c->vec) cudaFree(c->vec);
  c->vec = nullptr;
  c->vec_cap = 0;
  CUDA_TRY(c, cudaMalloc(&c->vec, sizeof(double) * 4 * (size_t)n));
  c->vec_cap = n;
  return EXAGEO_OK;
}

exageo_status ensure_workspace(exageo_ctx* c, const Layout& L) {
  const size_t need = (size_t)L.total() * sizeof(double) + 256 * sizeof(double);  // slack: masked tail reads
  const int64_t nslots = (int64_t)L.T * (L.nb / PB);
  if (c->slots_cap < nslots) {
    if (c->slots) cudaFree(c->slots);
    c->slots = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->slots, sizeof(double) * (size_t)nslots));
    c->slots_cap = nslots;
  }
  if (c->ws_external) {
    if (c->ws_bytes < need)
      return fail(c, EXAGEO_ENOMEM, "external workspace too small: need " + std::to_string(need) + " bytes");
    return EXAGEO_OK;
  }
  if (c->ws_bytes >= need) return EXAGEO_OK;
  if (c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  c->ws_bytes = 0;
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(c, cudaMemGetInfo(&free_b, &total_b));
  if (need > free_b)
    return fail(c, EXAGEO_ENOMEM,
                "tile workspace needs " + std::to_string(need) + " bytes, " + std::to_string(free_b) + " free");
  cudaError_t e = cudaMalloc(&c->ws, need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, EXAGEO_ENOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
  }
  c->ws_bytes = need;
  return EXAGEO_OK;
}

exageo_status check_launch(exageo_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, EXAGEO_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return EXAGEO_OK;
}

exageo_status do_generate(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                          const double* z) {
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  if (n < 1 || !x || !y) return fail(c, EXAGEO_EINVAL, "n < 1 or NULL location array");
  const int nb = c->nb_opt > 0 ? c->nb_opt : auto_nb(n);
  c->L = make_layout(n, nb);
  exageo_status st = ensure_workspace(c, c->L);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemsetAsync(c->info, 0, sizeof(int), c->stream));
  const MaternConsts mc = make_consts(*t);
  launch_gen_panels(c->L, c->ws, mc, x, y, z, c->stream);
  c->kernels += 1;
  c->have_matrix = true;
  return check_launch(c);
}

// Factor panel k (left-looking over PB-wide column blocks) on stream s.
void factor_panel(exageo_ctx* c, int k, cudaStream_t s) {
  const Layout& L = c->L;
  const int nsub = L.nb / PB;
  double* Pk = c->ws + L.off(k);
  const int64_t ldk = L.ld(k);
  for (int sb = 0; sb < nsub; ++sb) {
    const int64_t c0 = (int64_t)sb * PB;
    if (sb > 0) {
      launch_gemm_panel(ldk - c0, PB, (int)c0, Pk + c0, ldk, Pk + c0, ldk, Pk + c0 * ldk + c0, ldk, true, c->info, s);
      c->kernels += 1;
    }
    launch_potrf_block(Pk + c0 * ldk + c0, ldk, c->W, c->slots + (int64_t)k * nsub + sb, c->info,
                       (int64_t)k * L.nb + c0, s);
    double* below = Pk + c0 * ldk + c0 + PB;
    launch_gemm_panel(ldk - c0 - PB, PB, PB, below, ldk, c->W, PB, below, ldk, false, c->info, s);
    c->kernels += 2;
  }
}

// Right-looking tile Cholesky with depth-1 lookahead (the paper's "updates of the
// trailing submatrix may be triggered before the current panel factorization is
// complete"), as two prioritised CUDA streams instead of a runtime DAG:
//   s_la  (high priority): U1(k) = update of tile column k+1 by panel k, then F(k+1)
//   s_main (low priority): U2(k) = update of tile columns >= k+2 by panel k
// Dependencies: U1(k) after U2(k-1); U2(k) after F(k). F(k+1) overlaps U2(k).
exageo_status do_factor(exageo_ctx* c) {
  if (!c->have_matrix) return fail(c, EXAGEO_EINVAL, "no generated matrix in the workspace");
  const Layout& L = c->L;
  const int cpt = L.nb / 128;  // 128-column blocks per tile column
  c->n_u2 = 0;
  c->u2_flops = 0.0;
  CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->s_la, c->ev_fork, 0));
  CUDA_TRY(c, cudaStreamWaitEvent(c->s_main, c->ev_fork, 0));
  factor_panel(c, 0, c->s_la);
  CUDA_TRY(c, cudaEventRecord(c->ev_F, c->s_la));
  for (int k = 0; k + 1 < L.T; ++k) {
    CUDA_TRY(c, cudaStreamWaitEvent(c->s_main, c->ev_F, 0));    // U2(k) needs F(k)
    if (k > 0) CUDA_TRY(c, cudaStreamWaitEvent(c->s_la, c->ev_U2, 0));  // U1(k) needs U2(k-1)
    launch_syrk_trailing(L, c->ws, k, 0, cpt, c->info, c->s_la);       // U1(k)
    factor_panel(c, k + 1, c->s_la);                                   // F(k+1)
    CUDA_TRY(c, cudaEventRecord(c->ev_F, c->s_la));
    c->kernels += 1;
    if (k + 2 < L.T) {
      if ((int)c->ev_u2_beg.size() <= c->n_u2) {
        cudaEvent_t b, e;
        CUDA_TRY(c, cudaEventCreate(&b));
        CUDA_TRY(c, cudaEventCreate(&e));
        c->ev_u2_beg.push_back(b);
        c->ev_u2_end.push_back(e);
      }
      CUDA_TRY(c, cudaEventRecord(c->ev_u2_beg[c->n_u2], c->s_main));
      launch_syrk_trailing(L, c->ws, k, cpt, -1, c->info, c->s_main);  // U2(k)
      CUDA_TRY(c, cudaEventRecord(c->ev_u2_end[c->n_u2], c->s_main));
      ++c->n_u2;
      const double m = (double)(L.n - (int64_t)(k + 2) * L.nb);  // true columns updated
      if (m > 0) c->u2_flops += 2.0 * L.nb * (m * (m + 1) / 2 + m);
      c->kernels += 1;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_U2, c->s_main));
  }
  CUDA_TRY(c, cudaEventRecord(c->ev_join[0], c->s_la));
  CUDA_TRY(c, cudaEventRecord(c->ev_join[1], c->s_main));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join[0], 0));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join[1], 0));
  return check_launch(c);
}

exageo_status do_finish(exageo_ctx* c, double* out3, int64_t* pivot) {
  const Layout& L = c->L;
  launch_finish(L, c->ws, c->slots, L.T * (L.nb / PB), c->out, c->stream);
  c->kernels += 2;
  exageo_status st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  double h[3];
  int info = 0;
  CUDA_TRY(c, cudaMemcpyAsync(h, c->out, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&info, c->info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (pivot) *pivot = info > 0 ? (int64_t)info - 1 : -1;
  if (info > 0) {
    if (out3) {
      out3[0] = -std::numeric_limits<double>::infinity();
      out3[1] = out3[2] = std::numeric_limits<double>::quiet_NaN();
    }
    return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(info - 1));
  }
  if (out3) memcpy(out3, h, sizeof(h));
  return EXAGEO_OK;
}

exageo_status loglik_device(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                            const double* z, double* loglik, exageo_loglik_info* info) {
  if (!z) return fail(c, EXAGEO_EINVAL, "NULL z");
  const int64_t k0 = c->kernels;
  CUDA_TRY(c, cudaEventRecord(c->ev[0], c->stream));
  exageo_status st = do_generate(c, t, n, x, y, z);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev[1], c->stream));
  st = do_factor(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev[2], c->stream));
  double r3[3];
  int64_t piv = -1;
  st = do_finish(c, r3, &piv);  // records nothing after; ev[3] below
  if (st != EXAGEO_OK && st != EXAGEO_ENOTPD) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev[3], c->stream));
  CUDA_TRY(c, cudaEventSynchronize(c->ev[3]));
  if (loglik) *loglik = r3[0];
  if (info) {
    memset(info, 0, sizeof(*info));
    info->loglik = r3[0];
    info->logdet = r3[1];
    info->quad = r3[2];
    info->npd_pivot = piv;
    info->n = n;
    info->nb = c->L.nb;
    info->ntiles = c->L.T;
    info->flops = (double)n * (double)n * (double)n / 3.0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]);
    info->ms_total = ms;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    info->ms_gen = ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
    info->ms_chol = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    info->ms_reduce = ms;
    info->kernels = c->kernels - k0;
    info->trailing_launches = c->n_u2;
    info->trailing_flops = c->u2_flops;
    double tr = 0.0;
    for (int i = 0; i < c->n_u2; ++i) {
      cudaEventElapsedTime(&ms, c->ev_u2_beg[i], c->ev_u2_end[i]);
      tr += ms;
    }
    info->ms_trailing = tr;
  }
  return st;
}

}  // namespace

extern "C" {

const char* exageo_strerror(exageo_status s) {
  switch (s) {
    case EXAGEO_OK: return "ok";
    case EXAGEO_EINVAL: return "invalid argument";
    case EXAGEO_ENOTPD: return "covariance matrix not positive definite";
    case EXAGEO_ENOMEM: return "out of device memory";
    case EXAGEO_ECUDA: return "CUDA error";
    case EXAGEO_ENCCL: return "NCCL error";
    case EXAGEO_EFIT: return "every optimizer evaluation failed";
  }
  return "unknown status";
}

const char* exageo_last_error(const exageo_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

exageo_status exageo_create(exageo_ctx** out, const exageo_opts* opts) {
  if (!out) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx pointer");
  *out = nullptr;
  exageo_opts o{};
  if (opts) o = *opts;
  if (o.nb != 0 && (o.nb < 128 || o.nb % 128 != 0))
    return fail(nullptr, EXAGEO_EINVAL, "nb must be 0 (auto) or a positive multiple of 128");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, EXAGEO_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (o.device < 0 || o.device >= ndev) return fail(nullptr, EXAGEO_EINVAL, "device ordinal out of range");
  exageo_ctx* c = new exageo_ctx();
  c->device = o.device;
  c->nb_opt = o.nb;
  auto bail = [&](cudaError_t err, const char* what) {
    g_create_err = std::string(what) + ": " + cudaGetErrorString(err);
    exageo_destroy(c);
    return EXAGEO_ECUDA;
  };
  if ((e = cudaSetDevice(o.device)) != cudaSuccess) return bail(e, "cudaSetDevice");
  if ((e = gemm_init()) != cudaSuccess) return bail(e, "gemm_init");
  if ((e = potrf_init()) != cudaSuccess) return bail(e, "potrf_init");
  if (o.stream) {
    c->stream = (cudaStream_t)o.stream;
  } else {
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess)
      return bail(e, "cudaStreamCreate");
    c->own_stream = true;
  }
  for (auto& ev : c->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return bail(e, "cudaEventCreate");
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = numerically smallest = highest priority
    if ((e = cudaStreamCreateWithPriority(&c->s_la, cudaStreamNonBlocking, hi)) != cudaSuccess)
      return bail(e, "cudaStreamCreateWithPriority");
    if ((e = cudaStreamCreateWithPriority(&c->s_main, cudaStreamNonBlocking, lo)) != cudaSuccess)
      return bail(e, "cudaStreamCreateWithPriority");
    for (cudaEvent_t* ev : {&c->ev_fork, &c->ev_F, &c->ev_U2, &c->ev_join[0], &c->ev_join[1]})
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
  }
  if ((e = cudaMalloc(&c->W, sizeof(double) * PB * PB)) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaMalloc(&c->out, sizeof(double) * kOutDoubles)) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaMalloc(&c->info, sizeof(int))) != cudaSuccess) return bail(e, "cudaMalloc");
  *out = c;
  return EXAGEO_OK;
}

void exageo_destroy(exageo_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->ws && !c->ws_external) cudaFree(c->ws);
  cudaFree(c->W);
  cudaFree(c->slots);
  cudaFree(c->out);
  cudaFree(c->info);
  cudaFree(c->vec);
  cudaFree(c->part);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {c->ev_fork, c->ev_F, c->ev_U2, c->ev_join[0], c->ev_join[1]})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->ev_u2_beg) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->ev_u2_end) cudaEventDestroy(ev);
  if (c->s_la) cudaStreamDestroy(c->s_la);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

size_t exageo_workspace_bytes(int64_t n, int nb) {
  if (n < 1) return 0;
  if (nb <= 0) nb = auto_nb(n);
  const Layout L = make_layout(n, nb);
  return (size_t)L.total() * sizeof(double) + 256 * sizeof(double);
}

exageo_status exageo_set_workspace(exageo_ctx* c, void* ptr, size_t bytes) {
  if (!c) return EXAGEO_EINVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->ws && !c->ws_external) cudaFree(c->ws);
  c->ws = (double*)ptr;
  c->ws_bytes = ptr ? bytes : 0;
  c->ws_external = ptr != nullptr;
  c->have_matrix = false;
  return EXAGEO_OK;
}

exageo_status exageo_gen_locations(int64_t n, uint64_t seed, double* x, double* y) {
  if (n < 1 || !x || !y) return fail(nullptr, EXAGEO_EINVAL, "n < 1 or NULL output");
  return gen_locations_host(n, seed, x, y) == 0 ? EXAGEO_OK : EXAGEO_EINVAL;
}

exageo_status exageo_matern_cov(exageo_ctx* c, const exageo_theta* t, int64_t m, const double* x1, const double* y1,
                                int64_t n, const double* x2, const double* y2, double* C, int64_t ldc) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  if (m < 1 || n < 1 || !x1 || !y1 || !x2 || !y2 || !C || ldc < m) return fail(c, EXAGEO_EINVAL, "bad sizes/pointers");
  CUDA_TRY(c, cudaSetDevice(c->device));
  double *d = nullptr;
  const size_t bytes = sizeof(double) * (2 * (size_t)m + 2 * (size_t)n + (size_t)m * (size_t)n);
  CUDA_TRY(c, cudaMalloc(&d, bytes));
  double *dx1 = d, *dy1 = d + m, *dx2 = d + 2 * m, *dy2 = d + 2 * m + n, *dC = d + 2 * m + 2 * n;
  cudaMemcpyAsync(dx1, x1, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(dy1, y1, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(dx2, x2, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(dy2, y2, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  launch_matern_dense(make_consts(*t), m, dx1, dy1, n, dx2, dy2, dC, m, c->stream);
  c->kernels += 1;
  cudaError_t e = cudaMemcpy2DAsync(C, sizeof(double) * ldc, dC, sizeof(double) * m, sizeof(double) * m, n,
                                    cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, EXAGEO_ECUDA, std::string("matern_cov: ") + cudaGetErrorString(e));
  return check_launch(c);
}

exageo_status exageo_loglik_dev(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                                const double* z, double* loglik, exageo_loglik_info* info) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return loglik_device(c, t, n, x, y, z, loglik, info);
}

exageo_status exageo_loglik(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                            const double* z, double* loglik, exageo_loglik_info* info) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (n < 1 || !x || !y || !z) return fail(c, EXAGEO_EINVAL, "n < 1 or NULL array");
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  CUDA_TRY(c, cudaSetDevice(c->device));
  exageo_status st = ensure_vec(c, n);
  if (st != EXAGEO_OK) return st;
  double *dx = c->vec, *dy = c->vec + n, *dz = c->vec + 2 * n;
  CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dz, z, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  return loglik_device(c, t, n, dx, dy, dz, loglik, info);
}

exageo_status exageo_simulate(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                              const double* e, double* z) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (n < 1 || !x || !y || !e || !z) return fail(c, EXAGEO_EINVAL, "n < 1 or NULL array");
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  CUDA_TRY(c, cudaSetDevice(c->device));
  exageo_status st = ensure_vec(c, n);
  if (st != EXAGEO_OK) return st;
  double *dx = c->vec, *dy = c->vec + n, *de = c->vec + 2 * n, *dz = c->vec + 3 * n;
  CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(de, e, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  st = do_generate(c, t, n, dx, dy, nullptr);
  if (st != EXAGEO_OK) return st;
  st = do_factor(c);
  if (st != EXAGEO_OK) return st;
  int info = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&info, c->info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (info > 0) return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(info - 1));
  const size_t need = sizeof(double) * (size_t)c->L.T * (size_t)c->L.N;
  if (c->part_cap < need) {
    cudaFree(c->part);
    c->part = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->part, need));
    c->part_cap = need;
  }
  launch_trmv_lower(c->L, c->ws, de, dz, c->part, c->stream);
  c->kernels += 2;
  st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemcpyAsync(z, dz, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EXAGEO_OK;
}

exageo_status exageo_stage_generate_dev(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x,
                                        const double* y, const double* z) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return do_generate(c, t, n, x, y, z);
}

exageo_status exageo_stage_factor(exageo_ctx* c) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return do_factor(c);
}

exageo_status exageo_stage_finish(exageo_ctx* c, double* out3, int64_t* pivot) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!c->have_matrix) return fail(c, EXAGEO_EINVAL, "no generated matrix in the workspace");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return do_finish(c, out3, pivot);
}

exageo_status exageo_read_lower(exageo_ctx* c, double* dst, int64_t ld) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!c->have_matrix || !dst || ld < c->L.n) return fail(c, EXAGEO_EINVAL, "no matrix or bad ld");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t n = c->L.n;
  double* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(double) * (size_t)n * (size_t)n));
  cudaMemsetAsync(d, 0, sizeof(double) * (size_t)n * (size_t)n, c->stream);
  launch_read_lower(c->L, c->ws, d, n, c->stream);
  cudaError_t e = cudaGetLastError();
  // copy only the lower triangle column by column would be slow; copy all and mask on host
  double* h = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (e == cudaSuccess && h)
    e = cudaMemcpyAsync(h, d, sizeof(double) * (size_t)n * (size_t)n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess || !h) {
    free(h);
    return fail(c, EXAGEO_ECUDA, std::string("read_lower: ") + cudaGetErrorString(e));
  }
  for (int64_t j = 0; j < n; ++j) memcpy(dst + j * ld + j, h + j * n + j, sizeof(double) * (size_t)(n - j));
  free(h);
  return EXAGEO_OK;
}

exageo_status exageo_read_zrow(exageo_ctx* c, double* dst) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!c->have_matrix || !dst) return fail(c, EXAGEO_EINVAL, "no matrix or NULL dst");
  CUDA_TRY(c, cudaSetDevice(c->device));
  exageo_status st = ensure_vec(c, c->L.n);
  if (st != EXAGEO_OK) return st;
  launch_read_zrow(c->L, c->ws, c->vec + 3 * c->L.n, c->stream);
  st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemcpyAsync(dst, c->vec + 3 * c->L.n, sizeof(double) * (size_t)c->L.n, cudaMemcpyDeviceToHost,
                              c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EXAGEO_OK;
}

exageo_status exageo_read_entries(exageo_ctx* c, int64_t count, const int64_t* rows, const int64_t* cols,
                                  double* out) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!c->have_matrix || count < 0 || (count > 0 && (!rows || !cols || !out)))
    return fail(c, EXAGEO_EINVAL, "no matrix or NULL arrays");
  if (count == 0) return EXAGEO_OK;
  for (int64_t i = 0; i < count; ++i)
    if (cols[i] < 0 || cols[i] > rows[i] || rows[i] >= c->L.n)
      return fail(c, EXAGEO_EINVAL, "entry outside the lower triangle");
  CUDA_TRY(c, cudaSetDevice(c->device));
  void* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(int64_t) * 2 * (size_t)count + sizeof(double) * (size_t)count));
  int64_t* drc = (int64_t*)d;
  double* dout = (double*)(drc + 2 * count);
  cudaError_t e = cudaMemcpyAsync(drc, rows, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(drc + count, cols, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    launch_read_entries(c->L, c->ws, count, drc, dout, c->stream);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, EXAGEO_ECUDA, std::string("read_entries: ") + cudaGetErrorString(e));
  return EXAGEO_OK;
}

}  // extern "C"
