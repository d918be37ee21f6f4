// api.cu -- the C ABI (include/exageo.h) and the device-side schedule of one
// log-likelihood evaluation (Alg. 2):
//
//   K1 gen_panels                       Sigma(theta) lower panels + z row   (l.2)
//   for k = 0 .. T-1                    right-looking tile Cholesky          (l.3)
//     F(k): for s = 0 .. nb/64 - 1      left-looking factorization of panel k
//       gemm_panel  (s > 0)             P[c0:, c0:c0+64] -= P[c0:, :c0] P[c0:c0+64, :c0]^T
//       potrf_block                     L_ss, W = L_ss^{-1}, sum log L_ii, pivot check
//       gemm_panel  (TRSM)              P[c0+64:, c0:c0+64] = P[c0+64:, c0:c0+64] W^T
//     broadcast panel k                 (world > 1: NCCL, or device copies for virtual ranks)
//     U1/U2: syrk_panels                A_ij -= L_ik L_jk^T on owned panels > k (incl. z row ->
//                                       forward solve of l.4)
//   local partials + all-reduce + combine                                 (l.5-7)
//
// Distribution: panels 1-D block-cyclic over `world` ranks; each rank
// stores its panels, receives panel k before its step-k update. Lookahead depth 1 on
// two prioritised streams per rank: the owner of panel k+1 updates it first (U1) and
// factors it (F(k+1)) while every rank applies the bulk update U2(k).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "context.h"
#include "nccl_dyn.h"

namespace exageo {
int gen_locations_host(int64_t n, uint64_t seed, double* x, double* y);
}

using namespace exageo;

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

#define NCCL_TRY(ctx, call)                                                                          \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess)                                                                           \
      return fail((ctx), EXAGEO_ENCCL, std::string(#call) + ": " + nccl::GetErrorString(r_));       \
  } while (0)

bool theta_ok(const exageo_theta* t) {
  return t && std::isfinite(t->sigma2) && std::isfinite(t->beta) && std::isfinite(t->nu) && t->sigma2 > 0 &&
         t->beta > 0 && t->nu > 0;
}

// Tile size by n (tools/nb_sweep.py on B200): small n is bound by the panel critical
// path (smaller tiles = shorter POTRF chains), large n by the trailing-update efficiency.
// automatic tile size (tools/nb_sweep.py with the current kernels: 128 up to 12k, then 256,
// 384 from 15k, 512 from 21k, 1024 from 48k: 1024 wins at 50/60/90/100k by 1.4-1.7% and
// loses at 70/80k by 0.3-0.6%; the differences near the other switches are 1-4%)
int auto_nb(int64_t n, int world = 1) {
  if (world > 1) return n >= 14000 ? 512 : (n >= 6000 ? 256 : 128);  // more panels balance the ranks
  // round-2 sweeps (tools/nb_sweep.py): with the 12.7 us K2 the longer panel chain of a wide
  // tile costs less than the wider trailing update gains (K = nb per DMMA tile):
  // 40k: 1024 647 ms vs 512 655; 60k-120k: 2048 best (100k: 9803 ms vs 9875 at 1024)
  // after the CUTLASS-mainloop trailing update: 8192 / 10k / 16k 512 best, 20k / 30k / 40k
  // 1024, 60k / 100k 2048 (100k: 9281 ms vs 9312 at 1536, 9373 at 1024)
  if (n >= 56000) return 2048;
  if (n >= 20000) return 1024;
  if (n >= 6000) return 512;
  return 128;
}

Layout make_layout(int64_t n, int nb, int rank = 0, int world = 1, int ind = 0, int P = 1) {
  Layout L;
  L.ind = ind;
  L.n = n;
  L.nb = nb;
  L.T = (int)((n + nb - 1) / nb);
  L.N = (int64_t)L.T * nb;
  L.rank = rank;
  L.world = world;
  L.P = P;
  L.Q = world / P;
  L.p = rank / L.Q;
  L.q = rank % L.Q;
  return L;
}

// Per-theta constants of Eq. (2), long double on the host.
MaternConsts make_consts(const exageo_theta& t, const exageo_ctx* ctx) {
  MaternConsts c{};
  c.metric = ctx->metric;
  c.radius = ctx->radius;
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

exageo_status check_launch(exageo_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, EXAGEO_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return EXAGEO_OK;
}

// Record a timing event: inside a stream capture it must become an event-record node of the
// graph (cudaEventRecordExternal); a plain record there would only mark a dependency.
cudaError_t record_timing(exageo_ctx* c, cudaEvent_t ev, cudaStream_t s) {
  return c->capturing ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal) : cudaEventRecord(ev, s);
}

exageo_status ensure_vec(exageo_ctx* c, int64_t n) {
  if (c->vec_cap >= n) return EXAGEO_OK;
  cudaFree(c->vec);
  cudaFree(c->zsum);
  c->vec = c->zsum = nullptr;
  c->vec_cap = 0;
  CUDA_TRY(c, cudaMalloc(&c->vec, sizeof(double) * 4 * (size_t)n));
  CUDA_TRY(c, cudaMalloc(&c->zsum, sizeof(double) * (size_t)n));
  c->vec_cap = n;
  return EXAGEO_OK;
}

size_t local_bytes(const Layout& L) { return (size_t)L.total() * sizeof(double) + 256 * sizeof(double); }

// bytes of the receive buffer for slice pp of a broadcast panel: the largest local panel of
// process row pp (panel 0)
size_t slice_bytes(const Layout& L, int pp) { return (size_t)L.ld_of(pp, 0) * L.nb * sizeof(double); }
size_t lkk_bytes(int nb) { return ((size_t)nb * nb + (size_t)64 * nb) * sizeof(double); }

cudaError_t alloc_or_fail(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

// Allocate (or check) every rank state's panel storage, receive buffers and slots.
exageo_status ensure_buffers(exageo_ctx* c) {
  size_t need_all = 0;
  for (auto& R : c->rs) {
    need_all += R.ws_external ? 0 : (R.ws_bytes >= local_bytes(R.L) ? 0 : local_bytes(R.L));
    if (c->world > 1)
      for (int pp = 0; pp < R.L.P; ++pp)
        if (R.recv_bytes[pp] < slice_bytes(R.L, pp)) need_all += 2 * slice_bytes(R.L, pp);
  }
  if (need_all > 0) {
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(c, cudaMemGetInfo(&free_b, &total_b));
    size_t reclaim = 0;
    for (auto& R : c->rs) {
      reclaim += R.ws_external ? 0 : R.ws_bytes;
      for (int pp = 0; pp < kMaxP; ++pp) reclaim += 2 * R.recv_bytes[pp];
    }
    if (need_all > free_b + reclaim)
      return fail(c, EXAGEO_ENOMEM,
                  "tile workspace needs " + std::to_string(need_all) + " bytes, " + std::to_string(free_b) + " free");
  }
  for (auto& R : c->rs) {
    const Layout& L = R.L;
    const int64_t nslots = (int64_t)L.owned() * (L.nb / PB);
    if (R.slots_cap < nslots || R.slots == nullptr) {
      cudaFree(R.slots);
      R.slots = nullptr;
      CUDA_TRY(c, cudaMalloc(&R.slots, sizeof(double) * (size_t)(nslots > 0 ? nslots : 1)));
      R.slots_cap = nslots;
    }
    if (R.ws_external) {
      if (R.ws_bytes < local_bytes(L))
        return fail(c, EXAGEO_ENOMEM, "external workspace too small: need " + std::to_string(local_bytes(L)));
    } else if (R.ws_bytes < local_bytes(L)) {
      cudaFree(R.ws);
      R.ws = nullptr;
      R.ws_bytes = 0;
      c->dag_init_key.clear();  // a new allocation may reuse the address with other contents
      cudaError_t e = alloc_or_fail((void**)&R.ws, local_bytes(L));
      if (e != cudaSuccess) return fail(c, EXAGEO_ENOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
      R.ws_bytes = local_bytes(L);
    }
    if (R.lkk_bytes < lkk_bytes(L.nb)) {
      for (auto& b : R.lkk) {
        cudaFree(b);
        b = nullptr;
      }
      R.lkk_bytes = 0;
      for (auto& b : R.lkk) {
        cudaError_t e = alloc_or_fail((void**)&b, lkk_bytes(L.nb));
        if (e != cudaSuccess) return fail(c, EXAGEO_ENOMEM, std::string("cudaMalloc L_kk buffer: ") + cudaGetErrorString(e));
      }
      R.lkk_bytes = lkk_bytes(L.nb);
    }
    if (c->world > 1) {
      for (int pp = 0; pp < L.P; ++pp) {
        const size_t rb = slice_bytes(L, pp);
        if (R.recv_bytes[pp] >= rb) continue;
        for (auto& b : R.recv) {
          cudaFree(b[pp]);
          b[pp] = nullptr;
        }
        R.recv_bytes[pp] = 0;
        for (auto& b : R.recv) {
          cudaError_t e = alloc_or_fail((void**)&b[pp], rb);
          if (e != cudaSuccess)
            return fail(c, EXAGEO_ENOMEM, std::string("cudaMalloc receive buffer: ") + cudaGetErrorString(e));
        }
        R.recv_bytes[pp] = rb;
      }
    }
  }
  return EXAGEO_OK;
}

// P > 1: the local panel offsets of rank state R (host table + device copy), from ld().
exageo_status set_offsets(exageo_ctx* c, RankState& R) {
  Layout& L = R.L;
  if (L.P == 1) {
    L.offs_h = L.offs_d = nullptr;
    return EXAGEO_OK;
  }
  std::vector<int64_t> o(L.owned() + 1, 0);
  for (int m = 0; m < L.owned(); ++m) o[m + 1] = o[m] + (int64_t)L.nb * L.ld(L.owned_panel(m));
  if (o != R.offs_h || R.offs_d == nullptr) {
    if (R.offs_cap < o.size()) {
      cudaFree(R.offs_d);
      R.offs_d = nullptr;
      CUDA_TRY(c, cudaMalloc(&R.offs_d, sizeof(int64_t) * o.size()));
      R.offs_cap = o.size();
    }
    CUDA_TRY(c, cudaMemcpy(R.offs_d, o.data(), sizeof(int64_t) * o.size(), cudaMemcpyHostToDevice));
    R.offs_h = o;
  }
  L.offs_h = R.offs_h.data();
  L.offs_d = R.offs_d;
  return EXAGEO_OK;
}

// ---------------------------------------------------------------------------- tile-task executor
// The whole factorization as one persistent kernel over the 64 x 64 tile DAG (dag.cu): used
// where the stream schedule is bound by its critical path and launch count (small n).
// Automatic crossover (tools/tile_tasks_timing.py); EXAGEO_TILE_TASKS_N overrides it.
int64_t tile_tasks_auto_n() {
  static const int64_t v = [] {
    const char* e = getenv("EXAGEO_TILE_TASKS_N");
    return e ? (int64_t)atoll(e) : (int64_t)3200;
  }();
  return v;
}

bool tile_tasks_eligible(const exageo_ctx* c, int64_t n) {
  if (c->tile_tasks < 0 || c->world > 1 || c->virt || c->ind > 0 || c->comm) return false;
  return c->tile_tasks > 0 || n <= tile_tasks_auto_n();
}

// Tail hand-off: when the stream schedule runs a single-rank factorization, its last panels
// (trailing size <= 2900) are bound by the panel chain -- each step's trailing update is
// shorter than F(k+1) -- so the executor factors that trailing matrix instead. Returns the
// first panel it takes (0: no hand-off). EXAGEO_TAIL_N overrides the size (0 disables).
int tail_stop(const exageo_ctx* c, const Layout& G) {
  if (c->tile_tasks < 0 || c->world > 1 || c->virt || c->ind > 0 || c->comm) return 0;
  if (tile_tasks_eligible(c, G.n)) return 0;  // the executor runs the whole factorization
  static const int64_t tail_n = [] {
    const char* e = getenv("EXAGEO_TAIL_N");
    return e ? (int64_t)atoll(e) : (int64_t)2900;  // sweeps: 8192 best at 2560 rows, 10k at 2832 (profiles/r02_tail_sweep.txt)
  }();
  if (tail_n <= 0) return 0;
  int k = (int)((G.n - tail_n + G.nb - 1) / G.nb);  // first panel whose trailing size <= tail_n
  if (k < 1) k = 1;
  return k < G.T ? k : 0;
}

// Plan (host list schedule, cached by nt and the CTA count) and buffers for the executor run
// of this layout: the whole matrix (t0 = 0) or the trailing matrix from 64-block column t0.
exageo_status prepare_tile_tasks(exageo_ctx* c, int t0 = 0) {
  const Layout& G = c->G;
  const int nt = (int)((G.n + PB - 1) / PB) - t0;
  c->dag_t0 = t0;
  int nsm = 0;
  CUDA_TRY(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  if (c->dag_nt != nt || c->dag_nproc != nsm || c->dag_plan_t0 != t0) {
    std::vector<int4> order;
    dag_plan(nt, nsm, order);
    if ((int64_t)order.size() > c->dag_cap_tasks) {
      cudaFree(c->dag_tasks);
      c->dag_tasks = nullptr;
      c->dag_cap_tasks = 0;
      CUDA_TRY(c, cudaMalloc(&c->dag_tasks, sizeof(int4) * order.size()));
      c->dag_cap_tasks = (int64_t)order.size();
    }
    CUDA_TRY(c, cudaMemcpy(c->dag_tasks, order.data(), sizeof(int4) * order.size(), cudaMemcpyHostToDevice));
    const int64_t ntr = (int64_t)order.size() + 3 * (int64_t)nt;  // + the chain CTA's records
    if (!c->dag_trace_path.empty() && c->dag_trace_cap < ntr) {
      cudaFree(c->dag_trace);
      c->dag_trace = nullptr;
      c->dag_trace_cap = 0;
      CUDA_TRY(c, cudaMalloc(&c->dag_trace, sizeof(unsigned long long) * 4 * ntr));
      c->dag_trace_cap = ntr;
    }
    c->dag_ntasks = (int)order.size();
    c->dag_nt = nt;
    c->dag_nproc = nsm;
    c->dag_plan_t0 = t0;
  }
  if (c->dag_cap_nt < nt) {
    cudaFree(c->dag_sync);
    cudaFree(c->dag_W);
    c->dag_sync = nullptr;
    c->dag_W = nullptr;
    c->dag_cap_nt = 0;
    CUDA_TRY(c, cudaMalloc(&c->dag_sync, sizeof(int) * (size_t)dag_sync_ints(nt)));
    CUDA_TRY(c, cudaMemset(c->dag_sync, 0, sizeof(int) * (size_t)dag_sync_ints(nt)));
    CUDA_TRY(c, cudaMalloc(&c->dag_W, sizeof(double) * (size_t)nt * PB * PB));
    c->dag_cap_nt = nt;
  }
  return EXAGEO_OK;
}

// ---------------------------------------------------------------------------- generation
// Validate, set the layouts for n and make sure every buffer exists (no launches).
exageo_status prepare_generate(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y) {
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  if (n < 1 || !x || !y) return fail(c, EXAGEO_EINVAL, "n < 1 or NULL location array");
  const int nb = c->nb_opt > 0 ? c->nb_opt : auto_nb(n, c->world);
  c->G = make_layout(n, nb, 0, 1, c->ind);
  for (size_t i = 0; i < c->rs.size(); ++i) {
    const int rank = c->virt ? (int)i : c->rank;
    c->rs[i].L = make_layout(n, nb, rank, c->world, c->ind, c->P);
    exageo_status st = set_offsets(c, c->rs[i]);
    if (st != EXAGEO_OK) return st;
  }
  exageo_status st = ensure_buffers(c);
  if (st != EXAGEO_OK) return st;
  // the tile-task plan and buffers exist before any launch (and outside graph capture)
  if (const int ks = tail_stop(c, c->G)) return prepare_tile_tasks(c, ks * (nb / PB));
  if (!tile_tasks_eligible(c, n)) return EXAGEO_OK;
  if ((st = prepare_tile_tasks(c)) != EXAGEO_OK) return st;
  // the executor generates only the tiles inside n; the rest of the layout (identity padding,
  // the z block's zero rows) is theta-independent: generated once per workspace and layout
  const std::vector<const void*> key = {c->rs[0].ws, (const void*)(intptr_t)n, (const void*)(intptr_t)nb};
  if (c->dag_init_key != key) {
    const MaternConsts mc = make_consts(*t, c);
    launch_matern_table(mc, c->mtab, c->stream);
    launch_gen_panels(c->rs[0].L, c->rs[0].ws, mc, x, y, nullptr, c->mtab, c->stream);
    if ((st = check_launch(c)) != EXAGEO_OK) return st;
    c->dag_init_key = key;
  }
  return EXAGEO_OK;
}

exageo_status launch_generate(exageo_ctx* c, const MaternConsts& mc, const double* x, const double* y,
                              const double* z, bool defer = false) {
  const int tab = launch_matern_table(mc, c->mtab, c->stream);
  c->kernels += tab;
  c->gen_launches += tab;
  if (defer && tile_tasks_eligible(c, c->G.n)) {
    // Alg. 2 l.2 fused into the executor (its GEN tasks, ahead of the factorization's tasks)
    CUDA_TRY(c, cudaMemsetAsync(c->rs[0].info, 0, sizeof(int), c->stream));
    c->dag_gen = true;
    c->dag_mc = mc;
    c->dag_x = x;
    c->dag_y = y;
    c->dag_z = z;
    c->have_matrix = true;
    c->dag_finished = false;
    return check_launch(c);
  }
  c->dag_gen = false;
  for (auto& R : c->rs) {
    CUDA_TRY(c, cudaMemsetAsync(R.info, 0, sizeof(int), c->stream));
    if (R.L.P > 1)  // only the diagonal ranks write log-det slots (the others' stay zero)
      CUDA_TRY(c, cudaMemsetAsync(R.slots, 0, sizeof(double) * (size_t)R.L.owned() * (R.L.nb / PB), c->stream));
    launch_gen_panels(R.L, R.ws, mc, x, y, z, c->mtab, c->stream);
    c->kernels += 1;
    c->gen_launches += 1;
  }
  c->have_matrix = true;
  c->dag_finished = false;
  return check_launch(c);
}

// defer: the caller factors next (loglik, simulate, predict), so the executor may generate
exageo_status do_generate(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                          const double* z, bool defer = false) {
  exageo_status st = prepare_generate(c, t, n, x, y);
  if (st != EXAGEO_OK) return st;
  return launch_generate(c, make_consts(*t, c), x, y, z, defer);
}

// ---------------------------------------------------------------------------- factorization
// W_s = L_ss^{-1} of 64-block sb of panel k (written by F(k) on the diagonal rank, broadcast with
// L_kk down the process column for the other ranks' TRSM)
double* w_block(RankState& R, int k, int sb) {
  return R.lkk[k & 1] + (size_t)R.L.nb * R.L.nb + (size_t)sb * PB * PB;
}

// Factor local panel k on its diagonal rank (over PB-wide column blocks, right- or left-looking:
// panel_right_looking) on s:
// the diagonal tile is the top of the local panel, every row below (the rank's other tile rows
// of column k and the z row block, if stored here) gets the panel update and the TRSM.
// Right-looking inside the panel: after block sb's POTRF and TRSM one wide K = 64 update of all
// later column blocks, instead of each block's left-looking update with K = 64 sb on M / 64
// CTAs. Shorter panel chain where it is the critical path (n <= 24000: 8192 7.97 -> 7.64 ms,
// 10k 13.02 -> 12.72, 20k 83.6 -> 82.6); above, its wide launches take SMs from the concurrent
// bulk update (100k 9.26 -> 9.36 s), so the left-looking form stays. EXAGEO_PANEL_RIGHT=0/1 forces.
bool panel_right_looking(int64_t n) {
  static const int forced = [] {
    const char* e = getenv("EXAGEO_PANEL_RIGHT");
    return e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }();
  return forced >= 0 ? forced == 1 : n <= 24000;
}

exageo_status factor_panel(exageo_ctx* c, RankState& R, int k, cudaStream_t s) {
  const bool right = panel_right_looking(R.L.n);
  const Layout& L = R.L;
  const int nsub = L.nb / PB;
  double* Pk = R.ws + L.off(k);
  const int64_t ldk = L.ld(k);
  const int m = (k - L.q) / L.Q;  // local panel index
  for (int sb = 0; sb < nsub; ++sb) {
    const int64_t c0 = (int64_t)sb * PB;
    if ((int64_t)k * L.nb + c0 >= L.n) {
      // the rest of the (last) panel is identity padding (R12): generated as I with zero
      // rows/columns around it and never touched by an update, it already is its own factor
      // (L = I, log L_ii = 0) -- skip its POTRF/TRSM/GEMM launches
      CUDA_TRY(c, cudaMemsetAsync(R.slots + (int64_t)m * nsub + sb, 0, sizeof(double) * (nsub - sb), s));
      break;
    }
    // at small n the panel chain is the critical path: its kernels use programmatic
    // dependent launch (each launches while its predecessor runs and waits on the device)
    const bool pdl = L.n <= 32768;
    const bool first = sb == 0;  // follows U1 / an event wait: ordinary launch
    if (sb > 0 && !right) {
      launch_gemm_panel(ldk - c0, PB, (int)c0, Pk + c0, ldk, Pk + c0, ldk, Pk + c0 * ldk + c0, ldk, true, R.info, s,
                        pdl);
      c->kernels += 1;
    }
    double* W = w_block(R, k, sb);
    launch_potrf_block(Pk + c0 * ldk + c0, ldk, W, R.slots + (int64_t)m * nsub + sb, R.info, (int64_t)k * L.nb + c0,
                       s, pdl && !first, (int)std::min<int64_t>(PB, L.n - ((int64_t)k * L.nb + c0)));
    double* below = Pk + c0 * ldk + c0 + PB;
    launch_gemm_panel(ldk - c0 - PB, PB, PB, below, ldk, W, PB, below, ldk, false, R.info, s, pdl);
    c->kernels += 2;
    if (right) {  // the panel's later column blocks (inside n) -= L(:, block sb) L(rows of those blocks, block sb)^T
      const int64_t cols_left = std::min<int64_t>(L.nb, L.n - (int64_t)k * L.nb) - (c0 + PB);
      if (cols_left > 0) {
        launch_gemm_panel(ldk - c0 - PB, (int)((cols_left + PB - 1) / PB * PB), PB, below, ldk, below, ldk,
                          Pk + (c0 + PB) * ldk + c0 + PB, ldk, true, R.info, s, pdl);
        c->kernels += 1;
      }
    }
  }
  return EXAGEO_OK;
}

// Text trace of the last executor run: one line per ticket "t type i j k cta grab ready done"
// (times in ns from the first grab).
void dump_tile_task_trace(exageo_ctx* c) {
  const int ntr = c->dag_ntasks + 3 * c->dag_nt;
  std::vector<unsigned long long> tr((size_t)4 * ntr);
  std::vector<int4> tk(ntr);
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(tr.data(), c->dag_trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(tk.data(), c->dag_tasks, sizeof(int4) * c->dag_ntasks, cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  for (int k = 0; k < c->dag_nt; ++k) {  // chain CTA: POTRF(k), TRSM(k+1, k), SYRK(k+1, k+1, k)
    tk[c->dag_ntasks + 3 * k] = make_int4(0, k, k, k);
    tk[c->dag_ntasks + 3 * k + 1] = make_int4(1, k + 1, k, k);
    tk[c->dag_ntasks + 3 * k + 2] = make_int4(2, k + 1, k + 1, k);
  }
  FILE* f = fopen(c->dag_trace_path.c_str(), "w");
  if (!f) return;
  unsigned long long t0 = ~0ull;
  for (int t = 0; t < ntr; ++t)
    if (tr[4 * t + 1] && tr[4 * t + 1] < t0) t0 = tr[4 * t + 1];
  fprintf(f, "# ticket type i j k cta grab_ns ready_ns done_ns (n=%lld nt=%d)\n", (long long)c->G.n, c->dag_nt);
  for (int t = 0; t < ntr; ++t)
    fprintf(f, "%d %d %d %d %d %llu %lld %lld %lld\n", t, tk[t].x, tk[t].y, tk[t].z, tk[t].w, tr[4 * t],
            (long long)(tr[4 * t + 1] - t0), (long long)(tr[4 * t + 2] - t0), (long long)(tr[4 * t + 3] - t0));
  fclose(f);
}

exageo_status factor_tile_tasks(exageo_ctx* c) {
  if (c->dag_nt != (int)((c->G.n + PB - 1) / PB) - c->dag_t0 || c->dag_cap_nt < c->dag_nt)
    return fail(c, EXAGEO_EINVAL, "tile-task plan missing (prepare_generate)");
  RankState& R = c->rs[0];
  const Layout& L = R.L;
  // the counters are zero: set at allocation, reset by the last CTA of every launch
  if (c->dag_t0 == 0) {
    R.n_u2 = 0;
    R.u2_flops = 0.0;
    R.n_u1 = 0;
    R.u1_flops = 0.0;
  }
  const int nctas = 1 + std::min(c->dag_nproc - 1, std::max(c->dag_ntasks, 1));  // chain CTA + pool
  DagGen g{c->dag_gen, c->dag_mc, c->mtab, c->dag_x, c->dag_y, c->dag_z};
  launch_dag_factor(L, R.ws, c->dag_tasks, c->dag_ntasks, c->dag_nt, c->dag_t0, c->dag_sync, c->dag_W, R.slots, R.info,
                    c->out3, c->dag_res, c->dag_trace, g, nctas, c->stream);
  c->kernels += 1;
  if (c->dag_gen) c->gen_launches += 1;
  c->dag_gen = false;  // one generation per launch_generate
  c->dag_finished = true;
  return check_launch(c);
}

// P > 1: the other ranks of panel k's process column apply F(k)'s column operations to their
// tile rows with the received L_kk and W_s (lkk[k % 2]): for each 64-block s, the left-looking
// update A_s -= A_{<s} L_kk[s, <s]^T, then A_s <- A_s W_s^T (the TRSM of Fig. 2 by the inverse).
exageo_status trsm_panel(exageo_ctx* c, RankState& R, int k, cudaStream_t s) {
  const Layout& L = R.L;
  const int nsub = L.nb / PB;
  double* Pk = R.ws + L.off(k);
  const int64_t ldk = L.ld(k);
  const double* Lkk = R.lkk[k & 1];
  if (ldk <= 0) return EXAGEO_OK;
  for (int sb = 0; sb < nsub; ++sb) {
    const int64_t c0 = (int64_t)sb * PB;
    if ((int64_t)k * L.nb + c0 >= L.n) break;  // identity padding: no-op (R12)
    if (sb > 0) {
      launch_gemm_panel(ldk, PB, (int)c0, Pk, ldk, Lkk + c0, L.nb, Pk + c0 * ldk, ldk, true, R.info, s);
      c->kernels += 1;
    }
    launch_gemm_panel(ldk, PB, PB, Pk + c0 * ldk, ldk, w_block(R, k, sb), PB, Pk + c0 * ldk, ldk, false, R.info, s);
    c->kernels += 1;
  }
  return EXAGEO_OK;
}

RankState* local_state(exageo_ctx* c, int rank) {
  if (c->virt) return &c->rs[rank];
  return rank == c->rank ? &c->rs[0] : nullptr;
}

// Operands of panel k on rank state R: slice pp = the local panel k of rank (pp, k mod Q) --
// R's own storage when R is that rank, else the received copy.
void panel_slices(RankState& R, int k, const double** sl, int64_t* sld) {
  const Layout& L = R.L;
  for (int pp = 0; pp < L.P; ++pp) {
    sl[pp] = (L.owns(k) && pp == L.p) ? R.ws + L.off(k) : R.recv[k & 1][pp];
    sld[pp] = L.ld_of(pp, k);
  }
}

// algorithmic flops of updating local panels J0, J0 + Q, ... (npan) by one panel: 2 nb per
// (row, column) pair of the true lower triangle stored on this rank, plus the z row
double update_flops(const Layout& L, int k, int J0, int npan) {
  double f = 0.0;
  const int E = L.sb_end(k);
  for (int i = 0; i < npan; ++i) {
    const int J = J0 + i * L.Q;
    const int64_t c0 = (int64_t)J * L.nb;
    const int64_t c1 = (c0 + L.nb) < L.n ? (c0 + L.nb) : L.n;
    if (c1 <= c0) continue;
    for (int I = J; I < E; ++I) {
      if (I % L.P != L.p) continue;
      const int64_t r0 = (int64_t)I * L.nb, r1 = (r0 + L.nb) < L.n ? (r0 + L.nb) : L.n;
      if (r1 <= r0) continue;
      if (I > J) {
        f += 2.0 * L.nb * (double)(r1 - r0) * (double)(c1 - c0);
      } else {  // diagonal tile: pairs r >= c
        for (int64_t cc = c0; cc < c1; ++cc) f += 2.0 * L.nb * (double)(r1 - cc);
      }
    }
    if (L.has_z()) f += 2.0 * L.nb * (double)(c1 - c0);
  }
  return f;
}

ncclComm_t row_comm(const exageo_ctx* c) { return c->P == 1 ? c->comm : c->comm_row; }

// Make panel j (factored on its process column) available to every rank:
//   (a) P > 1: the diagonal rank broadcasts [L_jj | W_s] down process column j mod Q; the other
//       ranks of that column apply the column operations of F(j) to their tile rows (trsm_panel);
//   (b) each rank of process column j mod Q broadcasts its local panel j along its process row;
//   (c) P > 1: every rank re-broadcasts the slice of its process row down its process column,
//       so each rank holds all P slices (the rows of its tile rows and of its tile columns).
// NCCL on the row / column communicators, or device copies between virtual ranks. Buffers of
// parity j % 2 were last read by U1(j-2) / U2(j-2) (and L_kk by trsm(j-2)): those events gate
// the overwrite. Records ev_recv[j % 2] on every rank's s_comm.
exageo_status exchange_panel(exageo_ctx* c, int j) {
  if (c->world == 1 && !c->comm) return EXAGEO_OK;
  const Layout& G = c->G;
  const int P = c->P, Q = c->Q, qj = j % Q, pj = j % P;
  const size_t nbd = (size_t)G.nb;
  const size_t lkk_count = nbd * nbd + 64 * nbd;
  if (!c->virt) {
    RankState& R = c->rs[0];
    const Layout& L = R.L;
    const bool incol = L.owns(j);
    if (j >= 2) {  // release the parity-(j % 2) buffers
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_U2[j & 1], 0));
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_U1[j & 1], 0));
    }
    if (P > 1 && incol) {  // (a)
      double* buf = R.lkk[j & 1];
      if (L.diag(j)) {
        CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_F, 0));
        CUDA_TRY(c, cudaMemcpy2DAsync(buf, nbd * sizeof(double), R.ws + L.off(j), (size_t)L.ld(j) * sizeof(double),
                                      nbd * sizeof(double), nbd, cudaMemcpyDeviceToDevice, R.s_comm));
      }
      NCCL_TRY(c, nccl::Broadcast(buf, buf, lkk_count, ncclDouble, pj, c->comm_col, R.s_comm));
      if (!L.diag(j)) {
        CUDA_TRY(c, cudaEventRecord(R.ev_lkk, R.s_comm));
        CUDA_TRY(c, cudaStreamWaitEvent(R.s_la, R.ev_lkk, 0));
        exageo_status st = trsm_panel(c, R, j, R.s_la);
        if (st != EXAGEO_OK) return st;
        CUDA_TRY(c, cudaEventRecord(R.ev_F, R.s_la));
      }
    }
    double* own = incol ? R.ws + L.off(j) : R.recv[j & 1][L.p];
    if (incol) CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_F, 0));
    if (Q > 1 || P == 1)  // (b); with world 1 and a communicator: exercises the NCCL path
      NCCL_TRY(c, nccl::Broadcast(own, own, (size_t)L.ld(j) * nbd, ncclDouble, qj, row_comm(c), R.s_comm));
    if (P > 1) {  // (c)
      NCCL_TRY(c, nccl::GroupStart());
      for (int pp = 0; pp < P; ++pp) {
        double* buf = pp == L.p ? own : R.recv[j & 1][pp];
        NCCL_TRY(c, nccl::Broadcast(buf, buf, (size_t)L.ld_of(pp, j) * nbd, ncclDouble, pp, c->comm_col, R.s_comm));
      }
      NCCL_TRY(c, nccl::GroupEnd());
    }
    CUDA_TRY(c, cudaEventRecord(R.ev_recv[j & 1], R.s_comm));
    return EXAGEO_OK;
  }
  // virtual ranks: the same data movement as device copies, ordered by events
  auto rid = [&](int pp, int qq) { return pp * Q + qq; };
  for (auto& R : c->rs)
    if (j >= 2) {
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_U2[j & 1], 0));
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, R.ev_U1[j & 1], 0));
    }
  if (P > 1) {  // (a)
    RankState& D = c->rs[rid(pj, qj)];
    CUDA_TRY(c, cudaStreamWaitEvent(D.s_comm, D.ev_F, 0));
    CUDA_TRY(c, cudaMemcpy2DAsync(D.lkk[j & 1], nbd * sizeof(double), D.ws + D.L.off(j),
                                  (size_t)D.L.ld(j) * sizeof(double), nbd * sizeof(double), nbd,
                                  cudaMemcpyDeviceToDevice, D.s_comm));
    CUDA_TRY(c, cudaEventRecord(D.ev_lkk, D.s_comm));
    for (int pp = 0; pp < P; ++pp) {
      if (pp == pj) continue;
      RankState& R = c->rs[rid(pp, qj)];
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, D.ev_lkk, 0));
      CUDA_TRY(c, cudaMemcpyAsync(R.lkk[j & 1], D.lkk[j & 1], lkk_count * sizeof(double), cudaMemcpyDeviceToDevice,
                                  R.s_comm));
      CUDA_TRY(c, cudaEventRecord(R.ev_lkk, R.s_comm));
      CUDA_TRY(c, cudaStreamWaitEvent(D.s_comm, R.ev_lkk, 0));  // D's buffer is free again after this copy
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_la, R.ev_lkk, 0));
      exageo_status st = trsm_panel(c, R, j, R.s_la);
      if (st != EXAGEO_OK) return st;
      CUDA_TRY(c, cudaEventRecord(R.ev_F, R.s_la));
    }
  }
  // (b) row copies: rank (p, q != qj) receives the local panel j of rank (p, qj)
  for (auto& R : c->rs) {
    const Layout& L = R.L;
    if (L.owns(j)) continue;
    RankState& S = c->rs[rid(L.p, qj)];
    CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, S.ev_F, 0));
    CUDA_TRY(c, cudaMemcpyAsync(R.recv[j & 1][L.p], S.ws + S.L.off(j), (size_t)L.ld(j) * nbd * sizeof(double),
                                cudaMemcpyDeviceToDevice, R.s_comm));
    CUDA_TRY(c, cudaEventRecord(R.ev_row, R.s_comm));
  }
  // (c) column copies: rank (p, q) receives slice pp from rank (pp, q)
  if (P > 1) {
    for (auto& R : c->rs) {
      const Layout& L = R.L;
      for (int pp = 0; pp < P; ++pp) {
        if (pp == L.p) continue;
        RankState& S = c->rs[rid(pp, L.q)];
        const double* src = S.L.owns(j) ? S.ws + S.L.off(j) : S.recv[j & 1][pp];
        CUDA_TRY(c, cudaStreamWaitEvent(R.s_comm, S.L.owns(j) ? S.ev_F : S.ev_row, 0));
        CUDA_TRY(c, cudaMemcpyAsync(R.recv[j & 1][pp], src, (size_t)L.ld_of(pp, j) * nbd * sizeof(double),
                                    cudaMemcpyDeviceToDevice, R.s_comm));
      }
    }
    // a source's slice buffer may be refilled (step j + 2) only after its column peers copied it
    for (auto& R : c->rs) CUDA_TRY(c, cudaEventRecord(R.ev_row, R.s_comm));
    for (auto& S : c->rs)
      for (int pp = 0; pp < P; ++pp)
        if (pp != S.L.p) CUDA_TRY(c, cudaStreamWaitEvent(S.s_comm, c->rs[rid(pp, S.L.q)].ev_row, 0));
  }
  for (auto& R : c->rs) CUDA_TRY(c, cudaEventRecord(R.ev_recv[j & 1], R.s_comm));
  return EXAGEO_OK;
}

// Right-looking tile Cholesky with depth-1 lookahead (the paper's "updates of the
// trailing submatrix may be triggered before the current panel factorization is
// complete"), as prioritised CUDA streams instead of a runtime DAG:
//   s_la  (high priority): on the ranks of panel k+1's process column, U1(k) = update of
//                          local panel k+1 by panel k, then F(k+1) on its diagonal rank
//                          (trsm_panel on the others, in exchange_panel)
//   s_main (low priority): U2(k) = update of the rank's other local panels > k by panel k
//   s_comm:                exchange of panel k+1 once factored
// Dependencies: U1(k) after U2(k-1) and panel k; U2(k) after panel k. F(k+1) and the
// exchange overlap U2(k).
exageo_status do_factor(exageo_ctx* c) {
  if (!c->have_matrix) return fail(c, EXAGEO_EINVAL, "no generated matrix in the workspace");
  const Layout& G = c->G;
  if (tile_tasks_eligible(c, G.n)) return factor_tile_tasks(c);
  c->dag_finished = false;
  const int kstop = tail_stop(c, G);  // > 0: panels >= kstop go to the executor
  CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
  for (auto& R : c->rs) {
    for (cudaStream_t s : {R.s_la, R.s_main, R.s_comm}) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_fork, 0));
    R.n_u2 = 0;
    R.u2_flops = 0.0;
    R.n_u1 = 0;
    R.u1_flops = 0.0;
  }
  exageo_status st;
  for (auto& R : c->rs)
    if (R.L.diag(0)) {
      if ((st = factor_panel(c, R, 0, R.s_la)) != EXAGEO_OK) return st;
      CUDA_TRY(c, cudaEventRecord(R.ev_F, R.s_la));
    }
  if ((st = exchange_panel(c, 0)) != EXAGEO_OK) return st;
  for (int k = 0; k + 1 < (kstop > 0 ? kstop + 1 : G.T); ++k) {
    for (auto& R : c->rs) {
      const Layout& L = R.L;
      const double* sl[kMaxP];
      int64_t sld[kMaxP];
      panel_slices(R, k, sl, sld);
      // panel k's operands: the rank's own factored panel (1-D owner) or the exchange
      cudaEvent_t avail = (L.P == 1 && L.owns(k)) ? R.ev_F : R.ev_recv[k & 1];
      // at the hand-off step the bulk update also covers panel k + 1 (no U1 / F(k + 1))
      const bool owns_next = L.owns(k + 1) && k + 1 != kstop;
      // U2(k) needs panel k: wait now, before ev_F is re-recorded for F(k+1) below
      CUDA_TRY(c, cudaStreamWaitEvent(R.s_main, avail, 0));
      if (owns_next) {
        CUDA_TRY(c, cudaStreamWaitEvent(R.s_la, avail, 0));
        if (k > 0) CUDA_TRY(c, cudaStreamWaitEvent(R.s_la, R.ev_U2[(k - 1) & 1], 0));
        if (k + 1 < L.sb_end(k)) {  // (IND: panel k+1 opens a new super tile: no update)
          if ((int)R.u1b.size() <= R.n_u1) {
            cudaEvent_t b, e;
            CUDA_TRY(c, cudaEventCreate(&b));
            CUDA_TRY(c, cudaEventCreate(&e));
            R.u1b.push_back(b);
            R.u1e.push_back(e);
          }
          CUDA_TRY(c, record_timing(c, R.u1b[R.n_u1], R.s_la));
          if (L.P == 1) launch_syrk_panels(L, R.ws, sl[0], k, k + 1, 1, R.info, R.s_la);  // U1(k)
          else launch_syrk_panels_2d(L, R.ws, sl, sld, k, k + 1, 1, R.info, R.s_la);
          CUDA_TRY(c, record_timing(c, R.u1e[R.n_u1], R.s_la));
          ++R.n_u1;
          R.u1_flops += update_flops(L, k, k + 1, 1);
          c->kernels += 1;
        }
        CUDA_TRY(c, cudaEventRecord(R.ev_U1[k & 1], R.s_la));
        if (L.diag(k + 1)) {
          if ((st = factor_panel(c, R, k + 1, R.s_la)) != EXAGEO_OK) return st;  // F(k+1)
          CUDA_TRY(c, cudaEventRecord(R.ev_F, R.s_la));
        }
      } else {
        CUDA_TRY(c, cudaEventRecord(R.ev_U1[k & 1], R.s_la));  // nothing read on s_la this step
      }
      // local panels updated by panel k: up to the end of k's diagonal super tile (T when exact)
      const int Jend = L.sb_end(k);
      const int J0 = L.first_owned_from(owns_next ? k + 2 : k + 1);
      const int npan = J0 < Jend ? (Jend - 1 - J0) / L.Q + 1 : 0;
      if (npan > 0) {
        if ((int)R.u2b.size() <= R.n_u2) {
          cudaEvent_t b, e;
          CUDA_TRY(c, cudaEventCreate(&b));
          CUDA_TRY(c, cudaEventCreate(&e));
          R.u2b.push_back(b);
          R.u2e.push_back(e);
        }
        CUDA_TRY(c, record_timing(c, R.u2b[R.n_u2], R.s_main));
        if (L.P == 1) launch_syrk_panels(L, R.ws, sl[0], k, J0, npan, R.info, R.s_main);  // U2(k)
        else launch_syrk_panels_2d(L, R.ws, sl, sld, k, J0, npan, R.info, R.s_main);
        CUDA_TRY(c, record_timing(c, R.u2e[R.n_u2], R.s_main));
        ++R.n_u2;
        R.u2_flops += update_flops(L, k, J0, npan);
        c->kernels += 1;
      }
      CUDA_TRY(c, cudaEventRecord(R.ev_U2[k & 1], R.s_main));
    }
    if ((st = exchange_panel(c, k + 1)) != EXAGEO_OK) return st;
  }
  for (auto& R : c->rs) {
    CUDA_TRY(c, cudaEventRecord(R.ev_join[0], R.s_la));
    CUDA_TRY(c, cudaEventRecord(R.ev_join[1], R.s_main));
    CUDA_TRY(c, cudaEventRecord(R.ev_join[2], R.s_comm));
    for (auto& ev : R.ev_join) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ev, 0));
  }
  if (kstop > 0) {  // the trailing matrix from panel kstop on: one executor launch (dag.cu)
    st = check_launch(c);
    if (st != EXAGEO_OK) return st;
    return factor_tile_tasks(c);
  }
  return check_launch(c);
}

// ---------------------------------------------------------------------------- reductions
// First failing global pivot over all ranks (-1 if none). Synchronises.
exageo_status first_pivot(exageo_ctx* c, int64_t* pivot) {
  int64_t best = std::numeric_limits<int64_t>::max();
  for (auto& R : c->rs) {
    int info = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&info, R.info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (info > 0 && (int64_t)info - 1 < best) best = (int64_t)info - 1;
  }
  if (c->comm) {
    CUDA_TRY(c, cudaMemcpyAsync(c->pivbuf, &best, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(c, nccl::AllReduce(c->pivbuf, c->pivbuf, 1, ncclInt64, ncclMin, c->comm, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&best, c->pivbuf, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  *pivot = best == std::numeric_limits<int64_t>::max() ? -1 : best;
  return EXAGEO_OK;
}

// Launch the log-det / dot reductions and the combination into c->out3 (no host sync).
exageo_status launch_finish(exageo_ctx* c) {
  if (c->dag_finished) return EXAGEO_OK;  // the tile-task kernel wrote out3 itself
  for (size_t i = 0; i < c->rs.size(); ++i) {
    RankState& R = c->rs[i];
    launch_local_partials(R.L, R.ws, R.slots, R.L.owned() * (R.L.nb / PB), R.scratch, c->parts + 2 * i, c->stream);
    c->kernels += 2;
  }
  int nparts = (int)c->rs.size();
  if (c->comm) {
    NCCL_TRY(c, nccl::AllReduce(c->parts, c->parts, 2, ncclDouble, ncclSum, c->comm, c->stream));
    nparts = 1;
  }
  launch_combine(c->parts, nparts, c->G.n, c->out3, c->stream);
  c->kernels += 1;
  return check_launch(c);
}

exageo_status do_finish(exageo_ctx* c, double* out3, int64_t* pivot) {
  exageo_status st = launch_finish(c);
  if (st != EXAGEO_OK) return st;
  double h[3];
  CUDA_TRY(c, cudaMemcpyAsync(h, c->out3, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  int64_t piv = -1;
  st = first_pivot(c, &piv);  // synchronises
  if (st != EXAGEO_OK) return st;
  if (pivot) *pivot = piv;
  if (piv >= 0) {
    if (out3) {
      out3[0] = -std::numeric_limits<double>::infinity();
      out3[1] = out3[2] = std::numeric_limits<double>::quiet_NaN();
    }
    return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(piv));
  }
  if (out3) memcpy(out3, h, sizeof(h));
  return EXAGEO_OK;
}

// ---------------------------------------------------------------------------- CUDA graphs
// One evaluation (K1 .. K6 and the result copies) is captured once per problem shape and
// buffer set and replayed; only theta changes between replays, and it lives in the K1
// nodes' MaternConsts argument, rewritten with cudaGraphExecKernelNodeSetParams. This
// removes the per-launch host overhead and the launch gaps of the ~8 launches per panel
// that dominate small n (the MLE loop evaluates the same shape hundreds of times).
bool graph_eligible(const exageo_ctx* c, int64_t n) {
  // NCCL contexts too: NCCL collectives are captured as graph nodes (every rank captures and
  // replays the same SPMD sequence); the pivot all-reduce is part of the graph (graph_body)
  if (c->graphs < 0) return false;
  if (c->stream == nullptr || c->stream == cudaStreamLegacy || c->stream == cudaStreamPerThread) return false;
  return c->graphs > 0 || n <= 32768;
}

void destroy_graph(exageo_ctx* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  c->gexec = nullptr;
  c->graph = nullptr;
  c->gen_nodes.clear();
  c->gkey.clear();
}

std::vector<const void*> graph_key(const exageo_ctx* c, const double* x, const double* y, const double* z,
                                   int kind) {
  std::vector<const void*> k = {(const void*)(intptr_t)c->G.n, (const void*)(intptr_t)c->G.nb, x, y, z,
                                c->parts, c->out3, c->h_res, c->mtab, (const void*)(intptr_t)kind,
                                c->dag_tasks, c->dag_sync, c->dag_W, (const void*)(intptr_t)c->dag_ntasks};
  for (const auto& R : c->rs) {
    for (const void* p : {(const void*)R.ws, (const void*)R.slots, (const void*)R.lkk[0], (const void*)R.lkk[1],
                          (const void*)R.offs_d, (const void*)R.scratch, (const void*)R.info})
      k.push_back(p);
    for (int pp = 0; pp < kMaxP; ++pp) {
      k.push_back(R.recv[0][pp]);
      k.push_back(R.recv[1][pp]);
    }
  }
  return k;
}

// The captured body: timing events are event-record nodes (record_timing).
exageo_status graph_body(exageo_ctx* c, const MaternConsts& mc, const double* x, const double* y,
                         const double* z) {
  CUDA_TRY(c, record_timing(c, c->ev[0], c->stream));
  exageo_status st = launch_generate(c, mc, x, y, z, true);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, record_timing(c, c->ev[1], c->stream));
  c->dag_res = (double*)c->h_res;  // the executor writes the results straight into h_res
  st = do_factor(c);
  c->dag_res = nullptr;
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, record_timing(c, c->ev[2], c->stream));
  if ((st = launch_finish(c)) != EXAGEO_OK) return st;
  double* hd = (double*)c->h_res;
  int* hi = (int*)(hd + 4);
  if (!c->dag_finished) {
    CUDA_TRY(c, cudaMemcpyAsync(hd, c->out3, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    for (size_t i = 0; i < c->rs.size(); ++i)
      CUDA_TRY(c, cudaMemcpyAsync(hi + i, c->rs[i].info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  }
  if (c->comm) {  // the first failing pivot over all ranks (hd[3] holds it as an int64)
    launch_pivot_key(c->rs[0].info, c->pivbuf, c->stream);
    c->kernels += 1;
    NCCL_TRY(c, nccl::AllReduce(c->pivbuf, c->pivbuf, 1, ncclInt64, ncclMin, c->comm, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(hd + 3, c->pivbuf, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, record_timing(c, c->ev[3], c->stream));
  return EXAGEO_OK;
}

exageo_status run_graph(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                        const double* z, double* r3, int64_t* pivot) {
  exageo_status st = prepare_generate(c, t, n, x, y);
  if (st != EXAGEO_OK) return st;
  if (!c->h_res) CUDA_TRY(c, cudaMallocHost(&c->h_res, sizeof(double) * 4 + sizeof(int) * c->rs.size()));
  for (auto& R : c->rs)  // timing events of every U2 launch exist before the capture
    while ((int)R.u2b.size() < R.L.T || (int)R.u1b.size() < R.L.T) {
      cudaEvent_t b, e, b1, e1;
      CUDA_TRY(c, cudaEventCreate(&b));
      CUDA_TRY(c, cudaEventCreate(&e));
      CUDA_TRY(c, cudaEventCreate(&b1));
      CUDA_TRY(c, cudaEventCreate(&e1));
      R.u2b.push_back(b);
      R.u2e.push_back(e);
      R.u1b.push_back(b1);
      R.u1e.push_back(e1);
    }
  const MaternConsts mc = make_consts(*t, c);
  std::vector<const void*> key = graph_key(c, x, y, z, mc.kind);
  if (!c->gexec || key != c->gkey) {
    destroy_graph(c);
    const int64_t k0 = c->kernels;
    c->gen_launches = 0;
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    st = graph_body(c, mc, x, y, z);
    c->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (st != EXAGEO_OK || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return st != EXAGEO_OK ? st : fail(c, EXAGEO_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    }
    c->graph = g;
    CUDA_TRY(c, cudaGraphInstantiateWithFlags(&c->gexec, g, cudaGraphInstantiateFlagUseNodePriority));
    size_t nn = 0;
    CUDA_TRY(c, cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CUDA_TRY(c, cudaGraphGetNodes(g, nodes.data(), &nn));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      CUDA_TRY(c, cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      CUDA_TRY(c, cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == gen_panels_kernel_fn(mc.kind) || kp.func == matern_table_kernel_fn() ||
          (kp.func == dag_factor_kernel_fn() && dag_args_generate(kp.kernelParams[0])))
        c->gen_nodes.push_back(nd);
    }
    if ((int)c->gen_nodes.size() != c->gen_launches) {
      destroy_graph(c);
      return fail(c, EXAGEO_ECUDA, "graph capture: generator nodes not found");
    }
    c->gkey = key;
    c->graph_kernels = c->kernels - k0;
    c->kernels = k0;
    for (auto& R : c->rs) {
      R.g_n_u2 = R.n_u2;
      R.g_u2_flops = R.u2_flops;
      R.g_n_u1 = R.n_u1;
      R.g_u1_flops = R.u1_flops;
    }
  } else {
    for (auto& R : c->rs) {
      R.n_u2 = R.g_n_u2;
      R.u2_flops = R.g_u2_flops;
      R.n_u1 = R.g_n_u1;
      R.u1_flops = R.g_u1_flops;
    }
    for (cudaGraphNode_t nd : c->gen_nodes) {  // new theta into every K1 / K1T node
      cudaKernelNodeParams kp;
      CUDA_TRY(c, cudaGraphKernelNodeGetParams(nd, &kp));
      void* args[7];
      std::vector<char> dag_args;
      if (kp.func == dag_factor_kernel_fn()) {  // dag_factor_kernel(DagArgs): theta inside the struct
        dag_args_with_theta(kp.kernelParams[0], mc, dag_args);
        args[0] = dag_args.data();
      } else {
        const bool gen = kp.func == gen_panels_kernel_fn(mc.kind);
        const int nargs = gen ? 7 : 2, imc = gen ? 2 : 0;
        // gen_panels_kernel(Layout, ws, MaternConsts, x, y, z, tab); matern_table_kernel(MaternConsts, tab)
        for (int i = 0; i < nargs; ++i) args[i] = kp.kernelParams[i];
        args[imc] = (void*)&mc;
      }
      kp.kernelParams = args;
      CUDA_TRY(c, cudaGraphExecKernelNodeSetParams(c->gexec, nd, &kp));
    }
  }
  CUDA_TRY(c, cudaGraphLaunch(c->gexec, c->stream));
  c->kernels += c->graph_kernels;
  c->have_matrix = true;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const double* hd = (const double*)c->h_res;
  const int* hi = (const int*)(hd + 4);
  int64_t best = -1;
  for (size_t i = 0; i < c->rs.size(); ++i)
    if (hi[i] > 0 && (best < 0 || hi[i] - 1 < best)) best = hi[i] - 1;
  if (c->comm) {  // all-reduced in the graph
    int64_t g;
    memcpy(&g, hd + 3, sizeof(g));
    best = g == std::numeric_limits<int64_t>::max() ? -1 : g;
  }
  *pivot = best;
  if (best >= 0) {
    r3[0] = -std::numeric_limits<double>::infinity();
    r3[1] = r3[2] = std::numeric_limits<double>::quiet_NaN();
    return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(best));
  }
  memcpy(r3, hd, 3 * sizeof(double));
  return EXAGEO_OK;
}

exageo_status loglik_device(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                            const double* z, double* loglik, exageo_loglik_info* info) {
  if (!z) return fail(c, EXAGEO_EINVAL, "NULL z");
  const int64_t k0 = c->kernels;
  double r3[3];
  int64_t piv = -1;
  exageo_status st;
  if (graph_eligible(c, n)) {
    st = run_graph(c, t, n, x, y, z, r3, &piv);
    if (st != EXAGEO_OK && st != EXAGEO_ENOTPD) return st;
  } else {
    CUDA_TRY(c, cudaEventRecord(c->ev[0], c->stream));
    st = do_generate(c, t, n, x, y, z, true);
    if (st != EXAGEO_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[1], c->stream));
    st = do_factor(c);
    if (st != EXAGEO_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[2], c->stream));
    st = do_finish(c, r3, &piv);
    if (st != EXAGEO_OK && st != EXAGEO_ENOTPD) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev[3], c->stream));
    CUDA_TRY(c, cudaEventSynchronize(c->ev[3]));
  }
  if (loglik) *loglik = r3[0];
  if (info) {
    memset(info, 0, sizeof(*info));
    info->loglik = r3[0];
    info->logdet = r3[1];
    info->quad = r3[2];
    info->npd_pivot = piv;
    info->n = n;
    info->nb = c->G.nb;
    info->ntiles = c->G.T;
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
    const RankState& R = c->rs[0];  // dominant-kernel timing of (the first) local rank
    info->trailing_launches = R.n_u2;
    info->trailing_flops = R.u2_flops;
    double tr = 0.0;
    for (int i = 0; i < R.n_u2; ++i) {
      cudaEventElapsedTime(&ms, R.u2b[i], R.u2e[i]);
      tr += ms;
    }
    info->ms_trailing = tr;
    // all launches of the trailing-update kernel (U1 + U2): union of their spans
    std::vector<std::pair<float, float>> iv;
    auto span = [&](cudaEvent_t b, cudaEvent_t e) {
      float tb = 0.f, te = 0.f;
      if (cudaEventElapsedTime(&tb, c->ev[1], b) == cudaSuccess && cudaEventElapsedTime(&te, c->ev[1], e) == cudaSuccess)
        iv.push_back({tb, te});
    };
    for (int i = 0; i < R.n_u2; ++i) span(R.u2b[i], R.u2e[i]);
    for (int i = 0; i < R.n_u1; ++i) span(R.u1b[i], R.u1e[i]);
    std::sort(iv.begin(), iv.end());
    double uni = 0.0, cur_b = -1.0, cur_e = -1.0;
    for (auto& v : iv) {
      if (v.first > cur_e) {
        if (cur_e > cur_b) uni += cur_e - cur_b;
        cur_b = v.first;
        cur_e = v.second;
      } else if (v.second > cur_e) {
        cur_e = v.second;
      }
    }
    if (cur_e > cur_b) uni += cur_e - cur_b;
    info->update_launches = R.n_u2 + R.n_u1;
    info->ms_update_union = uni;
    info->update_flops = R.u2_flops + R.u1_flops;
    // tracing (env EXAGEO_U2_TRACE=<file>): each bulk trailing update's [start, end] in ms from
    // the start of the factorization, appended per evaluation -- the gaps between them are
    // the panel chain's stalls
    if (const char* tp = getenv("EXAGEO_U2_TRACE")) {
      if (FILE* f = fopen(tp, "a")) {
        fprintf(f, "# n=%lld nb=%d steps=%d\n", (long long)c->G.n, c->G.nb, R.n_u2);
        for (int i = 0; i < R.n_u2; ++i) {
          float b = 0.f, e = 0.f;
          cudaEventElapsedTime(&b, c->ev[1], R.u2b[i]);
          cudaEventElapsedTime(&e, c->ev[1], R.u2e[i]);
          fprintf(f, "%d %.4f %.4f\n", i, b, e);
        }
        float end = 0.f;
        cudaEventElapsedTime(&end, c->ev[1], c->ev[2]);
        fprintf(f, "end %.4f\n", end);
        fclose(f);
      }
    }
  }
  return st;
}

}  // namespace

namespace exageo {
exageo_status eval_loglik(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x_d, const double* y_d,
                          const double* z_d, double* ll, double* logdet, double* quad) {
  if (!logdet && !quad) return loglik_device(c, t, n, x_d, y_d, z_d, ll, nullptr);
  exageo_loglik_info info;
  const exageo_status st = loglik_device(c, t, n, x_d, y_d, z_d, ll, &info);
  if (logdet) *logdet = info.logdet;
  if (quad) *quad = info.quad;
  return st;
}
exageo_status staging(exageo_ctx* c, int64_t n, double** buf) {
  exageo_status st = ensure_vec(c, n);
  *buf = c->vec;
  return st;
}
exageo_status set_error(exageo_ctx* c, exageo_status s, const std::string& msg) { return fail(c, s, msg); }
}  // namespace exageo

namespace {

void destroy_rank(RankState& R) {
  if (R.ws && !R.ws_external) cudaFree(R.ws);
  for (auto& b : R.recv)
    for (auto p : b) cudaFree(p);
  for (auto p : R.lkk) cudaFree(p);
  cudaFree(R.offs_d);
  cudaFree(R.slots);
  cudaFree(R.scratch);
  cudaFree(R.info);
  cudaFree(R.part);
  for (cudaEvent_t ev : {R.ev_F, R.ev_U2[0], R.ev_U2[1], R.ev_U1[0], R.ev_U1[1], R.ev_recv[0], R.ev_recv[1], R.ev_lkk,
                         R.ev_row,
                         R.ev_join[0], R.ev_join[1], R.ev_join[2]})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : R.u2b) cudaEventDestroy(ev);
  for (cudaEvent_t ev : R.u2e) cudaEventDestroy(ev);
  for (cudaEvent_t ev : R.u1b) cudaEventDestroy(ev);
  for (cudaEvent_t ev : R.u1e) cudaEventDestroy(ev);
  for (cudaStream_t s : {R.s_la, R.s_main, R.s_comm})
    if (s) cudaStreamDestroy(s);
}

cudaError_t init_rank(RankState& R) {
  cudaError_t e;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = numerically smallest = highest priority
  if ((e = cudaStreamCreateWithPriority(&R.s_la, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&R.s_main, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&R.s_comm, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
  for (cudaEvent_t* ev : {&R.ev_F, &R.ev_U2[0], &R.ev_U2[1], &R.ev_U1[0], &R.ev_U1[1], &R.ev_recv[0], &R.ev_recv[1],
                          &R.ev_lkk, &R.ev_row,
                          &R.ev_join[0], &R.ev_join[1], &R.ev_join[2]})
    if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&R.scratch, sizeof(double) * kQuadBlocks)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&R.info, sizeof(int))) != cudaSuccess) return e;
  return cudaMemset(R.info, 0, sizeof(int));
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

exageo_status exageo_nccl_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId)) return fail(nullptr, EXAGEO_EINVAL, "need a 128-byte buffer");
  ncclUniqueId id;
  std::string lerr;
  if (!nccl::load(&lerr)) return fail(nullptr, EXAGEO_ENCCL, lerr);
  ncclResult_t r = nccl::GetUniqueId(&id);
  if (r != ncclSuccess)
    return fail(nullptr, EXAGEO_ENCCL, std::string("ncclGetUniqueId: ") + nccl::GetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return EXAGEO_OK;
}

exageo_status exageo_create(exageo_ctx** out, const exageo_opts* opts) {
  if (!out) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx pointer");
  *out = nullptr;
  exageo_opts o{};
  if (opts) o = *opts;
  if (o.nb != 0 && (o.nb < 128 || o.nb % 128 != 0))
    return fail(nullptr, EXAGEO_EINVAL, "nb must be 0 (auto) or a positive multiple of 128");
  if (o.ind_tiles < 0) return fail(nullptr, EXAGEO_EINVAL, "ind_tiles must be >= 0");
  if (o.distance < 0 || o.distance > 1 || !(o.radius >= 0) || !std::isfinite(o.radius))
    return fail(nullptr, EXAGEO_EINVAL, "distance must be 0 (Euclidean) or 1 (great-circle), radius >= 0");
  if (o.world < 0 || o.virtual_ranks < 0 || (o.world > 1 && o.virtual_ranks > 1) ||
      (o.world > 1 && (o.rank < 0 || o.rank >= o.world || !o.nccl_id)))
    return fail(nullptr, EXAGEO_EINVAL, "bad distribution options (world/rank/nccl_id/virtual_ranks)");
  {
    const int ranks = o.virtual_ranks > 1 ? o.virtual_ranks : (o.world > 1 ? o.world : 1);
    const int P = o.grid_rows > 1 ? o.grid_rows : 1;
    if (o.grid_rows < 0 || P > kMaxP || ranks % P != 0)
      return fail(nullptr, EXAGEO_EINVAL, "grid_rows must divide the number of ranks and be <= 8");
  }
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
  c->ind = o.ind_tiles > 0 ? o.ind_tiles : 0;
  c->graphs = o.graphs > 0 ? 1 : (o.graphs < 0 ? -1 : 0);
  c->tile_tasks = o.tile_tasks > 0 ? 1 : (o.tile_tasks < 0 ? -1 : 0);
  if (const char* tp = getenv("EXAGEO_TILE_TASK_TRACE")) c->dag_trace_path = tp;
  c->metric = o.distance;
  c->radius = o.radius > 0 ? o.radius : 6371.0;
  c->virt = o.virtual_ranks > 1;
  c->world = c->virt ? o.virtual_ranks : (o.world > 1 ? o.world : 1);
  c->rank = (!c->virt && o.world > 1) ? o.rank : 0;
  c->P = o.grid_rows > 1 ? o.grid_rows : 1;
  c->Q = c->world / c->P;
  auto bail = [&](cudaError_t err, const char* what) {
    g_create_err = std::string(what) + ": " + cudaGetErrorString(err);
    exageo_destroy(c);
    return EXAGEO_ECUDA;
  };
  if ((e = cudaSetDevice(o.device)) != cudaSuccess) return bail(e, "cudaSetDevice");
  if ((e = gemm_init()) != cudaSuccess) return bail(e, "gemm_init");
  if ((e = potrf_init()) != cudaSuccess) return bail(e, "potrf_init");
  if ((e = dag_init()) != cudaSuccess) return bail(e, "dag_init");
  if ((e = trsv_init()) != cudaSuccess) return bail(e, "trsv_init");
  if (o.stream) {
    c->stream = (cudaStream_t)o.stream;
  } else {
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess)
      return bail(e, "cudaStreamCreate");
    c->own_stream = true;
  }
  for (auto& ev : c->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return bail(e, "cudaEventCreate");
  if ((e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess)
    return bail(e, "cudaEventCreate");
  if ((e = cudaEventCreateWithFlags(&c->ev_wait, cudaEventDisableTiming)) != cudaSuccess)
    return bail(e, "cudaEventCreate");
  c->rs.resize(c->virt ? c->world : 1);
  for (auto& R : c->rs)
    if ((e = init_rank(R)) != cudaSuccess) return bail(e, "rank state");
  if ((e = cudaMalloc(&c->parts, sizeof(double) * 2 * c->world)) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaMalloc(&c->out3, sizeof(double) * 4)) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaMalloc(&c->mtab, sizeof(double) * matern_table_doubles())) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaMalloc(&c->pivbuf, sizeof(int64_t))) != cudaSuccess) return bail(e, "cudaMalloc");
  if (!c->virt && o.nccl_id) {  // world > 1, or a single-rank NCCL communicator (world 1)
    ncclUniqueId id;
    memcpy(&id, o.nccl_id, sizeof(id));
    std::string lerr;
    if (!nccl::load(&lerr)) {
      g_create_err = lerr;
      exageo_destroy(c);
      return EXAGEO_ENCCL;
    }
    ncclResult_t r = nccl::CommInitRank(&c->comm, c->world, id, c->rank);
    if (r != ncclSuccess) {
      g_create_err = std::string("ncclCommInitRank: ") + nccl::GetErrorString(r);
      c->comm = nullptr;
      exageo_destroy(c);
      return EXAGEO_ENCCL;
    }
    if (c->P > 1) {  // process-row (color p, key q) and process-column (color q, key p) communicators
      const int p = c->rank / c->Q, q = c->rank % c->Q;
      r = nccl::CommSplit(c->comm, p, q, &c->comm_row, nullptr);
      if (r == ncclSuccess) r = nccl::CommSplit(c->comm, q, p, &c->comm_col, nullptr);
      if (r != ncclSuccess) {
        g_create_err = std::string("ncclCommSplit: ") + nccl::GetErrorString(r);
        exageo_destroy(c);
        return EXAGEO_ENCCL;
      }
    }
  }
  *out = c;
  return EXAGEO_OK;
}

void exageo_destroy(exageo_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm_row) nccl::CommDestroy(c->comm_row);
  if (c->comm_col) nccl::CommDestroy(c->comm_col);
  if (c->comm) nccl::CommDestroy(c->comm);
  destroy_graph(c);
  if (c->h_res) cudaFreeHost(c->h_res);
  for (auto& R : c->rs) destroy_rank(R);
  cudaFree(c->parts);
  cudaFree(c->out3);
  cudaFree(c->mtab);
  cudaFree(c->pivbuf);
  cudaFree(c->vec);
  cudaFree(c->zsum);
  if (c->dag_trace && !c->dag_trace_path.empty()) dump_tile_task_trace(c);
  cudaFree(c->dag_tasks);
  cudaFree(c->dag_sync);
  cudaFree(c->dag_W);
  cudaFree(c->dag_trace);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_wait) cudaEventDestroy(c->ev_wait);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

size_t exageo_workspace_bytes(int64_t n, int nb) {
  if (n < 1) return 0;
  if (nb <= 0) nb = auto_nb(n);
  return local_bytes(make_layout(n, nb));
}

size_t exageo_rank_workspace_bytes(int64_t n, int nb, int world, int grid_rows, int rank) {
  const int P = grid_rows > 1 ? grid_rows : 1;
  if (n < 1 || world < 1 || rank < 0 || rank >= world || P > kMaxP || world % P != 0) return 0;
  if (nb <= 0) nb = auto_nb(n, world);
  if (nb % 128 != 0) return 0;
  Layout L = make_layout(n, nb, rank, world, 0, P);
  std::vector<int64_t> o(L.owned() + 1, 0);
  for (int m = 0; m < L.owned(); ++m) o[m + 1] = o[m] + (int64_t)L.nb * L.ld(L.owned_panel(m));
  L.offs_h = o.data();
  return local_bytes(L);
}

exageo_status exageo_set_workspace(exageo_ctx* c, void* ptr, size_t bytes) {
  if (!c) return EXAGEO_EINVAL;
  if (c->virt) return fail(c, EXAGEO_EINVAL, "external workspace is not supported with virtual ranks");
  // the generator stores double2 and the DMMA kernels load 16-byte cp.async chunks
  if ((uintptr_t)ptr % 256 != 0) return fail(c, EXAGEO_EINVAL, "workspace pointer must be 256-byte aligned");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  RankState& R = c->rs[0];
  if (R.ws && !R.ws_external) cudaFree(R.ws);
  R.ws = (double*)ptr;
  R.ws_bytes = ptr ? bytes : 0;
  R.ws_external = ptr != nullptr;
  c->have_matrix = false;
  c->dag_init_key.clear();
  return EXAGEO_OK;
}

exageo_status exageo_stream_wait(exageo_ctx* c, void* stream) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if ((cudaStream_t)stream == c->stream) return EXAGEO_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaEventRecord(c->ev_wait, (cudaStream_t)stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_wait, 0));
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
  double* d = nullptr;
  const size_t bytes = sizeof(double) * (2 * (size_t)m + 2 * (size_t)n + (size_t)m * (size_t)n);
  CUDA_TRY(c, cudaMalloc(&d, bytes));
  double *dx1 = d, *dy1 = d + m, *dx2 = d + 2 * m, *dy2 = d + 2 * m + n, *dC = d + 2 * m + 2 * n;
  cudaError_t e = cudaMemcpyAsync(dx1, x1, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dy1, y1, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dx2, x2, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dy2, y2, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    launch_matern_dense(make_consts(*t, c), m, dx1, dy1, n, dx2, dy2, dC, m, c->mtab, c->stream);
    c->kernels += 1;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(C, sizeof(double) * ldc, dC, sizeof(double) * m, sizeof(double) * m, n,
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
  st = do_generate(c, t, n, dx, dy, nullptr, true);
  if (st != EXAGEO_OK) return st;
  st = do_factor(c);
  if (st != EXAGEO_OK) return st;
  int64_t piv = -1;
  st = first_pivot(c, &piv);
  if (st != EXAGEO_OK) return st;
  if (piv >= 0) return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(piv));
  // Alg. 1 l.7: z = L e -- per-panel partial products, summed over all panels (and ranks)
  const Layout& G = c->G;
  size_t slices_all = 0;
  for (auto& R : c->rs) slices_all += (size_t)R.L.owned();
  const size_t need = sizeof(double) * (slices_all > 0 ? slices_all : 1) * (size_t)G.N;
  RankState& R0 = c->rs[0];
  if (R0.part_cap < need) {
    cudaFree(R0.part);
    R0.part = nullptr;
    CUDA_TRY(c, cudaMalloc(&R0.part, need));
    R0.part_cap = need;
  }
  int slices = 0;
  for (auto& R : c->rs) {
    launch_trmv_partial(R.L, R.ws, de, R0.part + (size_t)slices * G.N, c->stream);
    slices += R.L.owned();
    c->kernels += 1;
  }
  if (c->comm) {
    launch_trmv_sum(n, G.N, R0.part, slices, c->zsum, c->stream);
    NCCL_TRY(c, nccl::AllReduce(c->zsum, dz, n, ncclDouble, ncclSum, c->comm, c->stream));
  } else {
    launch_trmv_sum(n, G.N, R0.part, slices, dz, c->stream);
  }
  c->kernels += 1;
  st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemcpyAsync(z, dz, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EXAGEO_OK;
}

exageo_status exageo_predict(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                             const double* z, int64_t m, const double* xnew, const double* ynew, double* znew) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (n < 1 || m < 1 || !x || !y || !z || !xnew || !ynew || !znew)
    return fail(c, EXAGEO_EINVAL, "n < 1, m < 1 or NULL array");
  if (!theta_ok(t)) return fail(c, EXAGEO_EINVAL, "theta must be finite and > 0");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int nb = c->nb_opt > 0 ? c->nb_opt : auto_nb(n, c->world);
  const Layout G0 = make_layout(n, nb);
  // device scratch: x, y, z (n each), xnew, ynew, znew (m each), w (N), solve and krige partials
  const size_t nw = (size_t)G0.N;
  const size_t ntr = (size_t)trsv_chunks(G0.N) * nb;
  const size_t nkr = (size_t)krige_chunks(n) * (size_t)m;
  const size_t total = 3 * (size_t)n + 3 * (size_t)m + nw + ntr + nkr;
  double* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(double) * total));
  struct Free {
    double* p;
    ~Free() { cudaFree(p); }
  } guard{d};
  double *dx = d, *dy = dx + n, *dz = dy + n, *dxn = dz + n, *dyn = dxn + m, *dzn = dyn + m, *w = dzn + m,
         *ptr = w + nw, *pkr = ptr + ntr;
  CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dz, z, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dxn, xnew, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dyn, ynew, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  // Alg. 3 l.3-7: Sigma22 = L L^T with the forward solve y = L^{-1} z2 fused (z row)
  exageo_status st = do_generate(c, t, n, dx, dy, dz, true);
  if (st != EXAGEO_OK) return st;
  st = do_factor(c);
  if (st != EXAGEO_OK) return st;
  int64_t piv = -1;
  st = first_pivot(c, &piv);
  if (st != EXAGEO_OK) return st;
  if (piv >= 0) return fail(c, EXAGEO_ENOTPD, "covariance not positive definite at pivot " + std::to_string(piv));
  // backward solve L^T w = y, panel by panel from the last; each w_j is made available to
  // every rank (NCCL broadcast from the panel's diagonal rank; virtual ranks share w)
  const Layout& G = c->G;
  if (c->P == 1) {
    for (int j = G.T - 1; j >= 0; --j) {
      const int o = j % c->world;
      if (RankState* R = local_state(c, o)) {
        const double* P = R->ws + R->L.off(j);
        const int64_t rows = G.N - (int64_t)(j + 1) * G.nb;
        launch_backsolve_panel(P, G.ld(j), G.nb, (int64_t)(j + 1) * G.nb, rows, w, w + (int64_t)j * G.nb, ptr,
                               c->stream);
        c->kernels += rows > 0 ? 2 : 1;
      }
      if (c->comm)
        NCCL_TRY(c, nccl::Broadcast(w + (int64_t)j * G.nb, w + (int64_t)j * G.nb, G.nb, ncclDouble, o, c->comm,
                                    c->stream));
    }
  } else {
    // 2-D grid: y = L^{-1} z (the z rows, on one process row) replicated first; per panel j the
    // ranks of its process column form partial sums over their tile rows below the diagonal,
    // reduced onto the diagonal rank, which solves with L_jj and broadcasts w_j
    double* yv = nullptr;
    const size_t nvec = (size_t)G.N + (size_t)(kMaxP + 1) * G.nb;
    CUDA_TRY(c, cudaMalloc(&yv, sizeof(double) * nvec));
    Free g2{yv};
    double* vecs = yv + G.N;  // P partial vectors (virtual) or {own partial, reduced sum} (NCCL)
    CUDA_TRY(c, cudaMemsetAsync(yv, 0, sizeof(double) * (size_t)G.N, c->stream));
    for (auto& R : c->rs) launch_read_zrow(R.L, R.ws, yv, c->stream);
    c->kernels += (int64_t)c->rs.size();
    if (c->comm) NCCL_TRY(c, nccl::AllReduce(yv, yv, (size_t)G.N, ncclDouble, ncclSum, c->comm, c->stream));
    for (int j = G.T - 1; j >= 0; --j) {
      double* wj = w + (int64_t)j * G.nb;
      RankState* D = nullptr;
      for (auto& R : c->rs) {
        const Layout& L = R.L;
        if (!L.owns(j)) continue;
        if (L.diag(j)) D = &R;
        const int64_t lr0 = L.diag(j) ? G.nb : 0;
        const int64_t rows = L.lrows(j) - lr0;
        double* out = c->virt ? vecs + (size_t)L.p * G.nb : vecs;
        launch_backsolve_partial(L, j, R.ws + L.off(j), L.ld(j), lr0, rows, w, ptr, out, c->stream);
        c->kernels += 2;
      }
      if (c->virt) {
        launch_tile_solve(D->ws + D->L.off(j), D->L.ld(j), G.nb, yv + (int64_t)j * G.nb, vecs, c->P, wj, c->stream);
        c->kernels += 1;
      } else {
        RankState& R = c->rs[0];
        if (R.L.owns(j)) {
          NCCL_TRY(c, nccl::Reduce(vecs, vecs + G.nb, G.nb, ncclDouble, ncclSum, j % c->P, c->comm_col, c->stream));
          if (D) {
            launch_tile_solve(D->ws + D->L.off(j), D->L.ld(j), G.nb, yv + (int64_t)j * G.nb, vecs + G.nb, 1, wj,
                              c->stream);
            c->kernels += 1;
          }
        }
        NCCL_TRY(c, nccl::Broadcast(wj, wj, G.nb, ncclDouble, R.L.owner(j), c->comm, c->stream));
      }
    }
  }
  // Alg. 3 l.8 / Eq. (5): z1 = Sigma12 w with Sigma12 generated on the fly
  launch_krige(make_consts(*t, c), m, dxn, dyn, n, dx, dy, w, pkr, dzn, c->mtab, c->stream);
  c->kernels += 2;
  st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemcpyAsync(znew, dzn, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EXAGEO_OK;
}

}  // extern "C"

// Kriging variance on a distributed context (NCCL ranks or virtual ranks, any P x Q grid), after
// exageo_predict left L of Sigma22 in the tiles: V = L^{-1} Sigma21 by a distributed forward
// substitution over the tile rows I = 0 .. T-1 (the multi-right-hand-side form of Alg. 2 l.4):
//   U_I^(q) = -sum_{j < I, j = q mod Q} L_Ij V_j   accumulated on rank (I mod P, q),
//   S_I     = Sigma21[tile row I] + sum_q U_I^(q)  reduced along process row I mod P onto the
//                                                  diagonal rank (I mod P, I mod Q),
//   V_I     = L_II^{-1} S_I                         broadcast down process column I mod Q, whose
//             ranks apply U_I' -= L_I'I V_I to their tile rows I' > I (DMMA);
//   var_c   = theta1 - sum_I sum_r (V_I)_rc^2       (the diagonal ranks' column sums, all-reduced).
// Batches of mc new sites keep each rank's accumulator U (its tile rows x mc) within ~1 GB.
exageo_status predict_var_grid(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                               int64_t m, const double* xnew, const double* ynew, double* var) {
  const Layout& G = c->G;
  const int nb = G.nb, T = G.T, P = c->P, Q = c->Q;
  const Layout& L0 = c->rs[0].L;
  int64_t tp_max = 1;
  for (int pp = 0; pp < P; ++pp) tp_max = std::max<int64_t>(tp_max, L0.Tp_of(pp));
  int64_t mc = std::max<int64_t>(64, ((int64_t)1 << 27) / (tp_max * nb) / 64 * 64);  // 1 GB of U per rank
  mc = std::min<int64_t>(mc, (m + 63) / 64 * 64);
  std::vector<double*> U(c->rs.size(), nullptr);
  struct FreeAll {
    std::vector<double*>& v;
    double* d = nullptr;
    ~FreeAll() {
      for (double* p : v) cudaFree(p);
      cudaFree(d);
    }
  } guard{U};
  for (size_t i = 0; i < c->rs.size(); ++i)
    CUDA_TRY(c, cudaMalloc(&U[i], sizeof(double) * (size_t)c->rs[i].L.Tp() * nb * mc + 8));
  // shared: x, y (n), the batch's sites (2 mc), S_I / V_I (nb mc), V_I^T (mc nb), reduce buffer
  // (nb mc), column sums (mc) and variances (mc)
  const size_t tot = 2 * (size_t)n + 2 * (size_t)mc + 3 * (size_t)nb * mc + 2 * (size_t)mc;
  CUDA_TRY(c, cudaMalloc(&guard.d, sizeof(double) * tot));
  double *dx = guard.d, *dy = dx + n, *dxn = dy + n, *dyn = dxn + mc, *Sb = dyn + mc, *Vt = Sb + (size_t)nb * mc,
         *red = Vt + (size_t)nb * mc, *acc = red + (size_t)nb * mc, *dvar = acc + mc;
  CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  const MaternConsts mcs = make_consts(*t, c);
  for (int64_t i0 = 0; i0 < m; i0 += mc) {
    const int cols = (int)std::min<int64_t>(mc, m - i0);
    CUDA_TRY(c, cudaMemcpyAsync(dxn, xnew + i0, sizeof(double) * cols, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(dyn, ynew + i0, sizeof(double) * cols, cudaMemcpyHostToDevice, c->stream));
    for (size_t i = 0; i < c->rs.size(); ++i)
      CUDA_TRY(c, cudaMemsetAsync(U[i], 0, sizeof(double) * (size_t)c->rs[i].L.Tp() * nb * mc, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(acc, 0, sizeof(double) * mc, c->stream));
    for (int I = 0; I < T; ++I) {
      const int pI = I % P, qI = I % Q;
      const int64_t r0 = (int64_t)I * nb;
      const int rv = (int)std::max<int64_t>(0, std::min<int64_t>(nb, n - r0));  // rows of tile I inside n
      RankState* D = local_state(c, pI * Q + qI);
      // (1) S_I = Sigma21[tile I] + sum_q U_I^(q) on the diagonal rank
      auto gen_S = [&]() -> exageo_status {
        CUDA_TRY(c, cudaMemsetAsync(Sb, 0, sizeof(double) * (size_t)nb * mc, c->stream));
        if (rv > 0) launch_matern_dense(mcs, rv, dx + r0, dy + r0, cols, dxn, dyn, Sb, nb, c->mtab, c->stream);
        return EXAGEO_OK;
      };
      if (c->virt) {
        gen_S();
        for (int qq = 0; qq < Q; ++qq) {  // fixed order
          RankState& R = c->rs[pI * Q + qq];
          launch_add_block(Sb, nb, U[pI * Q + qq] + (int64_t)((I - pI) / P) * nb, (int64_t)R.L.Tp() * nb, nb, cols,
                           c->stream);
        }
      } else {
        RankState& R = c->rs[0];
        if (R.L.p == pI) {
          CUDA_TRY(c, cudaMemcpy2DAsync(red, sizeof(double) * nb, U[0] + (int64_t)((I - pI) / P) * nb,
                                        sizeof(double) * (size_t)R.L.Tp() * nb, sizeof(double) * nb, cols,
                                        cudaMemcpyDeviceToDevice, c->stream));
          NCCL_TRY(c, nccl::Reduce(red, red, (size_t)nb * cols, ncclDouble, ncclSum, qI, row_comm(c), c->stream));
        }
        if (D) {
          gen_S();
          launch_add_block(Sb, nb, red, nb, nb, cols, c->stream);
        }
      }
      // (2) V_I = L_II^{-1} S_I (tile I is the first tile row of the diagonal rank's local panel I)
      if (D) {
        launch_diag_solve_cols(D->ws + D->L.off(I), D->L.ld(I), nb, Sb, nb, cols, c->stream);
        launch_colsq_accum(Sb, nb, rv, cols, acc, c->stream);
      }
      // (3) V_I down process column I mod Q
      if (!c->virt && P > 1 && c->rs[0].L.q == qI)
        NCCL_TRY(c, nccl::Broadcast(Sb, Sb, (size_t)nb * cols, ncclDouble, pI, c->comm_col, c->stream));
      // (4) the column's ranks: U_I' -= L_I'I V_I for their tile rows I' > I
      bool transposed = false;
      for (size_t i = 0; i < c->rs.size(); ++i) {
        RankState& R = c->rs[i];
        if (R.L.q != qI) continue;
        const int64_t lr0 = R.L.p == pI ? nb : 0;
        const int64_t rows = R.L.lrows(I) - lr0;
        if (rows <= 0) continue;
        if (!transposed) {  // V_I^T with row stride mc (16-byte aligned rows for cp.async)
          launch_transpose(Sb, nb, nb, (int)mc, Vt, c->stream);
          transposed = true;
        }
        launch_gemm_panel(rows, cols, nb, R.ws + R.L.off(I) + lr0, R.L.ld(I), Vt, mc,
                          U[i] + (int64_t)R.L.i0(I) * nb + lr0, (int64_t)R.L.Tp() * nb, true, nullptr, c->stream);
        c->kernels += 2;
      }
      c->kernels += 3;
    }
    if (!c->virt && c->comm) NCCL_TRY(c, nccl::AllReduce(acc, acc, cols, ncclDouble, ncclSum, c->comm, c->stream));
    launch_var_from_acc(acc, cols, t->sigma2, dvar, c->stream);
    exageo_status st = check_launch(c);
    if (st != EXAGEO_OK) return st;
    CUDA_TRY(c, cudaMemcpyAsync(var + i0, dvar, sizeof(double) * cols, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return EXAGEO_OK;
}

extern "C" {

exageo_status exageo_predict_var(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x, const double* y,
                                 const double* z, int64_t m, const double* xnew, const double* ynew, double* znew,
                                 double* var) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!var) return fail(c, EXAGEO_EINVAL, "NULL var");
  if (c->nb_opt > 1024)
    return fail(c, EXAGEO_EINVAL, "the kriging variance supports tile sizes nb <= 1024 (one thread per tile row)");
  // mean (Eq. 5) -- leaves L of Sigma22 in the workspace; an automatic tile size above 1024
  // (single GPU, n >= 56k) is capped at 1024 for this call
  const int nb_saved = c->nb_opt;
  if (nb_saved == 0 && auto_nb(n, c->world) > 1024) c->nb_opt = 1024;
  exageo_status st = exageo_predict(c, t, n, x, y, z, m, xnew, ynew, znew);
  c->nb_opt = nb_saved;
  if (st != EXAGEO_OK) return st;
  if (c->world > 1 || c->virt) return predict_var_grid(c, t, n, x, y, m, xnew, ynew, var);
  // var_i = theta1 - sigma_i^T Sigma22^{-1} sigma_i = theta1 - ||L^{-1} sigma_i||^2, sigma_i = Sigma21[:, i]:
  // batches of mc new sites, S = Sigma21 (N x mc, identity padding rows zero), forward solve
  // panel by panel (diagonal tile substitution, then the DMMA update of the rows below).
  const Layout& G = c->G;
  RankState& R = c->rs[0];
  const int64_t N = G.N;
  const int nb = G.nb;
  int64_t mc = std::max<int64_t>(64, ((int64_t)2 << 30) / (8 * N) / 64 * 64);  // <= 2 GB per batch
  mc = std::min<int64_t>(mc, (m + 63) / 64 * 64);
  const size_t total = 2 * (size_t)n + 2 * (size_t)mc + (size_t)N * mc + (size_t)mc * nb + (size_t)mc;
  double* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(double) * total));
  struct Free {
    double* p;
    ~Free() { cudaFree(p); }
  } guard{d};
  double *dx = d, *dy = dx + n, *dxn = dy + n, *dyn = dxn + mc, *S = dyn + mc, *Bt = S + (size_t)N * mc,
         *dv = Bt + (size_t)mc * nb;
  CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  const MaternConsts mc_consts = make_consts(*t, c);
  for (int64_t i0 = 0; i0 < m; i0 += mc) {
    const int cols = (int)std::min<int64_t>(mc, m - i0);
    CUDA_TRY(c, cudaMemcpyAsync(dxn, xnew + i0, sizeof(double) * cols, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(dyn, ynew + i0, sizeof(double) * cols, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(S, 0, sizeof(double) * (size_t)N * mc, c->stream));
    launch_matern_dense(mc_consts, n, dx, dy, cols, dxn, dyn, S, N, c->mtab, c->stream);
    for (int j = 0; j < G.T; ++j) {
      const double* P = R.ws + R.L.off(j);
      const int64_t jb = (int64_t)j * nb;
      launch_diag_solve_cols(P, G.ld(j), nb, S + jb, N, cols, c->stream);
      const int64_t rows = N - jb - nb;
      if (rows > 0) {  // S[jb+nb:, :] -= L[jb+nb:, jb:jb+nb] V_j
        launch_transpose(S + jb, N, nb, (int)mc, Bt, c->stream);
        launch_gemm_panel(rows, cols, nb, P + nb, G.ld(j), Bt, mc, S + jb + nb, N, true, nullptr, c->stream);
        c->kernels += 2;
      }
      c->kernels += 1;
    }
    launch_column_var(S, N, n, cols, t->sigma2, dv, c->stream);
    c->kernels += 2;
    st = check_launch(c);
    if (st != EXAGEO_OK) return st;
    CUDA_TRY(c, cudaMemcpyAsync(var + i0, dv, sizeof(double) * cols, cudaMemcpyDeviceToHost, c->stream));
  }
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

static const int64_t kReadLowerMaxN = 32768;

exageo_status exageo_read_lower(exageo_ctx* c, double* dst, int64_t ld) {
  if (!c) return fail(nullptr, EXAGEO_EINVAL, "NULL ctx");
  if (!c->have_matrix || !dst || ld < c->G.n) return fail(c, EXAGEO_EINVAL, "no matrix or bad ld");
  const int64_t n = c->G.n;
  // a dense n x n staging copy on the device and the host: a debugging/test entry, bounded
  if (n > kReadLowerMaxN)
    return fail(c, EXAGEO_EINVAL, "read_lower stages a dense n x n copy; n > " + std::to_string(kReadLowerMaxN) +
                                      " (use exageo_read_entries)");
  CUDA_TRY(c, cudaSetDevice(c->device));
  double* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(double) * (size_t)n * (size_t)n));
  cudaError_t e = cudaMemsetAsync(d, 0, sizeof(double) * (size_t)n * (size_t)n, c->stream);
  for (auto& R : c->rs) launch_read_lower(R.L, R.ws, d, n, c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
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
  exageo_status st = ensure_vec(c, c->G.n);
  if (st != EXAGEO_OK) return st;
  double* d = c->vec + 3 * c->G.n;
  CUDA_TRY(c, cudaMemsetAsync(d, 0, sizeof(double) * (size_t)c->G.n, c->stream));
  for (auto& R : c->rs) launch_read_zrow(R.L, R.ws, d, c->stream);
  st = check_launch(c);
  if (st != EXAGEO_OK) return st;
  CUDA_TRY(c, cudaMemcpyAsync(dst, d, sizeof(double) * (size_t)c->G.n, cudaMemcpyDeviceToHost, c->stream));
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
    if (cols[i] < 0 || cols[i] > rows[i] || rows[i] >= c->G.n)
      return fail(c, EXAGEO_EINVAL, "entry outside the lower triangle");
  CUDA_TRY(c, cudaSetDevice(c->device));
  void* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(int64_t) * 2 * (size_t)count + sizeof(double) * (size_t)count));
  int64_t* drc = (int64_t*)d;
  double* dout = (double*)(drc + 2 * count);
  cudaError_t e = cudaMemcpyAsync(drc, rows, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(drc + count, cols, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(dout, 0, sizeof(double) * count, c->stream);
  if (e == cudaSuccess) {
    for (auto& R : c->rs) launch_read_entries(R.L, R.ws, count, drc, dout, c->stream);
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
