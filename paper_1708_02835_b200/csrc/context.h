// context.h -- the library context (exageo_ctx) and the per-rank state of the
// distributed executor (schedule.cu). Internal; not part of the C ABI.
#pragma once
#include <nccl.h>

#include <string>
#include <vector>

#include "../../include/exageo.h"
#include "internal.h"

namespace exageo {

// Everything one rank needs: its panels, receive buffers for broadcast panels,
// streams of the lookahead schedule and their events. In NCCL mode a process holds
// one RankState; in virtual mode one process holds `world` of them on one device.
struct RankState {
  Layout L;                    // rank-local layout (rank, world, process grid)
  double* ws = nullptr;        // owned panels
  size_t ws_bytes = 0;
  bool ws_external = false;
  std::vector<int64_t> offs_h; // P > 1: local panel offsets (host; L.offs_h points here)
  int64_t* offs_d = nullptr;   // P > 1: the same on the device (L.offs_d)
  size_t offs_cap = 0;
  // received slices of panel k (world > 1), by k % 2 and source process row: slice pp is the
  // local panel k of rank (pp, k mod Q); the rank's own slice when it stores panel k is its
  // own storage
  double* recv[2][kMaxP] = {};
  size_t recv_bytes[kMaxP] = {};
  // by k % 2: [L_kk (nb x nb, ld nb) | W_s = L_ss^{-1} of its nb/64 diagonal 64-blocks (64 x 64
  // each)], written by F(k) on the diagonal rank and broadcast down its process column (P > 1)
  double* lkk[2] = {nullptr, nullptr};
  size_t lkk_bytes = 0;
  double* slots = nullptr;     // log-det partials: (nb / PB) per owned panel
  int64_t slots_cap = 0;
  double* scratch = nullptr;   // kQuadBlocks doubles
  int* info = nullptr;         // 0 or first failing global pivot + 1
  double* part = nullptr;      // TRMV partial sums (owned * N doubles)
  size_t part_cap = 0;
  cudaStream_t s_la = nullptr, s_main = nullptr, s_comm = nullptr;
  cudaEvent_t ev_F = nullptr;                    // F(k) done (panel k factored)
  cudaEvent_t ev_U2[2] = {nullptr, nullptr};     // U2(k) done, by k % 2
  cudaEvent_t ev_U1[2] = {nullptr, nullptr};     // U1(k) done, by k % 2
  cudaEvent_t ev_recv[2] = {nullptr, nullptr};   // panel j received, by j % 2
  cudaEvent_t ev_lkk = nullptr;                  // L_kk and W received (P > 1)
  cudaEvent_t ev_row = nullptr;                  // row broadcast of the current panel done (virtual)
  cudaEvent_t ev_join[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> u2b, u2e;             // timing of the bulk trailing update
  int n_u2 = 0;
  double u2_flops = 0.0;
  int g_n_u2 = 0;                                // n_u2 / u2_flops of the captured graph
  double g_u2_flops = 0.0;
  std::vector<cudaEvent_t> u1b, u1e;             // timing of the lookahead updates U1
  int n_u1 = 0;
  double u1_flops = 0.0;
  int g_n_u1 = 0;
  double g_u1_flops = 0.0;
};

}  // namespace exageo

struct exageo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nb_opt = 0;
  int ind = 0;         // IND approximation: diagonal super tiles of `ind` tiles (0 = exact)
  int metric = 0;      // 0 Euclidean, 1 great-circle (lon/lat degrees)
  double radius = 6371.0;
  int world = 1;       // ranks of the distribution (NCCL processes or virtual ranks)
  int rank = 0;        // this process's rank (NCCL mode), 0 otherwise
  int P = 1, Q = 1;    // process grid (world = P Q)
  bool virt = false;   // virtual ranks: all `world` ranks in this process on one device
  ncclComm_t comm = nullptr;
  ncclComm_t comm_row = nullptr;  // ranks of this process row (Q of them; key q), P > 1 or Q > 1
  ncclComm_t comm_col = nullptr;  // ranks of this process column (P of them; key p)
  std::vector<exageo::RankState> rs;
  double* parts = nullptr;    // 2 * world doubles: per-rank {sum log L_ii, sum y^2}
  double* out3 = nullptr;     // {loglik, logdet, quad}
  double* mtab = nullptr;     // per-theta Chebyshev table of the Matern function (K1T)
  int64_t* pivbuf = nullptr;  // NCCL mode: all-reduced first failing pivot
  double* vec = nullptr;      // 4 n staging for host-pointer entry points
  int64_t vec_cap = 0;
  double* zsum = nullptr;     // NCCL TRMV: local partial z (n doubles)
  exageo::Layout G;           // global geometry (n, nb, T, N); rank/world unset
  bool have_matrix = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_wait = nullptr;  // exageo_stream_wait
  // tile-task executor (dag.cu; exageo_opts.tile_tasks): the whole factorization of a
  // single-rank context as one persistent kernel running the 64 x 64 tile DAG
  int tile_tasks = 0;          // 0 automatic (n <= tile_tasks_auto_n()), 1 always when eligible, -1 never
  int dag_nt = 0, dag_ntasks = 0, dag_nproc = 0;  // plan of the uploaded task list
  int dag_t0 = 0, dag_plan_t0 = -1;  // first 64-block column of the executor run (tail hand-off)
  int4* dag_tasks = nullptr;
  int* dag_sync = nullptr;     // ticket + tile / z version counters
  double* dag_W = nullptr;     // W_k = L_kk^{-1}, 64 x 64 per tile column
  int dag_cap_nt = 0;          // nt the sync / W buffers are sized for
  int64_t dag_cap_tasks = 0;
  bool dag_finished = false;   // the last factorization ran on the executor (out3 written by it)
  // fused generation: launch_generate defers Sigma's tiles inside n to the executor's GEN tasks
  bool dag_gen = false;        // the next executor launch generates (params below)
  double* dag_res = nullptr;   // set during graph capture: pinned result block the executor writes
  exageo::MaternConsts dag_mc{};
  const double *dag_x = nullptr, *dag_y = nullptr, *dag_z = nullptr;
  std::vector<const void*> dag_init_key;  // (ws, n, nb) whose padding / z block was generated
  int gen_launches = 0;        // kernels that take theta (K1T, K1, executor with GEN), counted per capture
  // tracing (env EXAGEO_TILE_TASK_TRACE=<file>): per ticket {cta, grabbed, ready, done} of the
  // last evaluation, written as text when the context is destroyed
  std::string dag_trace_path;
  unsigned long long* dag_trace = nullptr;
  int64_t dag_trace_cap = 0;
  int64_t kernels = 0;
  std::string err;
  // CUDA-graph replay of a whole evaluation (exageo_opts.graphs; api.cu loglik_graph)
  int graphs = 0;                          // 0 automatic, 1 always, -1 never
  bool capturing = false;                  // inside cudaStreamBeginCapture on `stream`
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<cudaGraphNode_t> gen_nodes;  // K1 nodes: theta is updated per replay
  std::vector<const void*> gkey;           // sizes + every device pointer the graph bakes in
  int64_t graph_kernels = 0;
  void* h_res = nullptr;                   // pinned: {loglik, logdet, quad, -} + one info word per rank
};

namespace exageo {
// One evaluation of l(theta) on device-resident inputs (api.cu), optionally with its parts
// log|Sigma| and z^T Sigma^-1 z. Returns EXAGEO_OK, EXAGEO_ENOTPD (ll = -inf), or another error.
exageo_status eval_loglik(exageo_ctx* c, const exageo_theta* t, int64_t n, const double* x_d, const double* y_d,
                          const double* z_d, double* ll, double* logdet = nullptr, double* quad = nullptr);
// Device staging buffer of at least 4 n doubles (api.cu).
exageo_status staging(exageo_ctx* c, int64_t n, double** buf);
exageo_status set_error(exageo_ctx* c, exageo_status s, const std::string& msg);
}  // namespace exageo
