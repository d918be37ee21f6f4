/*
 * exageo.h -- C ABI of the B200-native exact Gaussian log-likelihood library
 * (hot path of ExaGeoStat, arXiv 1708.02835). libexageo.so implements every
 * function declared here; the Python binding paper_1708_02835_b200 mirrors the
 * names one to one.
 *
 * Citations: "P:<line>" = PAPER.md line of arXiv 1708.02835 (LaTeX text);
 * "R<k>" = reading k in DESIGN.md (where the paper is silent or garbled).
 *
 * Conventions (all functions):
 *   - Plain pointers and sizes only. Unless a name ends in _dev, array
 *     arguments are HOST pointers owned by the caller; the library copies them.
 *     *_dev functions take DEVICE pointers on the context's device and enqueue
 *     work on the context's stream (they synchronise only where they return a
 *     host scalar, as documented).
 *   - Matrices are column-major with an explicit leading dimension.
 *   - Every function returns an exageo_status; nothing aborts the process.
 *     On failure, exageo_last_error(ctx) describes the cause.
 *   - theta = (theta1, theta2, theta3) = (variance, range, smoothness) of the
 *     Matern covariance Eq. (2); each must be finite and > 0,
 *     otherwise EXAGEO_EINVAL.
 *   - The library never falls back to a CPU implementation: without a usable
 *     CUDA device, context creation fails with EXAGEO_ECUDA.
 */
#ifndef EXAGEO_H
#define EXAGEO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Matern parameter vector theta. */
typedef struct {
  double sigma2; /* theta1 > 0: variance              */
  double beta;   /* theta2 > 0: spatial range          */
  double nu;     /* theta3 > 0: smoothness             */
} exageo_theta;

typedef enum {
  EXAGEO_OK = 0,
  EXAGEO_EINVAL = -1,  /* invalid argument (theta <= 0 / non-finite, n < 1, NULL, bad ld) */
  EXAGEO_ENOTPD = -2,  /* Sigma(theta) not positive definite; info.npd_pivot = global pivot */
  EXAGEO_ENOMEM = -3,  /* tile workspace does not fit in device memory                      */
  EXAGEO_ECUDA = -4,   /* CUDA runtime error (no device, launch failure, ...)                */
  EXAGEO_ENCCL = -5,   /* reserved: collective failure (multi-GPU)                           */
  EXAGEO_EFIT = -6     /* reserved: every optimizer evaluation failed (exageo_mle)           */
} exageo_status;

/* Opaque context: device, stream, tile workspace (panel layout, DESIGN.md
 * "Data layout"), per-step events. Not thread-safe; one per device/stream. */
typedef struct exageo_ctx exageo_ctx;

typedef struct {
  int device;   /* CUDA device ordinal                                               */
  int nb;       /* tile size (multiple of 128); 0 = automatic (single GPU: 128 below n = 6000, 512
                   below 20k, 1024 below 56k, else 2048; world > 1: at most 512)               */
  void* stream; /* cudaStream_t to run on; NULL = the library creates its own stream */
  /* Distribution: the tiles are dealt 2-D block-cyclically over a
   * grid_rows x (world / grid_rows) process grid (1 x world by default: panel j on rank
   * j % world); each step factors panel k on its process column, broadcasts its slices along
   * the process rows and then the process columns (NCCL), and the evaluation finishes with
   * an all-reduce. world <= 1: single GPU. Experimental beyond one GPU: the schedule is
   * verified on virtual ranks and a single-rank communicator; multi-rank NCCL transport has
   * not run on hardware (one-GPU build box). */
  int world;            /* number of ranks (one process per GPU, NCCL over NVLink)      */
  int rank;             /* this process's rank, 0 <= rank < world                        */
  const void* nccl_id;  /* 128-byte ncclUniqueId from exageo_nccl_unique_id on rank 0,
                           identical on every rank (world > 1)                           */
  int virtual_ranks;    /* > 1: run that many ranks inside this process on one device,
                           panel broadcasts as device copies (tests the distributed
                           schedule on one GPU); excludes world > 1                      */
  int ind_tiles;        /* > 0: Independent Blocks (IND) approximation: tiles
                           outside the diagonal super tiles of ind_tiles x ind_tiles tiles
                           are annihilated (Sigma becomes block diagonal over consecutive
                           groups of ind_tiles * nb locations) and the factorization skips
                           them; loglik, mle and predict (Sigma22 only) use the masked
                           matrix. 0: exact.                                             */
  int distance;         /* 0: Euclidean r = ||s - s'||. 1: great-circle distance by the
                           haversine formula: x = longitude, y = latitude in
                           degrees, r = 2 R asin(sqrt(hav(dlat) + cos lat1 cos lat2 hav(dlon))) */
  double radius;        /* sphere radius R for distance = 1 (units of theta2); 0 = 6371     */
  int graphs;           /* CUDA-graph replay of whole evaluations (capture once per problem
                           shape and buffer set, then replay with theta patched into the
                           generator nodes; with NCCL the collectives are graph nodes too): 0 = automatic
                           (n <= 32768, a non-default stream), 1 = always when possible, -1 = never */
  int grid_rows;        /* P of the P x Q process grid (the 2-D block-cyclic
                           distribution of P:450-453): tile (I, J) on rank (I mod P) Q + J mod Q,
                           Q = ranks / P. 0 or 1 = 1 x ranks (panel j on rank j % ranks); must
                           divide world (or virtual_ranks); P <= 8. NCCL row and column
                           communicators are split from the world communicator.             */
  int tile_tasks;       /* single-rank contexts (no IND): run the factorization as ONE persistent
                           kernel that executes the 64 x 64 tile-task DAG on the device (the
                           paper's dynamic runtime, moved onto the GPU; dag.cu) instead
                           of stream-launched panel kernels. 0 = automatic (n <= 3200),
                           1 = always when eligible, -1 = never                              */
} exageo_opts;

/* Per-evaluation details of exageo_loglik*. */
typedef struct {
  double loglik;      /* l(theta), Eq. (1)                                   */
  double logdet;      /* log|Sigma| = 2 sum log L_ii (R5)                    */
  double quad;        /* z^T Sigma^{-1} z = ||L^{-1} z||^2 (R6, R7)          */
  int64_t npd_pivot;  /* -1, or the 0-based global index of the first non-positive pivot */
  int64_t n, nb, ntiles; /* problem size, tile size, T = ceil(n/nb)           */
  double flops;       /* n^3/3 Cholesky flop count used for TFLOP/s */
  double ms_total;    /* device time of the whole evaluation (CUDA events)    */
  double ms_gen;      /* device time of the covariance generation (Alg. 2 l.2) */
  double ms_chol;     /* device time of factorization + fused forward solve   */
  double ms_reduce;   /* device time of the log-det / dot reduction            */
  int64_t kernels;    /* number of kernel launches this evaluation issued     */
  /* dominant kernel (the bulk trailing update U2 of each step): */
  int64_t trailing_launches; /* launches of the bulk trailing-update kernel          */
  double ms_trailing;        /* sum of their durations (CUDA events on their stream) */
  double trailing_flops;     /* algorithmic flops of those launches: 2 nb per (row, column)
                                pair of the true lower triangle updated, incl. the z row */
  /* the same trailing-update kernel over all its launches of the evaluation -- the bulk
     updates U2 and the lookahead updates U1 of the next panel, which run concurrently on
     another stream: their algorithmic flops and the union of their [start, end] spans */
  int64_t update_launches;
  double ms_update_union;
  double update_flops;
} exageo_loglik_info;

/* Human-readable name of a status. Never NULL. */
const char* exageo_strerror(exageo_status s);

/* Message of the most recent failure on ctx (or of the last context creation
 * when ctx is NULL). Valid until the next call on ctx. Never NULL. */
const char* exageo_last_error(const exageo_ctx* ctx);

/* Write a fresh NCCL unique id (128 bytes) to out (len >= 128). Call on rank 0 and
 * hand the bytes to every rank's exageo_opts.nccl_id (e.g. over torch.distributed). */
exageo_status exageo_nccl_unique_id(void* out, size_t len);

/* Create a context on opts->device. opts may be NULL (device 0, automatic nb,
 * own stream, single GPU). Fails with EXAGEO_ECUDA if no CUDA device is usable.
 * With opts->world > 1 the call is collective: every rank must call it (NCCL
 * communicator initialisation). Every later call on a distributed context is
 * collective too, with identical arguments on all ranks; results (l, info) are
 * returned on every rank. */
exageo_status exageo_create(exageo_ctx** ctx, const exageo_opts* opts);
void exageo_destroy(exageo_ctx* ctx);

/* Bytes of device workspace exageo_loglik needs for n locations with tile
 * size nb (0 = automatic): 8 * nb * sum_j (N - j*nb + 128), N = T*nb
 * (lower block-column panels plus the z row block). */
size_t exageo_workspace_bytes(int64_t n, int nb);

/* Bytes of device workspace one rank of a distributed context needs: its local panels of the
 * 2-D block-cyclic layout -- the tile rows I = p mod P, I >= J, of its tile
 * columns J = q mod Q, plus the z row block on the process row that holds it -- for n
 * locations, tile size nb (0 = automatic as on a context with `world` ranks), `world` ranks
 * on a grid_rows x (world / grid_rows) grid (0 = 1 x world) and rank = p Q + q. Host-only (no
 * device needed); the ranks' values sum to exageo_workspace_bytes(n, nb) plus 2 KB per rank.
 * Returns 0 on invalid arguments. */
size_t exageo_rank_workspace_bytes(int64_t n, int nb, int world, int grid_rows, int rank);

/* Hand the context a caller-owned device buffer (e.g. a torch tensor) to use
 * as tile workspace; it must stay alive while the context uses it. ptr = NULL
 * returns to library-managed allocation. ptr must be 256-byte aligned (the kernels
 * store double2 and load 16-byte cp.async chunks), else EXAGEO_EINVAL. */
exageo_status exageo_set_workspace(exageo_ctx* ctx, void* ptr, size_t bytes);

/* Order the context's stream after all work submitted so far to `stream` (a cudaStream_t
 * of the context's device, e.g. torch's current stream): records an event on `stream` and
 * makes the context stream wait on it (no host synchronisation). The *_dev entry points
 * read caller-owned device buffers on the context stream; call this first whenever those
 * buffers were written on another stream. stream == NULL means the legacy default stream.
 * EXAGEO_ECUDA on a CUDA failure. */
exageo_status exageo_stream_wait(exageo_ctx* ctx, void* stream);

/* Jittered-grid locations (Sec. 7.1; R1-R3):
 *   s_q = ((r - 0.5 + X_rl)/g, (l - 0.5 + Y_rl)/g), g = ceil(sqrt n),
 *   X, Y ~ U(-0.4, 0.4) from counter-based SplitMix64 streams; for non-square
 *   n the n grid cells with the smallest SplitMix64 keys are kept, in
 *   row-major cell order. Integer RNG + IEEE arithmetic without contraction:
 *   bit-exact across platforms. x, y: host arrays of n doubles (caller-owned).
 * Computed on the host (input preparation, not the timed path). */
exageo_status exageo_gen_locations(int64_t n, uint64_t seed, double* x, double* y);

/* Dense Matern covariance block, Eq. (2) (Alg. 3 l.3-6):
 *   C[i + j*ldc] = C(||s1_i - s2_j||; theta), 0 <= i < m, 0 <= j < n,
 * with C(0) = theta1 (R9). Host arrays x1,y1 (m), x2,y2 (n), C (ldc*n,
 * ldc >= m). Computed on the GPU by the same device evaluator as the tile
 * generator. */
exageo_status exageo_matern_cov(exageo_ctx* ctx, const exageo_theta* theta, int64_t m, const double* x1,
                                const double* y1, int64_t n, const double* x2, const double* y2, double* C,
                                int64_t ldc);

/* Exact Gaussian log-likelihood, Eq. (1) by Alg. 2:
 *   Sigma = genCovMatrix(theta); Sigma = L L^T; y = L^{-1} z;
 *   l = -0.5 y^T y - 0.5 (2 sum log L_ii) - (n/2) log(2 pi).
 * x, y, z: host arrays of n doubles. On success *loglik is set; info (may be
 * NULL) receives the details. Not positive definite -> EXAGEO_ENOTPD with
 * info->npd_pivot set and *loglik = -inf. Host<->device copies included. */
exageo_status exageo_loglik(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x,
                            const double* y, const double* z, double* loglik, exageo_loglik_info* info);

/* Same as exageo_loglik with DEVICE arrays x_d, y_d, z_d (n doubles each) on
 * the context's device. Enqueued on the context stream; returns after the
 * 32-byte result has been copied back (the only synchronisation). */
exageo_status exageo_loglik_dev(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x_d,
                                const double* y_d, const double* z_d, double* loglik,
                                exageo_loglik_info* info);

/* Synthetic data generator, Alg. 1 (R18): z = L e with
 * Sigma(theta) = L L^T. The normal variates e (n doubles, host) are an input.
 * Writes z (n doubles, host). Non-PD -> EXAGEO_ENOTPD. */
exageo_status exageo_simulate(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x,
                              const double* y, const double* e, double* z);

/* Maximum-likelihood estimate theta_hat = argmax_theta l(theta) over the box
 * lo <= theta <= hi, the paper's optimization loop with a
 * derivative-free bound-constrained search (R16): Nelder-Mead on log(theta), trial
 * points projected onto the box, restarted from the best vertex while that improves;
 * each evaluation is one exageo_loglik on inputs copied to the device once. A
 * parameter with lo == hi is held fixed. Non-positive-definite evaluations count as
 * l = -inf. Stops when the simplex diameter in log(theta) (= relative change
 * of theta) is below xtol_rel, or after max_evals evaluations.
 * x, y, z: host arrays of n doubles. Outputs: *theta_hat, *loglik = l(theta_hat)
 * (may be NULL), *nevals (may be NULL), trace (may be NULL): 4 doubles
 * {theta1, theta2, theta3, l} per evaluation, room for max_evals.
 * EXAGEO_EINVAL unless 0 < lo <= start <= hi; EXAGEO_EFIT if every evaluation failed.
 * Collective on distributed contexts: every rank runs the same deterministic search
 * on the same (all-reduced) l values. */
exageo_status exageo_mle(exageo_ctx* ctx, int64_t n, const double* x, const double* y, const double* z,
                         const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start, double xtol_rel,
                         int max_evals, exageo_theta* theta_hat, double* loglik, int* nevals, double* trace);

/* Same contract as exageo_mle, but the search runs over (theta2, theta3) only: theta1
 * is profiled out in closed form. Eq. (2) is linear in theta1, Sigma = theta1 R, so one
 * factorization of R (theta1 = 1) gives log|R| and q = z^T R^-1 z, and
 *   l(s, theta2, theta3) = -q / (2 s) - (n log s + log|R|) / 2 - (n / 2) log 2 pi
 * is maximised over s in [lo.sigma2, hi.sigma2] by s = clamp(q / n). Same maximiser as
 * exageo_mle with one dimension fewer (fewer evaluations); the trace records s. */
exageo_status exageo_mle_profile(exageo_ctx* ctx, int64_t n, const double* x, const double* y, const double* z,
                                 const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start,
                                 double xtol_rel, int max_evals, exageo_theta* theta_hat, double* loglik,
                                 int* nevals, double* trace);

/* Options of exageo_mle_ex. */
typedef struct {
  double xtol_rel; /* stop when the search scale in log(theta) (simplex diameter / trust-region
                      radius) falls below this                                                 */
  int max_evals;   /* evaluation budget                                                        */
  int profile;     /* 1: theta1 profiled out in closed form (as exageo_mle_profile)            */
  int method;      /* 0: Nelder-Mead (as exageo_mle); 1: quadratic-model trust region (the
                      BOBYQA/UOBYQA class): fully determined quadratic interpolation
                      models on (d+1)(d+2)/2 points, exact box-constrained trust-region steps,
                      Lagrange-function point replacement; falls back to Nelder-Mead if the
                      initial interpolation set cannot be evaluated                           */
} exageo_mle_opts;

/* exageo_mle / exageo_mle_profile with the search method selectable (exageo_mle_opts);
 * same arguments, outputs and errors (EXAGEO_EINVAL also for a bad method). */
exageo_status exageo_mle_ex(exageo_ctx* ctx, int64_t n, const double* x, const double* y, const double* z,
                            const exageo_theta* lo, const exageo_theta* hi, const exageo_theta* start,
                            const exageo_mle_opts* opts, exageo_theta* theta_hat, double* loglik, int* nevals,
                            double* trace);

/* Kriging prediction, Eq. (5) by Alg. 3 (R19):
 *   Sigma22 = L L^T (with the forward solve y = L^{-1} z fused into the factorization),
 *   L^T w = y (blocked backward solve), znew = Sigma12 w with the m x n block Sigma12
 *   generated on the fly (never stored); zero mean (mu1 = mu2 = 0).
 * x, y, z: the n observed locations and measurements; xnew, ynew: the m prediction
 * locations; znew: m predictions. Host arrays. Non-PD -> EXAGEO_ENOTPD.
 * Collective on distributed contexts: per panel j (from the last) the ranks of its process
 * column reduce their partial sums onto the diagonal rank, which solves with L_jj and
 * broadcasts w_j (1 x Q grids: the panel's owner solves alone). */
exageo_status exageo_predict(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x,
                             const double* y, const double* z, int64_t m, const double* xnew, const double* ynew,
                             double* znew);

/* exageo_predict plus the kriging (conditional) variance of every new site,
 *   var_i = theta1 - sigma_i^T Sigma22^{-1} sigma_i = theta1 - ||L^{-1} sigma_i||^2,
 * sigma_i = Sigma21[:, i] (the simple-kriging variance belonging to Eq. (5)),
 * from the same factor: batches of new sites, Sigma21 generated on the GPU, a blocked
 * multi-right-hand-side forward solve with L (diagonal-tile substitution + DMMA update of
 * the rows below), column sums of squares. var: host array of m doubles. Work ~ n^2 m flop.
 * Collective on distributed contexts (NCCL or virtual ranks, any P x Q grid): per tile row I
 * the ranks of process row I mod P reduce their partial updates onto the diagonal rank, which
 * solves with L_II and broadcasts V_I down its process column, whose ranks update their tile
 * rows below; the diagonal ranks' column sums are all-reduced. Tile size nb <= 1024
 * (EXAGEO_EINVAL otherwise). */
exageo_status exageo_predict_var(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x,
                                 const double* y, const double* z, int64_t m, const double* xnew,
                                 const double* ynew, double* znew, double* var);

/* --- Stage-level entry points (same kernels as exageo_loglik_dev, exposed
 *     so that each step of Alg. 2 can be checked on its own). ---------- */

/* Alg. 2 l.2: generate Sigma(theta) into the workspace (lower panels, identity
 * padding, z in the z row block). Device arrays. Enqueued, no sync. */
exageo_status exageo_stage_generate_dev(exageo_ctx* ctx, const exageo_theta* theta, int64_t n, const double* x_d,
                                        const double* y_d, const double* z_d);
/* Alg. 2 l.3-4: factor the workspace in place (Sigma -> L) with the fused
 * forward solve of the z row (y = L^{-1} z). Enqueued, no sync. */
exageo_status exageo_stage_factor(exageo_ctx* ctx);
/* Alg. 2 l.5-7: reductions; synchronises and writes out[3] =
 * {loglik, logdet, quad} (host) and *npd_pivot (host, may be NULL). */
exageo_status exageo_stage_finish(exageo_ctx* ctx, double* out3, int64_t* npd_pivot);
/* Copy the lower triangle (incl. diagonal) of the current workspace matrix
 * (Sigma after generate, L after factor) to host dense column-major
 * dst[i + j*ld], 0 <= j <= i < n; the strict upper triangle of dst is not
 * written. Synchronises. The read_* functions return the columns held by this
 * process (all of them unless world > 1 with NCCL; other columns read as 0).
 * read_lower stages a dense n x n copy on the device and the host, so it is limited
 * to n <= 32768 (EXAGEO_EINVAL above; use exageo_read_entries for sampled entries). */
exageo_status exageo_read_lower(exageo_ctx* ctx, double* dst, int64_t ld);
/* Copy the current z row (z after generate, y = L^{-1} z after factor) to the
 * host array dst (n doubles). Synchronises. */
exageo_status exageo_read_zrow(exageo_ctx* ctx, double* dst);
/* Gather count entries (rows[i], cols[i]) of the current workspace matrix,
 * 0 <= cols[i] <= rows[i] < n (host int64 arrays), into host out[count]
 * (sampled full-size checks). EXAGEO_EINVAL on an index outside the lower
 * triangle. Synchronises. */
exageo_status exageo_read_entries(exageo_ctx* ctx, int64_t count, const int64_t* rows, const int64_t* cols,
                                  double* out);

#ifdef __cplusplus
}
#endif
#endif /* EXAGEO_H */
