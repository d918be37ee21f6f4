// internal.h -- shared declarations of the sm_100a kernels and their host launchers.
//
// Data layout of the tile workspace ("lower block-column panels"):
//   n locations, tile size nb (multiple of 128), T = ceil(n/nb), N = T*nb.
//   Panel j (0 <= j < T) holds global rows j*nb .. N-1 of columns j*nb .. j*nb+nb-1
//   followed by ZR = 128 extra rows (the "z row block": its first row is z^T,
//   the rest zeros), column-major with leading dimension ld_j = N - j*nb + ZR.
//   Row r = N is the z row: after the factorization it holds y = L^{-1} z
//   (the forward solve of Alg. 2 l.4 fused as an augmented row).
//   Rows/cols n..N-1 are identity padding (exact for log|Sigma| and z^T Sigma^-1 z).
//
// Distribution: 2-D block-cyclic over a P x Q process grid, the layout of
// ScaLAPACK the paper builds on: tile (I, J) lives on rank (I mod P, J mod Q),
// rank id = p Q + q. A rank stores, for each of its tile columns J (J = q mod Q), its tile
// rows I >= J (I = p mod P) stacked into one column-major "local panel" of lrows(J) rows,
// followed by the z row block when its process row holds tile row T (T mod P == p); the
// local panels lie back to back in increasing J. Local row lr < lrows(J) of panel J is global
// row grow(J, lr); local panel J starts at ws + off(J) with leading dimension ld(J).
// P = 1 is the 1-D column-cyclic layout (panel j on rank j % world, every tile row local:
// ld(j) = N - j nb + ZR, closed-form offsets); world = 1 is the single-GPU case.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <vector>

namespace exageo {

constexpr int ZR = 128;  // height of the z row block appended to every panel
constexpr int PB = 64;   // inner panel block (POTRF block size)
constexpr int kQuadBlocks = 148;  // CTAs of the local dot-product reduction
constexpr int kMaxP = 8;          // process-grid rows supported by the trailing-update map

struct Layout {
  int64_t n = 0;   // true problem size
  int nb = 0;      // tile size
  int T = 0;       // number of panels (tile columns)
  int64_t N = 0;   // padded size T*nb
  int rank = 0;    // this rank = p Q + q
  int world = 1;   // number of ranks = P Q
  int P = 1, Q = 1, p = 0, q = 0;  // process grid and this rank's coordinates
  int ind = 0;     // IND approximation: diagonal super tiles of `ind` tiles; 0 = exact
  // P > 1: offsets (doubles) of the local panels, owned() + 1 entries (host and device copies)
  const int64_t* offs_h = nullptr;
  const int64_t* offs_d = nullptr;

  // one past the last panel of the diagonal super tile holding panel k (T when exact)
  __host__ __device__ int sb_end(int k) const {
    if (ind <= 0) return T;
    const int e = (k / ind + 1) * ind;
    return e < T ? e : T;
  }
  // IND: is global element (r, c) (r, c < N) inside a diagonal super tile?
  __host__ __device__ bool in_super_tile(int64_t r, int64_t c) const {
    if (ind <= 0) return true;
    const int64_t w = (int64_t)ind * nb;
    return r / w == c / w;
  }

  // ---- tile rows of process row pp ----
  // local tile rows of process row pp (tiles I = pp mod P, I < T)
  __host__ __device__ int Tp_of(int pp) const { return T > pp ? (T - pp + P - 1) / P : 0; }
  // index of the first local tile row of process row pp that is >= J (= the count of those < J)
  __host__ __device__ int i0_of(int pp, int J) const { return J <= pp ? 0 : (J - pp + P - 1) / P; }
  __host__ __device__ bool has_z_of(int pp) const { return T % P == pp; }
  __host__ __device__ int64_t lrows_of(int pp, int J) const {
    const int t = Tp_of(pp) - i0_of(pp, J);
    return t > 0 ? (int64_t)t * nb : 0;
  }
  __host__ __device__ int64_t ld_of(int pp, int J) const {
    return P == 1 ? N - (int64_t)J * nb + ZR : lrows_of(pp, J) + (has_z_of(pp) ? ZR : 0);
  }
  // ---- this rank ----
  __host__ __device__ int Tp() const { return Tp_of(p); }
  __host__ __device__ int i0(int J) const { return P == 1 ? J : i0_of(p, J); }
  __host__ __device__ bool has_z() const { return has_z_of(p); }
  __host__ __device__ int64_t lrows(int J) const { return P == 1 ? N - (int64_t)J * nb : lrows_of(p, J); }
  __host__ __device__ int64_t ld(int J) const { return ld_of(p, J); }
  // global row of local row lr < lrows(J) of local panel J
  __host__ __device__ int64_t grow(int J, int64_t lr) const {
    if (P == 1) return (int64_t)J * nb + lr;
    const int64_t t = lr / nb;
    return ((int64_t)p + ((int64_t)i0(J) + t) * P) * nb + lr % nb;
  }
  // local row of global row r (r >= N: the z row block) in local panel J; -1 if not stored here
  __host__ __device__ int64_t lrow(int J, int64_t r) const {
    if (r >= N) return has_z() ? lrows(J) + (r - N) : -1;
    if (r < (int64_t)J * nb) return -1;
    const int I = (int)(r / nb);
    if (I % P != p) return -1;
    return (int64_t)((I - p) / P - i0(J)) * nb + r % nb;
  }
  // tile column j is stored on this rank's process column
  __host__ __device__ bool owns(int j) const { return j % Q == q; }
  // the rank holding the diagonal tile (j, j): it factors panel j
  __host__ __device__ int owner(int j) const { return (j % P) * Q + j % Q; }
  __host__ __device__ bool diag(int j) const { return j % Q == q && j % P == p; }
  // number of tile columns this rank stores
  __host__ __device__ int owned() const { return T > q ? (T - q + Q - 1) / Q : 0; }
  // j of the m-th owned tile column
  __host__ __device__ int owned_panel(int m) const { return q + m * Q; }
  // first owned tile column >= j
  __host__ __device__ int first_owned_from(int j) const {
    const int d = ((q - j) % Q + Q) % Q;
    return j + d;
  }
  // local offset (doubles) of the m-th owned panel; P = 1:
  //   nb * sum_{i<m} ld(q + i Q) = nb [m (N + ZR - q nb) - Q nb m (m-1)/2]
  __host__ __device__ int64_t off_m(int64_t m) const {
    if (P == 1) return (int64_t)nb * (m * (N + ZR - (int64_t)q * nb) - (int64_t)Q * nb * (m * (m - 1) / 2));
#ifdef __CUDA_ARCH__
    return offs_d[m];
#else
    return offs_h[m];
#endif
  }
  // local offset of owned panel j
  __host__ __device__ int64_t off(int j) const { return off_m((j - q) / Q); }
  // local storage (doubles)
  __host__ __device__ int64_t total() const { return off_m(owned()); }
};

// Per-theta constants of the Matern evaluator (computed on the host in long
// double, see matern.cu): Eq. (2) prefactor theta1 / (2^(nu-1) Gamma(nu)) and
// Temme's coefficients for mu = nu - round(nu).
struct MaternConsts {
  double theta1, inv_theta2, nu;
  double pref;          // theta1 / (2^(nu-1) Gamma(nu))
  double mu;            // nu - nl, |mu| <= 1/2
  int nl;               // round(nu) (half up)
  int kind;             // 0 general, 1: nu=1/2, 2: nu=3/2, 3: nu=5/2
  double gam1, gam2;    // Temme gamma_1(mu), gamma_2(mu)
  double gampl, gammi;  // 1/Gamma(1+mu), 1/Gamma(1-mu)
  double pimu_sin;      // pi mu / sin(pi mu)  (1 at mu = 0)
  int metric;           // 0: Euclidean r = ||s - s'||; 1: great-circle (haversine)
  double radius;        // sphere radius for the great-circle distance (length units of theta2)
};

// Set kernel attributes (dynamic shared memory) on the current device.
cudaError_t gemm_init();
cudaError_t potrf_init();
cudaError_t trsv_init();

// ---- launchers (all asynchronous on `s`) ----
// K1T: per-theta Chebyshev table of the Matern function for general nu (matern.cu);
// returns 1 if a table kernel was launched (kind == 0), 0 for the closed forms.
int matern_table_doubles();
int launch_matern_table(const MaternConsts& mc, double* tab, cudaStream_t s);
const void* matern_table_kernel_fn();  // CUDA-graph node identification
// K1: generate this rank's panels of Sigma(theta) (identity padding, z in the z row block);
// tab = the table built by launch_matern_table for this theta (used when kind == 0).
void launch_gen_panels(const Layout& L, double* ws, const MaternConsts& mc, const double* x, const double* y,
                       const double* z, const double* tab, cudaStream_t s);
const void* gen_panels_kernel_fn(int kind);  // the K1 kernel for MaternConsts::kind (CUDA-graph nodes)
// Dense Matern block and kriging sums (build the table themselves into tab when needed).
void launch_matern_dense(const MaternConsts& mc, int64_t m, const double* x1, const double* y1, int64_t n,
                         const double* x2, const double* y2, double* C, int64_t ldc, double* tab, cudaStream_t s);

// C (M x N, ldc) = C - A (M x K, lda) * B (N x K, ldb)^T      (accumulate = true)
// C (M x N, ldc) =     A (M x K, lda) * B (N x K, ldb)^T      (accumulate = false; may alias A when N == K <= 64)
// Variant tuned for N = 64 panel columns.
void launch_gemm_panel(int64_t M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* C, int64_t ldc, bool accumulate, const int* info, cudaStream_t s,
                       bool pdl = false);
// Trailing update by panel k (operand Pk, leading dimension ld(k): a rank's own panel k
// or its received copy) of the owned panels J0, J0 + world, ..., (npan of them):
// A_rc -= sum_t L_rt L_ct for every lower element and the z row of those panels.
void launch_syrk_panels(const Layout& L, double* ws, const double* Pk, int k, int J0, int npan, const int* info,
                        cudaStream_t s);
// The same on a 2-D process grid (P > 1): panel k arrives as P slices (slices[pp] with
// leading dimension slds[pp]: the local panel k of rank (pp, k mod Q)), gemm_dmma.cuh Syrk2DMap.
void launch_syrk_panels_2d(const Layout& L, double* ws, const double* const* slices, const int64_t* slds, int k,
                           int J0, int npan, const int* info, cudaStream_t s);
// Tile-task executor (dag.cu): the factorization (with the fused forward solve) of a
// single-rank layout as one persistent kernel over the 64 x 64 tile DAG -- the whole matrix
// (t0 = 0), or the trailing matrix from 64-block column t0 on, handed over by the stream
// schedule after the panels < t0 (already applied to it; no generation then). dag_plan lists the
// tasks of nt = ceil(n / 64) tile columns in ticket order for nproc CTAs; sync holds
// dag_sync_ints(nt) ints, zeroed before each launch; W holds nt 64 x 64 blocks. The last CTA to
// finish writes out3 = {loglik, logdet, quad} (so no separate reduction kernels follow).
void dag_plan(int nt, int nproc, std::vector<int4>& order);
// Fused generation (Alg. 2 l.2): when generate is set, the executor's GEN tasks write Sigma's
// tiles inside n and the z row (Eq. (2) with mc; tab = the K1T table for general nu) ahead of
// the factorization; otherwise they only mark the tiles ready.
struct DagGen {
  bool generate;
  MaternConsts mc;
  const double* tab;
  const double *x, *y, *z;
};
// CUDA-graph support: does a captured executor node generate, and its argument block with
// a new theta (for cudaGraphExecKernelNodeSetParams).
bool dag_args_generate(const void* args);
void dag_args_with_theta(const void* args, const MaternConsts& mc, std::vector<char>& out);
int dag_sync_ints(int nt);
cudaError_t dag_init();
void launch_dag_factor(const Layout& L, double* ws, const int4* tasks, int ntasks, int nt, int t0, int* sync, double* W,
                       double* slots, int* info, double* out3, double* res_h, unsigned long long* trace,
                       const DagGen& gen, int nctas, cudaStream_t s);
const void* dag_factor_kernel_fn();

// Factor the PB x PB diagonal block at `a` (ld) in place, write W = L^{-1} (PB x PB,
// ld PB) and slot = sum log L_ii; info = first bad global pivot + 1. ncols < PB: only the
// first ncols columns are inside n (the rest is identity padding; only their strips run).
void launch_potrf_block(double* a, int64_t lda, double* W, double* logdet_slot, int* info, int64_t pivot_base,
                        cudaStream_t s, bool pdl = false, int ncols = PB);
// out2 = {sum of this rank's log-det partials (nslots), sum of y_c^2 over this rank's columns};
// scratch: kQuadBlocks doubles.
void launch_local_partials(const Layout& L, const double* ws, const double* slots, int nslots, double* scratch,
                           double* out2, cudaStream_t s);
// key = this rank's first failing global pivot (info - 1), or INT64_MAX when none.
void launch_pivot_key(const int* info, int64_t* key, cudaStream_t s);
// out3 = {loglik, logdet, quad} from nparts pairs {logdet/2 partial, quad partial} summed in order.
void launch_combine(const double* parts, int nparts, int64_t n, double* out3, cudaStream_t s);
// Copy this rank's columns of the lower triangle to dense column-major dst (device).
void launch_read_lower(const Layout& L, const double* ws, double* dst, int64_t ld, cudaStream_t s);
void launch_read_zrow(const Layout& L, const double* ws, double* dst, cudaStream_t s);
// out[i] = entry (rc[i], rc[count + i]) if this rank owns column rc[count + i] (else untouched).
void launch_read_entries(const Layout& L, const double* ws, int64_t count, const int64_t* rc, double* out,
                         cudaStream_t s);
// z (Alg. 1 l.7, dtrmm): part[m][r] = sum over the m-th owned panel's columns c <= r of L_rc e_c
// (part: owned() * N doubles); then z[r] = sum of nparts slices of N doubles.
void launch_trmv_partial(const Layout& L, const double* ws, const double* e, double* part, cudaStream_t s);
void launch_trmv_sum(int64_t n, int64_t N, const double* part, int nparts, double* z, cudaStream_t s);

// K5^T (trsv.cu): one panel step of the backward solve L^T w = y. P = panel j (ld), rows
// local nb .. nb + rows - 1 are global rows row_after .. row_after + rows - 1; w is indexed
// by global row (entries below the panel already solved); writes wj = w[j nb .. j nb + nb).
// part: trsv_chunks(rows) * nb doubles of scratch.
int trsv_chunks(int64_t rows);
void launch_backsolve_panel(const double* P, int64_t ld, int nb, int64_t row_after, int64_t rows,
                            const double* w, double* wj, double* part, cudaStream_t s);
// 2-D layouts: out (nb) = sum over local rows lr0 .. lr0 + rows - 1 of local panel j (global
// row L.grow(j, lr)) of L_rc w_r; part: trsv_chunks(rows) * nb scratch.
void launch_backsolve_partial(const Layout& L, int j, const double* P, int64_t ld, int64_t lr0, int64_t rows,
                              const double* w, double* part, double* out, cudaStream_t s);
// L_jj^T w_j = y_j - sum_s parts[s] with the diagonal tile at the top of P (ld), y_j given.
void launch_tile_solve(const double* P, int64_t ld, int nb, const double* yj, const double* parts, int nparts,
                       double* wj, cudaStream_t s);
// Kriging variance (trsv.cu): multi-RHS forward solve pieces. diag_solve: S (nb x cols, ld
// lds) <- L_jj^{-1} S with the panel's diagonal tile; transpose: Bt = S^T (cols x rows);
// column_var: var_c = theta1 - sum_{k<n} V_kc^2.
void launch_diag_solve_cols(const double* P, int64_t ld, int nb, double* S, int64_t lds, int cols, cudaStream_t s);
void launch_transpose(const double* S, int64_t lds, int rows, int cols, double* Bt, cudaStream_t s);
void launch_column_var(const double* V, int64_t ldv, int64_t n, int cols, double theta1, double* var,
                       cudaStream_t s);
// Distributed kriging variance pieces: dst += src (rows x cols blocks); acc[c] += sum_{r<rows}
// V_rc^2; var[c] = theta1 - acc[c].
void launch_add_block(double* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols, cudaStream_t s);
void launch_colsq_accum(const double* V, int64_t ldv, int rows, int cols, double* acc, cudaStream_t s);
void launch_var_from_acc(const double* acc, int cols, double theta1, double* var, cudaStream_t s);
// K8 (matern.cu): znew_i = sum_j C(||snew_i - s_j||; theta) w_j (Eq. (5), Alg. 3 l.8), the
// covariance block Sigma12 generated on the fly and never stored. part: krige_chunks(n) * m.
int krige_chunks(int64_t n);
void launch_krige(const MaternConsts& mc, int64_t m, const double* xn, const double* yn, int64_t n,
                  const double* x, const double* y, const double* w, double* part, double* znew, double* tab,
                  cudaStream_t s);

}  // namespace exageo
