// internal.h -- shared declarations of the sm_100a kernels and their host launchers.
//
// Data layout of the tile workspace ("lower block-column panels"):
//   n locations, tile size nb (multiple of 128), T = ceil(n/nb), N = T*nb.
//   Panel j (0 <= j < T) holds global rows j*nb .. N-1 of columns j*nb .. j*nb+nb-1
//   followed by ZR = 128 extra rows (the "z row block": its first row is z^T,
//   the rest zeros), column-major with leading dimension ld_j = N - j*nb + ZR.
//   Global element (r, c), c <= r < N + ZR, lives at
//     base + off_j + (c - j*nb) * ld_j + (r - j*nb),   j = c / nb.
//   Row r = N is the z row: after the factorization it holds y = L^{-1} z
//   (the forward solve of Alg. 2 l.4 fused as an augmented row).
//   Rows/cols n..N-1 are identity padding (exact for log|Sigma| and z^T Sigma^-1 z).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace exageo {

constexpr int ZR = 128;  // height of the z row block appended to every panel
constexpr int PB = 64;   // inner panel block (POTRF block size)
constexpr int kOutDoubles = 4 + 148;  // finish(): 3 results + scratch partials

struct Layout {
  int64_t n = 0;   // true problem size
  int nb = 0;      // tile size
  int T = 0;       // number of panels
  int64_t N = 0;   // padded size T*nb
  __host__ __device__ int64_t ld(int j) const { return N - (int64_t)j * nb + ZR; }
  __host__ __device__ int64_t off(int j) const {
    // sum_{t<j} nb * (N - t*nb + ZR)
    return (int64_t)nb * ((int64_t)j * (N + ZR) - (int64_t)nb * ((int64_t)j * (j - 1) / 2));
  }
  __host__ __device__ int64_t total() const { return off(T); }
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
};

// Set kernel attributes (dynamic shared memory) on the current device.
cudaError_t gemm_init();
cudaError_t potrf_init();

// ---- launchers (all asynchronous on `s`) ----
void launch_gen_panels(const Layout& L, double* ws, const MaternConsts& mc, const double* x, const double* y,
                       const double* z, cudaStream_t s);
void launch_matern_dense(const MaternConsts& mc, int64_t m, const double* x1, const double* y1, int64_t n,
                         const double* x2, const double* y2, double* C, int64_t ldc, cudaStream_t s);

// C (M x N, ldc) = C - A (M x K, lda) * B (N x K, ldb)^T      (accumulate = true)
// C (M x N, ldc) =     A (M x K, lda) * B (N x K, ldb)^T      (accumulate = false; may alias A when N == K <= 64)
// Variant tuned for N = 64 panel columns.
void launch_gemm_panel(int64_t M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* C, int64_t ldc, bool accumulate, const int* info, cudaStream_t s);
// Trailing update of step k: for the 128x128 blocks (rb >= cb) of columns >= (k+1) nb,
// rows >= (k+1) nb including the z row block: A_rc -= sum_t L_rt L_ct over panel k.
// Restricted to 128-column blocks cb in [cb_lo, cb_hi) (cb_hi < 0: to the end).
void launch_syrk_trailing(const Layout& L, double* ws, int k, int cb_lo, int cb_hi, const int* info,
                          cudaStream_t s);
// Factor the PB x PB diagonal block at `a` (ld) in place, write W = L^{-1} (PB x PB,
// ld PB) and slot = sum log L_ii; info = first bad global pivot + 1.
void launch_potrf_block(double* a, int64_t lda, double* W, double* logdet_slot, int* info, int64_t pivot_base,
                        cudaStream_t s);
// out[0..2] = {loglik, logdet, quad}, from nslots logdet partial sums and the z row.
// out must hold kOutDoubles doubles (the tail is scratch).
void launch_finish(const Layout& L, const double* ws, const double* slots, int nslots, double* out,
                   cudaStream_t s);
// Copy the lower triangle of the workspace matrix to dense column-major dst (device).
void launch_read_lower(const Layout& L, const double* ws, double* dst, int64_t ld, cudaStream_t s);
void launch_read_zrow(const Layout& L, const double* ws, double* dst, cudaStream_t s);
// out[i] = entry (rc[i], rc[count + i]) of the workspace matrix (lower triangle / z row).
void launch_read_entries(const Layout& L, const double* ws, int64_t count, const int64_t* rc, double* out,
                         cudaStream_t s);
// z = L e with L the factor in the workspace (Alg. 1 l.7, dtrmm): lower TRMV.
// part: scratch of T * N doubles.
void launch_trmv_lower(const Layout& L, const double* ws, const double* e, double* z, double* part,
                       cudaStream_t s);

}  // namespace exageo
