// gemm_dmma.cu -- instantiations and launchers of the DMMA contraction kernels
// (gemm_dmma.cuh) used by the tiled Cholesky schedule in api.cu.
#include "gemm_dmma.cuh"

namespace exageo {

namespace {
using namespace gemm;
// Panel update / TRSM: 64 x 64 tiles, 4 warps of 32 x 32, BK 8 x 4 stages, 4 CTAs per SM.
using PanelCfg = Cfg<64, 64, 8, 2, 2, 4, 4>;
// Trailing update: 64 x 64 tiles, 4 warps of 32 x 32, BK 8 x 4 stages, 4 CTAs per SM
// (tools/gemm_tune.cu at n=100k: 33.8 TF vs 30.3 for 128x64 at 2 CTAs/SM).
using TrailCfg = Cfg<64, 64, 8, 2, 2, 4, 4>;
// Rasterization band (128-column blocks swept together, see SyrkMap).
constexpr int kTrailBand = 8;
}  // namespace

cudaError_t gemm_init() {
  cudaError_t e;
  if ((e = set_smem<PanelCfg, true, DenseMap>()) != cudaSuccess) return e;
  if ((e = set_smem<PanelCfg, false, DenseMap>()) != cudaSuccess) return e;
  return set_smem<TrailCfg, true, SyrkMap>();
}

void launch_gemm_panel(int64_t M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* C, int64_t ldc, bool accumulate, const int* info, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  DenseMap map;
  map.A = A;
  map.B = B;
  map.C = C;
  map.lda = lda;
  map.ldb = ldb;
  map.ldc = ldc;
  map.M = M;
  map.N = N;
  map.K = K;
  map.mblocks = (int)((M + PanelCfg::BM - 1) / PanelCfg::BM);
  if (accumulate) launch<PanelCfg, true>(map, info, s);
  else launch<PanelCfg, false>(map, info, s);
}

void launch_syrk_trailing(const Layout& L, double* ws, int k, int cb_lo, int cb_hi, const int* info,
                          cudaStream_t s) {
  const int64_t c0 = (int64_t)(k + 1) * L.nb;
  if (c0 >= L.N) return;
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.k = k;
  map.Mb = (int)((L.N - c0) / 128);
  map.cb_lo = cb_lo < 0 ? 0 : cb_lo;
  map.cb_hi = (cb_hi < 0 || cb_hi > map.Mb) ? map.Mb : cb_hi;
  if (map.cb_hi <= map.cb_lo) return;
  map.band = kTrailBand;
  launch<TrailCfg, true>(map, info, s);
}

}  // namespace exageo
