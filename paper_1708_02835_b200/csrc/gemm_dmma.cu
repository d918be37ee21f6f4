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

void launch_syrk_panels(const Layout& L, double* ws, const double* Pk, int k, int J0, int npan, const int* info,
                        cudaStream_t s) {
  if (npan <= 0) return;
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.Pk = Pk;
  map.k = k;
  map.J0 = J0;
  map.npan = npan;
  launch<TrailCfg, true>(map, info, s);
}

}  // namespace exageo
