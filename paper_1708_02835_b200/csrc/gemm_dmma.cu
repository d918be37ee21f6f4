#include <cstdlib>
// gemm_dmma.cu -- instantiations and launchers of the DMMA contraction kernels
// (gemm_dmma.cuh) used by the tiled Cholesky schedule in api.cu.
#include "gemm_dmma.cuh"

namespace exageo {

namespace {
using namespace gemm;
// 64 x 64 tiles, 4 warps of 32 x 32, BK 16 x 2 stages, 4 CTAs per SM; accumulating
// launches start from C (PRE) so the epilogue only stores. tools/gemm_tune.cu, U2(0) at
// n = 100k (algorithmic TFLOP/s): 128x64 at 2 CTAs/SM 30.3; 64x64x8 x4 33.27;
// 64x64x8 x4 PRE 33.37; 64x64x16 x2 PRE 33.56 (90% of the 37.2 TF DMMA peak).
using PanelCfg = Cfg<64, 64, 16, 2, 2, 2, 4>;
using TrailCfg = Cfg<64, 64, 16, 2, 2, 2, 4>;
}  // namespace

cudaError_t gemm_init() {
  cudaError_t e;
  if ((e = set_smem<PanelCfg, true, DenseMap>()) != cudaSuccess) return e;
  if ((e = set_smem<PanelCfg, false, DenseMap>()) != cudaSuccess) return e;
  if ((e = set_smem<TrailCfg, true, SyrkMap>()) != cudaSuccess) return e;
  return set_smem<TrailCfg, true, Syrk2DMap>();
}

void launch_gemm_panel(int64_t M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* C, int64_t ldc, bool accumulate, const int* info, cudaStream_t s, bool pdl) {
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
  if (accumulate) launch<PanelCfg, true, DenseMap, true>(map, info, s, pdl);
  else launch<PanelCfg, false>(map, info, s, pdl);
}

// super-panel size of the trailing update (single rank): the super panel's B operand
// (group * nb rows of panel k, group * nb^2 doubles) is kept near 16 MB so it stays
// L2-resident (nb = 512: 8 panels; nb = 1024: 2; measured: 8 x 1024 = 64 MB thrashes and
// re-reads 225 GB per U2(0) at n = 100k). EXAGEO_SYRK_GROUP overrides (tuning).
int syrk_group(int nb) {
  static const int forced = [] {
    const char* e = getenv("EXAGEO_SYRK_GROUP");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= 64 ? v : 0;
  }();
  if (forced) return forced;
  const int64_t g = ((int64_t)2 << 20) / ((int64_t)nb * nb);  // 2 Mi doubles = 16 MiB
  return (int)(g < 1 ? 1 : (g > 8 ? 8 : g));
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
  map.row_end = (int64_t)L.sb_end(k) * L.nb;  // N unless IND
  map.group = L.world == 1 ? syrk_group(L.nb) : 1;  // super panels: panel k's rows read once per group
  launch<TrailCfg, true, SyrkMap, true>(map, info, s);
}

void launch_syrk_panels_2d(const Layout& L, double* ws, const double* const* slices, const int64_t* slds, int k,
                           int J0, int npan, const int* info, cudaStream_t s) {
  if (npan <= 0) return;
  Syrk2DMap map;
  map.L = L;
  map.ws = ws;
  for (int i = 0; i < kMaxP; ++i) {
    map.slice[i] = i < L.P ? slices[i] : nullptr;
    map.sld[i] = i < L.P ? slds[i] : 0;
  }
  map.k = k;
  map.J0 = J0;
  map.npan = npan;
  map.Eb = L.sb_end(k);
  launch<TrailCfg, true, Syrk2DMap, true>(map, info, s);
}

}  // namespace exageo
