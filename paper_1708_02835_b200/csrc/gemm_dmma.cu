// gemm_dmma.cu -- instantiations and launchers of the DMMA contraction kernels
// (gemm_dmma.cuh) used by the tiled Cholesky schedule in api.cu, and the trailing-update
// kernel (U1/U2: SyrkMap / Syrk2DMap tiles) whose mainloop and epilogue are CUTLASS's SM80
// FP64 tensor-op templates (mma.sync.m8n8k4.f64 = DMMA, 3-stage cp.async, 64x128x16 CTA tile,
// 32x64 warp tiles: the tiling of the cuBLAS DGEMM kernel on this B200) instantiated inside our
// own kernel: the tile -> (A, B, C) pointers come from our maps (triangular tile enumeration,
// panel layout, skipped padding tiles), the epilogue is C <- C - A B^T in place.
#include <cstdlib>

#include "cutlass/cutlass.h"
#include "cutlass/epilogue/thread/linear_combination.h"
#include "cutlass/gemm/kernel/default_gemm.h"
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

// ---- CUTLASS-mainloop trailing update ------------------------------------------------------
// Per CTA tile (BM = 64 rows x BN = 128 columns of C, K = nb) the transposed problem:
// C^T (BN x BM, a row-major view of our column-major C, ld ldc) <- C^T - B (BN x K, column-major,
// ld ldb) . A^T (K x BM, a row-major view of our column-major A, ld lda). tools/gemm_cutlass_tune.cu:
// U2(0) at n = 100k, nb = 2048: 36.28 TF vs 34.25 for gemm_nt_dmma 64x64x16 (profiles/).
using TrailGK = cutlass::gemm::kernel::DefaultGemm<
    double, cutlass::layout::ColumnMajor, 1, double, cutlass::layout::RowMajor, 1, double, cutlass::layout::RowMajor,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<128, 64, 16>,
    cutlass::gemm::GemmShape<64, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 3, false, cutlass::arch::OpMultiplyAdd>::GemmKernel;
constexpr int kTrailBM = 64, kTrailBN = 128;
constexpr int kTrailSmem = (int)sizeof(TrailGK::SharedStorage);

template <class Map>
__global__ void __launch_bounds__(TrailGK::kThreadCount, 2) trail_update_kernel(Map map, const int* __restrict__ info) {
  extern __shared__ __align__(16) uint8_t smem_t[];
  GemmTile t;
  if (!map.template operator()<kTrailBM, kTrailBN>((int64_t)blockIdx.x, t)) return;
  if (info != nullptr && *(volatile const int*)info != 0) return;  // a pivot failed upstream
  using Mma = TrailGK::Mma;
  using Epi = TrailGK::Epilogue;
  auto& ss = *reinterpret_cast<TrailGK::SharedStorage*>(smem_t);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  Mma::IteratorA itA(Mma::IteratorA::Params(cutlass::layout::ColumnMajor(t.ldb)), const_cast<double*>(t.B),
                     {kTrailBN, t.K}, tid, {0, 0});
  Mma::IteratorB itB(Mma::IteratorB::Params(cutlass::layout::RowMajor(t.lda)), const_cast<double*>(t.A),
                     {t.K, kTrailBM}, tid, {0, 0});
  Mma mma(ss.main_loop, tid, warp, lane);
  Mma::FragmentC acc;
  acc.clear();
  mma(t.K / 16, acc, itA, itB, acc);
  __syncthreads();  // the epilogue reuses the mainloop's shared memory
  Epi::OutputTileIterator::Params pC(cutlass::layout::RowMajor(t.ldc));
  Epi::OutputTileIterator itC(pC, t.C, {kTrailBN, kTrailBM}, tid, {0, 0});
  Epi::OutputTileIterator itD(pC, t.C, {kTrailBN, kTrailBM}, tid, {0, 0});
  Epi epi(ss.epilogue, tid, warp, lane);
  Epi::OutputOp op(Epi::OutputOp::Params(-1.0, 1.0));
  epi(op, itD, acc, itC);
}

template <class Map>
void launch_trail(const Map& map, const int* info, cudaStream_t s) {
  const int64_t nblk = map.blocks(kTrailBM, kTrailBN);
  if (nblk <= 0) return;
  trail_update_kernel<Map><<<(unsigned)nblk, TrailGK::kThreadCount, kTrailSmem, s>>>(map, info);
}

// ---- CUTLASS-mainloop panel kernels (N = 64: the left-looking panel update and the TRSM by
// the inverted diagonal block) -------------------------------------------------------------
// 64 x 64 CTA tiles (32 x 32 warps, 3 stages) over the rows of the panel, transposed as above;
// partial row tiles through the predicated iterators; accumulate: C <- C - A B^T, else
// C <- A B^T (C may alias A: the CTA owns all 64 columns of its rows and reads them first).
using PanelGK = cutlass::gemm::kernel::DefaultGemm<
    double, cutlass::layout::ColumnMajor, 1, double, cutlass::layout::RowMajor, 1, double, cutlass::layout::RowMajor,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 64, 16>,
    cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 3, false, cutlass::arch::OpMultiplyAdd>::GemmKernel;
constexpr int kPanelSmem = (int)sizeof(PanelGK::SharedStorage);

__global__ void __launch_bounds__(PanelGK::kThreadCount, 4) panel_gemm_kernel(DenseMap map, bool accumulate,
                                                                              const int* __restrict__ info) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // programmatic dependent launch (panel chain)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(16) uint8_t smem_p[];
  GemmTile t;
  map.operator()<64, 64>((int64_t)blockIdx.x, t);
  if (info != nullptr && *(volatile const int*)info != 0) return;
  using Mma = PanelGK::Mma;
  using Epi = PanelGK::Epilogue;
  auto& ss = *reinterpret_cast<PanelGK::SharedStorage*>(smem_p);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  Mma::IteratorA itA(Mma::IteratorA::Params(cutlass::layout::ColumnMajor(t.ldb)), const_cast<double*>(t.B),
                     {t.n_valid, t.K}, tid, {0, 0});
  Mma::IteratorB itB(Mma::IteratorB::Params(cutlass::layout::RowMajor(t.lda)), const_cast<double*>(t.A),
                     {t.K, t.m_valid}, tid, {0, 0});
  Mma mma(ss.main_loop, tid, warp, lane);
  Mma::FragmentC acc;
  acc.clear();
  mma((t.K + 15) / 16, acc, itA, itB, acc);
  __syncthreads();  // C may alias A: every warp has consumed its tiles of A before any store
  Epi::OutputTileIterator::Params pC(cutlass::layout::RowMajor(t.ldc));
  Epi::OutputTileIterator itC(pC, t.C, {t.n_valid, t.m_valid}, tid, {0, 0});
  Epi::OutputTileIterator itD(pC, t.C, {t.n_valid, t.m_valid}, tid, {0, 0});
  Epi epi(ss.epilogue, tid, warp, lane);
  Epi::OutputOp op(accumulate ? Epi::OutputOp::Params(-1.0, 1.0) : Epi::OutputOp::Params(1.0, 0.0));
  epi(op, itD, acc, itC);
}

cudaError_t gemm_init() {
  cudaError_t e;
  if ((e = set_smem<PanelCfg, true, DenseMap>()) != cudaSuccess) return e;
  if ((e = set_smem<PanelCfg, false, DenseMap>()) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(trail_update_kernel<SyrkMap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kTrailSmem)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(panel_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem)) !=
      cudaSuccess)
    return e;
  return cudaFuncSetAttribute(trail_update_kernel<Syrk2DMap>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrailSmem);
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
  static const int min_k = [] {  // tuning: EXAGEO_PANEL_CUTLASS_MINK
    const char* e = getenv("EXAGEO_PANEL_CUTLASS_MINK");
    return e ? atoi(e) : 512;
  }();
  if (N == 64 && K >= min_k) {  // long panel updates: CUTLASS mainloop (64 x 64 tiles)
    const unsigned nblk = (unsigned)map.blocks(64, 64);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(PanelGK::kThreadCount);
    cfg.dynamicSmemBytes = kPanelSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, panel_gemm_kernel, map, accumulate, info);
    return;
  }
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
  launch_trail(map, info, s);
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
  launch_trail(map, info, s);
}

}  // namespace exageo
