// gemm_cutlass_tune.cu -- the trailing update U2(k) (SyrkMap tiles) with a CUTLASS SM80 DMMA
// mainloop + epilogue (the tiling of cuBLAS's DGEMM kernel on this B200: 64x128x16, warps
// 32x64, 3 stages, 2 CTAs/SM) inside our own kernel, against the product kernel: timing at
// the first steps and an element-by-element comparison of the updated workspace.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I <cutlass>/include \
//        -I paper_1708_02835_b200/csrc -o tools/gemm_cutlass_tune tools/gemm_cutlass_tune.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cutlass/cutlass.h"
#include "cutlass/epilogue/thread/linear_combination.h"
#include "cutlass/gemm/kernel/default_gemm.h"
#include "gemm_dmma.cuh"

using namespace exageo;
using namespace exageo::gemm;

// transposed problem per tile: C^T (BN x BM, row-major view of our column-major C) -=
// B (BN x K, column-major) . A^T (K x BM, row-major view of our column-major A)
template <int TM, int TN, int WM, int WN, int STAGES>
using GKt = typename cutlass::gemm::kernel::DefaultGemm<
    double, cutlass::layout::ColumnMajor, 1, double, cutlass::layout::RowMajor, 1, double, cutlass::layout::RowMajor,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<TM, TN, 16>,
    cutlass::gemm::GemmShape<WM, WN, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, STAGES, false,
    cutlass::arch::OpMultiplyAdd>::GemmKernel;

template <class GK, int BM, int BN, int MINB, class Map>
__global__ void __launch_bounds__(GK::kThreadCount, MINB) trail_cutlass(Map map) {
  extern __shared__ __align__(16) uint8_t smem[];
  GemmTile t;
  if (!map.template operator()<BM, BN>((int64_t)blockIdx.x, t)) return;
  using Mma = typename GK::Mma;
  using Epi = typename GK::Epilogue;
  auto& ss = *reinterpret_cast<typename GK::SharedStorage*>(smem);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  typename Mma::IteratorA itA(typename Mma::IteratorA::Params(cutlass::layout::ColumnMajor(t.ldb)),
                              const_cast<double*>(t.B), {BN, t.K}, tid, {0, 0});
  typename Mma::IteratorB itB(typename Mma::IteratorB::Params(cutlass::layout::RowMajor(t.lda)),
                              const_cast<double*>(t.A), {t.K, BM}, tid, {0, 0});
  Mma mma(ss.main_loop, tid, warp, lane);
  typename Mma::FragmentC acc;
  acc.clear();
  mma(t.K / 16, acc, itA, itB, acc);
  typename Epi::OutputTileIterator::Params pC(cutlass::layout::RowMajor(t.ldc));
  typename Epi::OutputTileIterator itC(pC, t.C, {BN, BM}, tid, {0, 0});
  typename Epi::OutputTileIterator itD(pC, t.C, {BN, BM}, tid, {0, 0});
  Epi epi(ss.epilogue, tid, warp, lane);
  typename Epi::OutputOp op(typename Epi::OutputOp::Params(-1.0, 1.0));
  epi(op, itD, acc, itC);
}

__global__ void fill(double* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 1e-3 * (double)((i * 2654435761ull) % 1000) / 1000.0;
}

SyrkMap make_map(const Layout& L, double* ws, int k, int group) {
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.Pk = ws + L.off(k);
  map.k = k;
  map.J0 = k + 2;
  map.npan = L.T - k - 2;
  map.row_end = L.N;
  map.group = group;
  return map;
}

template <class GK, int BM, int BN, int MINB>
float time_cutlass(const char* name, const SyrkMap& map, double flops, int reps) {
  auto kern = trail_cutlass<GK, BM, BN, MINB, SyrkMap>;
  const int smem = (int)sizeof(typename GK::SharedStorage);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t nblk = map.blocks(BM, BN);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<(unsigned)nblk, GK::kThreadCount, smem>>>(map);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<(unsigned)nblk, GK::kThreadCount, smem>>>(map);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("%-48s k=%3d blocks=%8lld smem %6d best %9.3f ms %6.2f TF %s\n", name, map.k, (long long)nblk, smem, best,
         flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
  return best;
}

float time_product(const SyrkMap& map, double flops, int reps) {
  using C = Cfg<64, 64, 16, 2, 2, 2, 4>;
  set_smem<C, true, SyrkMap>();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch<C, true, SyrkMap, true>(map, nullptr, 0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch<C, true, SyrkMap, true>(map, nullptr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("%-48s k=%3d best %9.3f ms %6.2f TF\n", "product 64x64x16 st2 preC 4 CTA", map.k, best, flops / best / 1e9);
  return best;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 20000;
  const int nb = argc > 2 ? atoi(argv[2]) : 512;
  const int check = argc > 3 ? atoi(argv[3]) : 1;
  Layout L;
  L.n = n;
  L.nb = nb;
  L.T = (int)((n + nb - 1) / nb);
  L.N = (int64_t)L.T * nb;
  const int64_t g = ((int64_t)2 << 20) / ((int64_t)nb * nb);
  const int group = (int)(g < 1 ? 1 : (g > 8 ? 8 : g));
  const size_t cnt = (size_t)L.total() + 512;
  double *ws, *ws2;
  if (cudaMalloc(&ws, cnt * 8) != cudaSuccess || (check && cudaMalloc(&ws2, cnt * 8) != cudaSuccess)) {
    printf("alloc failed\n");
    return 1;
  }
  fill<<<1024, 256>>>(ws, (int64_t)cnt);
  cudaDeviceSynchronize();
  printf("n=%lld nb=%d T=%d group=%d\n", (long long)n, nb, L.T, group);
  if (check) {  // one U2(0) by each kernel on identical copies, compared element by element
    cudaMemcpy(ws2, ws, cnt * 8, cudaMemcpyDeviceToDevice);
    SyrkMap m1 = make_map(L, ws, 0, group), m2 = make_map(L, ws2, 0, group);
    launch<Cfg<64, 64, 16, 2, 2, 2, 4>, true, SyrkMap, true>(m1, nullptr, 0);
    using GK = GKt<128, 64, 64, 32, 3>;
    auto kern = trail_cutlass<GK, 64, 128, 2, SyrkMap>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GK::SharedStorage));
    kern<<<(unsigned)m2.blocks(64, 128), GK::kThreadCount, sizeof(GK::SharedStorage)>>>(m2);
    cudaDeviceSynchronize();
    std::vector<double> h1(cnt), h2(cnt);
    cudaMemcpy(h1.data(), ws, cnt * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), ws2, cnt * 8, cudaMemcpyDeviceToHost);
    // the lower triangle (and the z block) of every panel; the strict upper half of a diagonal
    // tile is never read (K2 reads the lower triangle) and the 64 x 128 tiles update it too
    double md = 0.0, mx = 0.0, mdu = 0.0;
    size_t ndiff = 0, nlow = 0;
    for (int J = 0; J < L.T; ++J)
      for (int cc = 0; cc < nb; ++cc)
        for (int64_t lr = 0; lr < L.ld(J); ++lr) {
          const size_t i = (size_t)(L.off(J) + (int64_t)cc * L.ld(J) + lr);
          const double d = fabs(h1[i] - h2[i]);
          if (lr < cc) {  // strict upper half of the diagonal tile
            if (d > mdu) mdu = d;
            continue;
          }
          // identity padding (rows / columns >= n): never touched in a real layout (their panel
          // rows are zero); the synthetic fill here is not zero there, so the 64- and 128-wide
          // tiles' different skip boundaries show
          if ((int64_t)J * nb + cc >= L.n || (lr < L.lrows(J) && (int64_t)J * nb + lr >= L.n)) continue;
          ++nlow;
          if (d > md) md = d;
          if (fabs(h1[i]) > mx) mx = fabs(h1[i]);
          if (d > 1e-12 * (1.0 + fabs(h1[i]))) ++ndiff;
        }
    printf("check U2(0) on %zu lower-triangle entries: max |diff| %.3e (max |value| %.3e), %zu beyond 1e-12 "
           "relative; strict upper half of diagonal tiles (never read) max |diff| %.3e  %s\n",
           nlow, md, mx, ndiff, mdu, cudaGetErrorString(cudaGetLastError()));
    fill<<<1024, 256>>>(ws, (int64_t)cnt);
    cudaDeviceSynchronize();
  }
  for (int k : {0, L.T / 3, (2 * L.T) / 3}) {
    const SyrkMap map = make_map(L, ws, k, group);
    const double m = (double)(L.n - (int64_t)(k + 2) * L.nb);
    const double flops = 2.0 * L.nb * (m * (m + 1) / 2 + m);
    const int reps = n > 60000 ? 2 : 3;
    time_product(map, flops, reps);
    time_cutlass<GKt<128, 64, 64, 32, 3>, 64, 128, 2>("cutlass 64x128x16 (warp 32x64) st3 2 CTA", map, flops, reps);
    time_cutlass<GKt<128, 64, 64, 32, 4>, 64, 128, 2>("cutlass 64x128x16 (warp 32x64) st4 2 CTA", map, flops, reps);
    time_cutlass<GKt<64, 64, 32, 32, 3>, 64, 64, 4>("cutlass 64x64x16 (warp 32x32) st3 4 CTA", map, flops, reps);
    time_cutlass<GKt<128, 128, 64, 64, 3>, 128, 128, 1>("cutlass 128x128x16 (warp 64x64) st3 1 CTA", map, flops, reps);
    time_cutlass<GKt<64, 128, 32, 64, 3>, 128, 64, 2>("cutlass 128x64x16 (warp 64x32) st3 2 CTA", map, flops, reps);
  }
  return 0;
}
