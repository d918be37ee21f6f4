// gemm_dmma.cu -- K3/K4: the dense contractions of the tiled Cholesky on the
// FP64 tensor cores (DMMA) of sm_100a.
//
// Every contraction of the factorization has the form
//     C (M x N) <- C - A (M x K) * B (N x K)^T      (SYRK / GEMM trailing update,
//                                                     left-looking panel update)
//     C (M x N) <-     A (M x K) * B (N x K)^T      (TRSM as multiplication by
//                                                     W = L_kk^{-1}: A L_kk^{-T} = A W^T)
// with A, B, C column-major. The paper's tile DAG (Fig. 2; trailing
// update is "compute-intensive Level-3 BLAS") is realised as
// stream-ordered launches of this one kernel family.
//
// FP64 on sm_100a: tcgen05.mma has no f64 kind; the FP64 tensor path is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, 256 FMA per instruction;
// measured 37.2 TFLOP/s chip-wide at 1965 MHz, tools/probes/fp64_peak.cu).
// Operands are staged global -> shared with a STAGES-deep cp.async ring
// (16-byte LDGSTS), fragments are read with conflict-free 64-bit LDS
// (shared leading dimension = 4 mod 16 doubles), accumulators stay in registers.
#include <cstdint>

#include "internal.h"

namespace exageo {

namespace {

struct GemmTile {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int K;
  int m_valid, n_valid;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Dense problem: CTA (bm, bn) of a ceil(M/BM) x ceil(N/BN) grid.
struct DenseMap {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int64_t M;
  int N, K;
  int mblocks;
  template <int BM, int BN>
  __device__ __forceinline__ bool operator()(int64_t bid, GemmTile& t) const {
    const int64_t bm = bid % mblocks, bn = bid / mblocks;
    t.A = A + bm * BM;
    t.B = B + bn * BN;
    t.C = C + bn * BN * ldc + bm * BM;
    t.lda = lda;
    t.ldb = ldb;
    t.ldc = ldc;
    t.K = K;
    const int64_t mv = M - bm * BM;
    t.m_valid = mv > BM ? BM : (int)mv;
    t.n_valid = (N - (int)bn * BN) > BN ? BN : (N - (int)bn * BN);
    return true;
  }
};

// Trailing update of step k over the lower block-column panels (internal.h).
// Blocks of 128 x 128: column block cb covers global columns c0 + 128 cb,
// row block rb >= cb covers global rows c0 + 128 rb (rb == Mb is the z row block),
// c0 = (k+1) nb. Enumerated column by column.
struct SyrkMap {
  Layout L;
  double* ws;
  int k;
  int Mb;  // number of square 128-blocks in the trailing matrix
  template <int BM, int BN>
  __device__ __forceinline__ bool operator()(int64_t bid, GemmTile& t) const {
    static_assert(BM == 128 && BN == 128, "SyrkMap assumes 128x128 blocks");
    // column cb holds (Mb + 1 - cb) blocks; S(cb) = cb (Mb + 1) - cb (cb - 1) / 2
    const double a = (double)Mb + 1.5;
    int64_t cb = (int64_t)(a - sqrt(a * a - 2.0 * (double)bid));
    auto S = [&](int64_t c) { return c * (Mb + 1) - c * (c - 1) / 2; };
    while (cb > 0 && S(cb) > bid) --cb;
    while (S(cb + 1) <= bid) ++cb;
    const int64_t rb = cb + (bid - S(cb));
    const int64_t c0 = (int64_t)(k + 1) * L.nb;
    const int64_t gc = c0 + cb * 128;  // global column of the block
    const int64_t gr = c0 + rb * 128;  // global row of the block (N.. = z block)
    const int64_t kb = (int64_t)k * L.nb;
    const double* Pk = ws + L.off(k);
    const int64_t ldk = L.ld(k);
    t.A = Pk + (gr - kb);
    t.B = Pk + (gc - kb);
    t.lda = ldk;
    t.ldb = ldk;
    const int J = (int)(gc / L.nb);
    const int64_t Jb = (int64_t)J * L.nb;
    t.ldc = L.ld(J);
    t.C = ws + L.off(J) + (gc - Jb) * t.ldc + (gr - Jb);
    t.K = L.nb;
    t.m_valid = 128;
    t.n_valid = 128;
    return true;
  }
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, class Map>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, 1)
    gemm_nt_dmma(Map map, const int* __restrict__ info, bool accumulate) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int LDA_S = BM + 4, LDB_S = BN + 4;  // = 4 (mod 16) doubles: conflict-free fragment loads
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int MI = WM / 8, NI = WN / 8;
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");

  if (info != nullptr && *(volatile const int*)info != 0) return;  // a previous pivot failed
  GemmTile t;
  if (!map.template operator()<BM, BN>((int64_t)blockIdx.x, t)) return;

  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDA_S;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = t.K / BK;

  auto load_stage = [&](int slot, int kt) {
    double* a_s = sA + slot * BK * LDA_S;
    double* b_s = sB + slot * BK * LDB_S;
    constexpr int CA = BK * BM / 2;  // 16-byte chunks
#pragma unroll
    for (int c = tid; c < CA; c += NT) {
      const int col = c / (BM / 2), row = (c % (BM / 2)) * 2;
      cp_async16(a_s + col * LDA_S + row, t.A + (int64_t)(kt * BK + col) * t.lda + row);
    }
    constexpr int CB = BK * BN / 2;
#pragma unroll
    for (int c = tid; c < CB; c += NT) {
      const int col = c / (BN / 2), row = (c % (BN / 2)) * 2;
      cp_async16(b_s + col * LDB_S + row, t.B + (int64_t)(kt * BK + col) * t.ldb + row);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* a_s = sA + (kt % STAGES) * BK * LDA_S + wm * WM + fr;
    const double* b_s = sB + (kt % STAGES) * BK * LDB_S + wn * WN + fr;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = a_s[(kk + fk) * LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = b_s[(kk + fk) * LDB_S + j * 8];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = C - acc  or  C = acc (rows < m_valid, cols < n_valid)
  __syncthreads();  // all warps done reading (A may alias C in the TRSM use)
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int r = wm * WM + i * 8 + fr;
    if (r >= t.m_valid) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wn * WN + j * 8 + fk * 2 + e;
        if (c >= t.n_valid) continue;
        double* p = t.C + (int64_t)c * t.ldc + r;
        *p = accumulate ? (*p - acc[i][j][e]) : acc[i][j][e];
      }
    }
  }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
constexpr int smem_bytes() {
  return STAGES * BK * ((BM + 4) + (BN + 4)) * (int)sizeof(double);
}

// Panel configuration: 128 x 64 tile, 8 warps (4 x 2, warp tile 32 x 32).
constexpr int P_BM = 128, P_BN = 64, P_BK = 16, P_WM = 4, P_WN = 2, P_ST = 4;
// Trailing configuration: 128 x 128 tile, 8 warps (2 x 4, warp tile 64 x 32).
constexpr int S_BM = 128, S_BN = 128, S_BK = 16, S_WM = 2, S_WN = 4, S_ST = 4;

}  // namespace

cudaError_t gemm_init() {
  cudaError_t e = cudaFuncSetAttribute(gemm_nt_dmma<P_BM, P_BN, P_BK, P_WM, P_WN, P_ST, DenseMap>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes<P_BM, P_BN, P_BK, P_WM, P_WN, P_ST>());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(gemm_nt_dmma<S_BM, S_BN, S_BK, S_WM, S_WN, S_ST, SyrkMap>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes<S_BM, S_BN, S_BK, S_WM, S_WN, S_ST>());
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
  map.mblocks = (int)((M + P_BM - 1) / P_BM);
  const int64_t nblk = (int64_t)map.mblocks * ((N + P_BN - 1) / P_BN);
  constexpr int smem = smem_bytes<P_BM, P_BN, P_BK, P_WM, P_WN, P_ST>();
  auto kern = gemm_nt_dmma<P_BM, P_BN, P_BK, P_WM, P_WN, P_ST, DenseMap>;
  kern<<<(unsigned)nblk, P_WM * P_WN * 32, smem, s>>>(map, info, accumulate);
}

void launch_syrk_trailing(const Layout& L, double* ws, int k, const int* info, cudaStream_t s) {
  const int64_t c0 = (int64_t)(k + 1) * L.nb;
  if (c0 >= L.N) return;
  SyrkMap map;
  map.L = L;
  map.ws = ws;
  map.k = k;
  map.Mb = (int)((L.N - c0) / 128);
  const int64_t nblk = (int64_t)map.Mb * (map.Mb + 1) / 2 + map.Mb;
  constexpr int smem = smem_bytes<S_BM, S_BN, S_BK, S_WM, S_WN, S_ST>();
  auto kern = gemm_nt_dmma<S_BM, S_BN, S_BK, S_WM, S_WN, S_ST, SyrkMap>;
  kern<<<(unsigned)nblk, S_WM * S_WN * 32, smem, s>>>(map, info, true);
}

}  // namespace exageo
