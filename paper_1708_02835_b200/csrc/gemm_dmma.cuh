// gemm_dmma.cuh -- the FP64 tensor-core (DMMA) contraction kernel family of the
// tiled Cholesky (K3 TRSM-by-inverse, K4 SYRK/GEMM trailing update, and the
// left-looking panel update). Included by gemm_dmma.cu (the product) and by
// tools/gemm_tune.cu (the tuning harness).
//
//     C (M x N) <- C - A (M x K) * B (N x K)^T      (ACC = true)
//     C (M x N) <-     A (M x K) * B (N x K)^T      (ACC = false; C may alias A when
//                                                    one CTA owns all N columns)
// A, B, C column-major. Paper: tile DAG of Fig. 2; the trailing
// update is the compute-intensive Level-3 BLAS phase.
//
// sm_100a FP64: tcgen05.mma has no f64 kind; the FP64 tensor path is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4 = 256 FMA; chip peak measured
// 37.2 TFLOP/s at 1965 MHz, tools/probes/fp64_peak.cu). Operands are staged
// global -> shared by a STAGES-deep cp.async (LDGSTS.128, L2-only) ring;
// fragments are read with conflict-free LDS.64 (shared leading dimension
// = 4 mod 16 doubles); accumulators live in registers.
#pragma once
#include <cstdint>

#include "internal.h"

namespace exageo {
namespace gemm {

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

// D = A(8x4) B(4x8) + C(8x8); lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4)+{0,1}].
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
  __host__ __device__ __forceinline__ bool operator()(int64_t bid, GemmTile& t) const {
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
  __host__ int64_t blocks(int BM, int BN) const { return (int64_t)((M + BM - 1) / BM) * ((N + BN - 1) / BN); }
};

// Trailing update by panel k of a set of panels owned by this rank (internal.h):
// panels J_i = J0 + i * world, i < npan. Panel J's part of the trailing matrix is
// its columns J nb .. J nb + nb - 1 and rows from its diagonal down to the z row
// block, cut into 128 x 128 blocks: column block cb in [0, cpt), cpt = nb / 128,
// row block rb in [cb, Mr] (rb = Mr = (N - J nb) / 128 is the z row block).
// A 128-block is split into (128/BM) x (128/BN) CTA tiles; consecutive bids share
// a 128-block. Order: super panel by super panel -- `group` consecutive panels taken as one
// panel of width group * nb (single-rank layouts; group = 1 otherwise) -- and inside a
// super panel row block by row block: the row's A operand (rows of panel k) is reused
// group * cpt times back to back, and the super panel's B operand (group * nb rows of
// panel k, 16 MB for 8 x 512) stays L2-resident for its sweep. With group = 1 panel k's
// rows are re-streamed from HBM once per trailing panel (ncu: 40 GB of the 119 GB of
// U2(0) at n = 100k); grouping divides that by the group size.
// Operand: Pk = panel k (this rank's own storage or the received copy), ld(k).
struct SyrkMap {
  Layout L;
  double* ws;        // this rank's panel storage
  const double* Pk;  // panel k operand
  int k;
  int J0;            // first panel of this launch (owned)
  int npan;          // number of panels (J0, J0 + world, ...)
  int64_t row_end;   // rows updated: [J nb, row_end) and the z block (N for the exact problem;
                     // the end of the diagonal super tile for IND: zero tiles are skipped)
  int group = 1;     // panels per super panel (1 unless world == 1)

  __host__ __device__ int cpt() const { return L.nb / 128; }
  __host__ __device__ int64_t Mr0() const { return (row_end - (int64_t)J0 * L.nb) / 128; }
  // 128-blocks of panel i: cpt (Mr_i + 1) - cpt (cpt - 1) / 2, Mr_i = Mr0 - i world cpt
  __host__ __device__ int64_t panel_blocks(int64_t i) const {
    const int64_t c = cpt(), Mr = Mr0() - i * L.world * c;
    return c * (Mr + 1) - c * (c - 1) / 2;
  }
  // 128-blocks of panels before panel i: i a - D i (i - 1) / 2, a = panel_blocks(0), D = world cpt^2
  __host__ __device__ int64_t Sp(int64_t i) const {
    const int64_t c = cpt(), D = (int64_t)L.world * c * c;
    return i * panel_blocks(0) - D * (i * (i - 1) / 2);
  }
  // the same for full super panels (world == 1) of width W = group cpt blocks: a super panel
  // is a panel of width W, so Sg(s) = s a_g - W^2 s (s - 1) / 2, a_g = W (Mr0 + 1) - W (W - 1) / 2
  __host__ __device__ int64_t Sg(int64_t sp) const {
    const int64_t W = (int64_t)group * cpt();
    const int64_t ag = W * (Mr0() + 1) - W * (W - 1) / 2;
    return sp * ag - W * W * (sp * (sp - 1) / 2);
  }

  template <int BM, int BN>
  __host__ __device__ __forceinline__ bool operator()(int64_t bid, GemmTile& t) const {
    static_assert((BM == 128 || BM == 64) && (BN == 128 || BN == 64), "SyrkMap: {64,128} x {64,128} tiles");
    constexpr int SPLIT_C = 128 / BN, SPLIT = (128 / BM) * SPLIT_C;
    const int sub = (int)(bid % SPLIT);
    const int half = sub % SPLIT_C, rhalf = sub / SPLIT_C;
    const int64_t q = bid / SPLIT;
    const int64_t nsup = (npan + group - 1) / group;  // super panels (group = 1: panels)
    // super panel: largest i with Sg(i) <= q  (quadratic guess, exact integer fix-up)
    const int64_t Wf = (int64_t)group * cpt();
    const double Dg = (double)(group == 1 ? L.world * cpt() * cpt() : Wf * Wf);
    const double a = (double)(group == 1 ? panel_blocks(0) : Sg(1));
    const double beta = a + 0.5 * Dg;
    const double disc = beta * beta - 2.0 * Dg * (double)q;
    int64_t i = (int64_t)((beta - sqrt(disc > 0.0 ? disc : 0.0)) / Dg);
    if (i >= nsup) i = nsup - 1;
    if (i < 0) i = 0;
    auto S = [&](int64_t v) { return group == 1 ? Sp(v) : Sg(v); };
    while (i > 0 && S(i) > q) --i;
    while (i + 1 < nsup && S(i + 1) <= q) ++i;
    int64_t qq = q - S(i);
    const int gn = (int)((npan - i * group) < group ? (npan - i * group) : group);  // panels in it
    const int Jfirst = J0 + (int)(i * group) * L.world;
    const int64_t w = (int64_t)gn * cpt();  // width in 128-blocks
    const int64_t head = w * (w + 1) / 2;
    int64_t rb, cb;
    if (qq < head) {  // diagonal 128-blocks of the panel: row rb holds columns 0..rb
      int64_t r = 0;
      while ((r + 1) * (r + 2) / 2 <= qq) ++r;
      rb = r;
      cb = qq - r * (r + 1) / 2;
    } else {
      qq -= head;
      rb = w + qq / w;
      cb = qq % w;
    }
    const int64_t Sb = (int64_t)Jfirst * L.nb;       // first row / column of the super panel
    const int64_t Mri = Mr0() - i * group * L.world * cpt();  // row block index of the z block
    const int64_t gc = Sb + cb * 128 + half * BN;    // global column of the tile
    const int J = (int)(gc / L.nb);                  // its panel (group > 1: world == 1)
    const int64_t Jb = (int64_t)J * L.nb;
    const int64_t gr = (rb == Mri ? L.N : Sb + rb * 128) + rhalf * BM;  // global row (N.. = z block)
    const int64_t kb = (int64_t)k * L.nb;
    const int64_t ldk = L.ld(k);
    t.A = Pk + (gr - kb);
    t.B = Pk + (gc - kb);
    t.lda = ldk;
    t.ldb = ldk;
    t.ldc = L.ld(J);
    t.C = ws + L.off(J) + (gc - Jb) * t.ldc + (gr - Jb);
    t.K = L.nb;
    t.m_valid = BM;
    t.n_valid = BN;
    // skipped (false): tiles strictly above the diagonal; tiles of the identity padding (all
    // rows or all columns >= n: their rows of panel k are zero, so the update is a no-op, R12);
    // z-block tiles below its first BM rows (zero rows: only row N, the z row, is live)
    if (gr + BM <= gc) return false;
    if (gc >= L.n || (gr < L.N && gr >= L.n)) return false;
    return gr < L.N + BM;
  }
  __host__ int64_t blocks(int BM, int BN) const {
    if (npan <= 0) return 0;
    return Sp(npan) * (128 / BN) * (128 / BM);
  }
};

// Trailing update on a 2-D process grid (P > 1, internal.h): this rank's local panels
// J = J0, J0 + Q, ... (npan of them) by panel k, whose rows arrive as P slices -- slice pp
// is the local panel k of rank (pp, k mod Q): the tile rows I = pp (mod P), I >= k, plus the
// z row block on the process row that holds it. The A operand of local panel J is this
// rank's own slice p at the same local row shifted by (i0(J) - i0(k)) tiles (the z block
// follows the square rows in both, so the shift is uniform); the B operand is tile J of
// slice J mod P. Rows: the square rows of the tiles < Eb (T, or the end of the diagonal
// super tile for IND) and the z block. CTA tiles BM x BN run panel by panel, row block by
// row block (A rows reused across the nb / BN column tiles, tile J of B L2-resident for the
// panel); sub-tiles strictly above the diagonal (only in the diagonal tile, on the rank of
// process row J mod P) are skipped.
struct Syrk2DMap {
  Layout L;
  double* ws;
  const double* slice[kMaxP];
  int64_t sld[kMaxP];
  int k, J0, npan, Eb;

  __host__ __device__ int64_t rows_sq(int J) const {
    const int t = L.i0_of(L.p, Eb) - L.i0(J);
    return t > 0 ? (int64_t)t * L.nb : 0;
  }
  __host__ __device__ int64_t mrows(int J) const { return rows_sq(J) + (L.has_z() ? ZR : 0); }

  template <int BM, int BN>
  __host__ __device__ __forceinline__ bool operator()(int64_t bid, GemmTile& t) const {
    const int ct = L.nb / BN;
    int64_t rem = bid;
    int J = J0;
    for (int m = 0; m < npan; ++m) {
      J = J0 + m * L.Q;
      const int64_t cnt = mrows(J) / BM * ct;
      if (rem < cnt) break;
      rem -= cnt;
    }
    const int64_t mt = rem / ct;
    const int nt = (int)(rem % ct);
    const int64_t rsq = rows_sq(J);
    const int64_t lr = mt * BM < rsq ? mt * BM : L.lrows(J) + (mt * BM - rsq);
    const int64_t shift = (int64_t)(L.i0(J) - L.i0(k)) * L.nb;
    const int pJ = J % L.P;
    const int64_t tB = (int64_t)((J - pJ) / L.P - L.i0_of(pJ, k)) * L.nb;
    t.A = slice[L.p] + shift + lr;
    t.lda = sld[L.p];
    t.B = slice[pJ] + tB + (int64_t)nt * BN;
    t.ldb = sld[pJ];
    t.ldc = L.ld(J);
    t.C = ws + L.off(J) + (int64_t)nt * BN * t.ldc + lr;
    t.K = L.nb;
    t.m_valid = BM;
    t.n_valid = BN;
    // strictly above the diagonal: only inside the diagonal tile (local rows [0, nb) of a
    // panel whose diagonal tile is on this process row)
    return !(pJ == L.p && lr < L.nb && lr + BM <= (int64_t)nt * BN);
  }
  __host__ int64_t blocks(int BM, int BN) const {
    int64_t b = 0;
    for (int m = 0; m < npan; ++m) b += mrows(J0 + m * L.Q) / BM * (L.nb / BN);
    return b;
  }
};

template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_,
                       MINB = MINB_;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int LDA_S = BM + 4, LDB_S = BN + 4;  // = 4 (mod 16) doubles
  static constexpr int SMEM = STAGES * BK * (LDA_S + LDB_S) * (int)sizeof(double);
};

// PRE (ACC only): the accumulators start from C (loads issued with the prologue, their
// latency hidden behind it) and the A fragments are negated, so the epilogue only
// stores -- no read-modify-write stall at the end of the tile.
template <class C, bool ACC, class Map, bool PRE = false>
__global__ void __launch_bounds__(C::NT, C::MINB) gemm_nt_dmma(Map map, const int* __restrict__ info) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, STAGES = C::STAGES, NT = C::NT;
  constexpr bool LOADC = ACC && PRE;
  constexpr int LDA_S = C::LDA_S, LDB_S = C::LDB_S;
  constexpr int WM = BM / C::WARPS_M, WN = BN / C::WARPS_N;
  constexpr int MI = WM / 8, NI = WN / 8;
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
  static_assert((LDA_S % 16) == 4 && (LDB_S % 16) == 4, "conflict-free fragment loads");

  // programmatic dependent launch (panel kernels at small n): wait for the preceding kernel
  // of the stream before touching memory, then let the next one launch and wait in turn
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  GemmTile t;
  if (!map.template operator()<BM, BN>((int64_t)blockIdx.x, t)) return;

  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDA_S;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
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
  // A failed pivot upstream makes the rest of the factorization meaningless: exit
  // (checked after the prologue loads are in flight, to hide the load latency).
  if (info != nullptr && *(volatile const int*)info != 0) {
    cp_async_wait<0>();
    return;
  }

  const int fr = lane >> 2, fk = lane & 3;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (LOADC) {
          const int r = wm * WM + i * 8 + fr, c = wn * WN + j * 8 + fk * 2 + e;
          acc[i][j][e] = (r < t.m_valid && c < t.n_valid) ? t.C[(int64_t)c * t.ldc + r] : 0.0;
        } else {
          acc[i][j][e] = 0.0;
        }
      }

  for (int kt = 0; kt < KT; ++kt) {
    if (ACC && !LOADC && kt == KT / 2) {
      // pull this tile's C into L2 ahead of the read-modify-write epilogue (128-byte lines)
      constexpr int LPC = BM / 16;  // lines per column
      for (int l = tid; l < BN * LPC; l += NT) {
        const double* p = t.C + (int64_t)(l / LPC) * t.ldc + (l % LPC) * 16;
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
      }
    }
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
      for (int i = 0; i < MI; ++i) af[i] = LOADC ? -a_s[(kk + fk) * LDA_S + i * 8] : a_s[(kk + fk) * LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = b_s[(kk + fk) * LDB_S + j * 8];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (!ACC) __syncthreads();  // C may alias A: every warp must be done reading

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
        if (ACC && !LOADC) *p = *p - acc[i][j][e];
        else *p = acc[i][j][e];
      }
    }
  }
}

template <class C, bool ACC, class Map>
cudaError_t set_smem() {
  cudaError_t e =
      cudaFuncSetAttribute(gemm_nt_dmma<C, ACC, Map>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(gemm_nt_dmma<C, ACC, Map, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              C::SMEM);
}

template <class C, bool ACC, class Map, bool PRE = false>
void launch(const Map& map, const int* info, cudaStream_t s, bool pdl = false) {
  const int64_t nblk = map.blocks(C::BM, C::BN);
  if (nblk <= 0) return;
  if (!pdl) {
    gemm_nt_dmma<C, ACC, Map, PRE><<<(unsigned)nblk, C::NT, C::SMEM, s>>>(map, info);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nblk);
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemm_nt_dmma<C, ACC, Map, PRE>, map, info);
}

}  // namespace gemm
}  // namespace exageo
