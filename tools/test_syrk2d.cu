// test_syrk2d.cu -- host-side check of the 2-D block-cyclic layout (internal.h Layout with
// P > 1) and of the trailing-update tile enumeration on a process grid (Syrk2DMap): for
// every grid P x Q, rank, step k and the panel selection do_factor makes (U1: panel k+1 on
// its process column; U2: the other local panels > k, up to the IND super tile), every
// 64 x 64 sub-tile of the lower triangle stored on the rank (its tile rows I = p mod P,
// I >= J, and the z row block on the process row that holds it) is produced exactly once,
// with C, A and B pointers that agree with the layout's local-row formula; local panel
// offsets tile the rank's storage, and all ranks together store every lower tile once.
#include <cstdio>
#include <set>
#include <tuple>
#include <vector>

#include "gemm_dmma.cuh"

using namespace exageo;
using namespace exageo::gemm;

Layout grid_layout(int T, int nb, int P, int Q, int rank, int ind, std::vector<int64_t>& offs) {
  Layout L;
  L.nb = nb;
  L.T = T;
  L.N = (int64_t)T * nb;
  L.n = L.N - 3;
  L.world = P * Q;
  L.rank = rank;
  L.P = P;
  L.Q = Q;
  L.p = rank / Q;
  L.q = rank % Q;
  L.ind = ind;
  offs.assign(L.owned() + 1, 0);
  for (int m = 0; m < L.owned(); ++m) offs[m + 1] = offs[m] + (int64_t)nb * L.ld(L.owned_panel(m));
  L.offs_h = offs.data();
  return L;
}

static double ws_dummy[1];
static double slice_dummy[kMaxP][1];

template <int BM, int BN>
int check(int T, int nb, int P, int Q, int rank, int k, int J0, int npan, int ind) {
  std::vector<int64_t> offs;
  Layout L = grid_layout(T, nb, P, Q, rank, ind, offs);
  Syrk2DMap m;
  m.L = L;
  m.ws = ws_dummy;
  for (int pp = 0; pp < kMaxP; ++pp) {
    m.slice[pp] = slice_dummy[pp];
    m.sld[pp] = pp < P ? L.ld_of(pp, k) : 0;
  }
  m.k = k;
  m.J0 = J0;
  m.npan = npan;
  m.Eb = L.sb_end(k);
  // the layout of the rank that stores slice pp: local rows of panel k on process row pp
  std::vector<std::vector<int64_t>> so(P);
  std::vector<Layout> SL;
  for (int pp = 0; pp < P; ++pp) SL.push_back(grid_layout(T, nb, P, Q, pp * Q + k % Q, ind, so[pp]));
  const int64_t nblk = m.blocks(BM, BN);
  std::set<std::tuple<int, int64_t, int64_t>> seen;  // (J, global row, global col)
  for (int64_t b = 0; b < nblk; ++b) {
    GemmTile t;
    if (!m.operator()<BM, BN>(b, t)) continue;
    // locate the C tile: which local panel, which local row / column
    int J = -1;
    int64_t lr = -1, cc = -1;
    for (int mm = 0; mm < L.owned(); ++mm) {
      const int j = L.owned_panel(mm);
      const int64_t o = t.C - ws_dummy - L.off(j);
      if (o >= 0 && o < (int64_t)nb * L.ld(j)) {
        J = j;
        cc = o / L.ld(j);
        lr = o % L.ld(j);
      }
    }
    if (J < 0 || t.ldc != L.ld(J)) {
      printf("C outside the local panels\n");
      return 1;
    }
    if (J < J0 || (J - J0) % Q != 0 || (J - J0) / Q >= npan) {
      printf("panel %d not selected\n", J);
      return 1;
    }
    const int64_t gr = lr < L.lrows(J) ? L.grow(J, lr) : L.N + (lr - L.lrows(J));
    const int64_t gc = (int64_t)J * nb + cc;
    if (L.lrow(J, gr) != lr) {
      printf("lrow(grow) mismatch\n");
      return 1;
    }
    // A: slice p at the local row of gr in panel k; B: slice J mod P at the local row of gc
    const int pJ = J % P;
    if (t.A != slice_dummy[L.p] + SL[L.p].lrow(k, gr) || t.lda != SL[L.p].ld(k) ||
        t.B != slice_dummy[pJ] + SL[pJ].lrow(k, gc) || t.ldb != SL[pJ].ld(k) || t.K != nb) {
      printf("bad A/B (T=%d nb=%d P=%d Q=%d rank=%d k=%d J=%d gr=%lld gc=%lld)\n", T, nb, P, Q, rank, k, J,
             (long long)gr, (long long)gc);
      return 1;
    }
    if (gr < L.N && (gr / nb >= L.sb_end(k) || gr + BM <= gc)) {
      printf("tile outside the updated lower triangle\n");
      return 1;
    }
    if (!seen.insert({J, gr, gc}).second) {
      printf("duplicate\n");
      return 1;
    }
  }
  int64_t expect = 0;
  for (int i = 0; i < npan; ++i) {
    const int J = J0 + i * Q;
    for (int I = J; I < L.sb_end(k); ++I)
      if (I % P == L.p)
        for (int rt = 0; rt < nb / BM; ++rt)
          for (int ct = 0; ct < nb / BN; ++ct)
            if (I > J || rt * BM + BM > ct * BN) ++expect;  // not strictly above the diagonal
    if (L.has_z()) expect += (int64_t)(ZR / BM) * (nb / BN);
  }
  if ((int64_t)seen.size() != expect) {
    printf("count %lld != %lld (T=%d nb=%d P=%d Q=%d rank=%d k=%d J0=%d npan=%d)\n", (long long)seen.size(),
           (long long)expect, T, nb, P, Q, rank, k, J0, npan);
    return 1;
  }
  return 0;
}

int check_storage(int T, int nb, int P, int Q) {
  // every rank's local panels are contiguous (off(j) increasing by nb ld(j)); together the
  // ranks store each lower tile once and each column's z row block once
  int64_t sum = 0;
  std::set<std::tuple<int, int>> tiles;
  for (int r = 0; r < P * Q; ++r) {
    std::vector<int64_t> offs;
    Layout L = grid_layout(T, nb, P, Q, r, 0, offs);
    int64_t expect_off = 0;
    for (int mm = 0; mm < L.owned(); ++mm) {
      const int j = L.owned_panel(mm);
      if (L.off(j) != expect_off) {
        printf("offset mismatch\n");
        return 1;
      }
      expect_off += (int64_t)nb * L.ld(j);
      for (int64_t lr = 0; lr < L.lrows(j); lr += nb) {
        const int I = (int)(L.grow(j, lr) / nb);
        if (I < j || I % P != L.p || !tiles.insert({I, j}).second) {
          printf("tile (%d, %d) misplaced or stored twice\n", I, j);
          return 1;
        }
      }
    }
    sum += L.total();
  }
  if ((int64_t)tiles.size() != (int64_t)T * (T + 1) / 2) {
    printf("lower tiles missing\n");
    return 1;
  }
  std::vector<int64_t> o1;
  Layout G = grid_layout(T, nb, 1, 1, 0, 0, o1);
  if (sum != G.total()) {
    printf("storage %lld != %lld\n", (long long)sum, (long long)G.total());
    return 1;
  }
  return 0;
}

int main() {
  int bad = 0, n = 0;
  const int grids[][2] = {{2, 1}, {2, 2}, {2, 4}, {4, 2}, {3, 2}, {4, 1}, {8, 1}, {2, 3}};
  for (const auto& g : grids) {
    const int P = g[0], Q = g[1];
    for (int nb : {128, 256, 512})
      for (int T : {1, 2, 3, 5, 8, 13})
        for (int ind : {0, 3}) {
          bad += check_storage(T, nb, P, Q);
          ++n;
          for (int rank = 0; rank < P * Q; ++rank)
            for (int k = 0; k + 1 < T; ++k) {
              std::vector<int64_t> offs;
              Layout L = grid_layout(T, nb, P, Q, rank, ind, offs);
              const int e = L.sb_end(k);
              if (L.owns(k + 1) && k + 1 < e)
                bad += check<64, 64>(T, nb, P, Q, rank, k, k + 1, 1, ind) +
                       check<64, 128>(T, nb, P, Q, rank, k, k + 1, 1, ind);
              const int J0 = L.first_owned_from(L.owns(k + 1) ? k + 2 : k + 1);
              const int npan = J0 < e ? (e - 1 - J0) / Q + 1 : 0;
              if (npan > 0)
                bad += check<64, 64>(T, nb, P, Q, rank, k, J0, npan, ind) +
                       check<64, 128>(T, nb, P, Q, rank, k, J0, npan, ind);  // the trailing-update tile
              n += 2;
            }
        }
  }
  printf("%s: %d failures in %d enumerations\n", bad ? "FAIL" : "OK", bad, n);
  return bad ? 1 : 0;
}
