// test_syrkmap.cu -- host-side check of the trailing-update tile enumeration (SyrkMap)
// and of the distributed layout: for every (world, rank, k, J0, npan) every lower
// 128-block of the selected owned panels (incl. the z row block) is produced exactly
// once (as BM x BN sub-tiles) except the tiles skipped by design (identity padding rows or
// columns >= n, the z block's zero rows below its first BM rows), and A/B/C pointers agree
// with the panel layout formula;
// owned-panel offsets tile the rank's storage without overlap.
#include <cstdio>
#include <set>
#include <tuple>

#include "gemm_dmma.cuh"

using namespace exageo;
using namespace exageo::gemm;

template <int BM, int BN>
int check(int T, int nb, int world, int rank, int k, int J0, int npan, int64_t row_end = 0, int group = 1) {
  Layout L;
  L.nb = nb;
  L.T = T;
  L.N = (int64_t)T * nb;
  L.n = L.N - ((k & 1) ? 100 : 3);  // ragged last tile: a few padding rows, or whole padding tiles
  L.rank = rank;
  L.world = world;
  L.Q = world;
  L.q = rank;
  static double ws_dummy[1], pk_dummy[1];
  SyrkMap m;
  m.L = L;
  m.ws = ws_dummy;
  m.Pk = pk_dummy;
  m.k = k;
  m.J0 = J0;
  m.npan = npan;
  m.row_end = row_end > 0 ? row_end : L.N;
  m.group = group;
  const int64_t nblk = m.blocks(BM, BN);
  std::set<std::tuple<int64_t, int64_t>> seen;
  const int64_t kb = (int64_t)k * nb;
  for (int64_t b = 0; b < nblk; ++b) {
    GemmTile t;
    const bool active = m.operator()<BM, BN>(b, t);
    const int64_t gr = (t.A - pk_dummy) + kb;
    const int64_t gc = (t.B - pk_dummy) + kb;
    // skipped by design: above the diagonal; identity padding (all rows or all columns >= n);
    // the z block's zero rows below its first BM rows
    const bool skip_ok = gr + BM <= gc || gc >= L.n || (gr < L.N && gr >= L.n) || gr >= L.N + BM;
    if (!active) {
      if (!skip_ok) {
        printf("lower tile skipped gr=%lld gc=%lld\n", (long long)gr, (long long)gc);
        return 1;
      }
      continue;
    }
    const int J = (int)(gc / nb);
    const int64_t Jb = (int64_t)J * nb;
    if (!L.owns(J) || J < J0 || (J - J0) % world != 0 || (J - J0) / world >= npan) {
      printf("panel %d not selected\n", J);
      return 1;
    }
    if (t.C != ws_dummy + L.off(J) + (gc - Jb) * L.ld(J) + (gr - Jb)) {
      printf("bad C ptr\n");
      return 1;
    }
    if (t.lda != L.ld(k) || t.ldb != L.ld(k) || t.ldc != L.ld(J) || t.K != nb) {
      printf("bad ld/K\n");
      return 1;
    }
    // tile must intersect the lower triangle of panel J below row_end, or be in the z block
    if (gr + BM - 1 < gc || gr > L.N + ZR - BM || (gr >= m.row_end && gr < L.N)) {
      printf("out of range gr=%lld gc=%lld\n", (long long)gr, (long long)gc);
      return 1;
    }
    if (skip_ok) {
      printf("tile that should be skipped gr=%lld gc=%lld\n", (long long)gr, (long long)gc);
      return 1;
    }
    if (!seen.insert({gr, gc}).second) {
      printf("duplicate\n");
      return 1;
    }
  }
  // expected: for each selected panel, each 128-col block cb, rows from cb to the z block
  int64_t expect = 0;  // sub-tiles of the lower 128-blocks that reach the lower triangle
  for (int i = 0; i < npan; ++i) {
    const int J = J0 + i * world;
    const int64_t Mr = (m.row_end - (int64_t)J * nb) / 128;
    for (int cb = 0; cb < nb / 128; ++cb)
      for (int64_t rb = cb; rb <= Mr; ++rb)
        for (int rh = 0; rh < 128 / BM; ++rh)
          for (int ch = 0; ch < 128 / BN; ++ch) {
            const int64_t gr = (rb == Mr ? L.N : (int64_t)J * nb + rb * 128) + rh * BM,
                          gc = (int64_t)J * nb + cb * 128 + ch * BN;
            if (gr + BM > gc && !(gc >= L.n || (gr < L.N && gr >= L.n) || gr >= L.N + BM)) ++expect;
          }
  }
  if ((int64_t)seen.size() != expect) {
    printf("count %lld != %lld (T=%d nb=%d world=%d rank=%d k=%d J0=%d npan=%d)\n", (long long)seen.size(),
           (long long)expect, T, nb, world, rank, k, J0, npan);
    return 1;
  }
  return 0;
}

int check_offsets(int T, int nb, int world) {
  // panels of all ranks: each rank's offsets are disjoint, increasing, and sum to total()
  int64_t sum = 0;
  for (int r = 0; r < world; ++r) {
    Layout L;
    L.nb = nb;
    L.T = T;
    L.N = (int64_t)T * nb;
    L.rank = r;
    L.world = world;
    L.Q = world;
    L.q = r;
    int64_t expect_off = 0;
    for (int j = r; j < T; j += world) {
      if (L.off(j) != expect_off) {
        printf("offset mismatch world=%d rank=%d j=%d\n", world, r, j);
        return 1;
      }
      expect_off += (int64_t)nb * L.ld(j);
    }
    if (L.total() != expect_off) {
      printf("total mismatch\n");
      return 1;
    }
    sum += L.total();
  }
  Layout G;
  G.nb = nb;
  G.T = T;
  G.N = (int64_t)T * nb;
  if (sum != G.total()) {
    printf("ranks do not partition the matrix\n");
    return 1;
  }
  return 0;
}

int main() {
  int bad = 0, n = 0;
  for (int nb : {128, 256, 384, 512, 1024, 2048})
    for (int T : {2, 3, 7, 20})
      if (nb <= 512 || T <= 7)
      for (int world : {1, 2, 3, 4, 8}) {
        bad += check_offsets(T, nb, world);
        ++n;
        for (int rank = 0; rank < world; ++rank)
          for (int k = 0; k + 1 < T; ++k) {
            Layout L;
            L.T = T;
            L.rank = rank;
            L.world = world;
            L.Q = world;
            L.q = rank;
            // U1(k): panel k+1 on its owner; U2(k): owned panels from k+1 (or k+2)
            if (L.owns(k + 1)) {
              bad += check<64, 64>(T, nb, world, rank, k, k + 1, 1);
              bad += check<128, 64>(T, nb, world, rank, k, k + 1, 1);
            }
            const int J0 = L.first_owned_from(L.owns(k + 1) ? k + 2 : k + 1);
            const int npan = J0 < T ? (T - 1 - J0) / world + 1 : 0;
            if (npan > 0) {
              bad += check<64, 64>(T, nb, world, rank, k, J0, npan);
              bad += check<64, 128>(T, nb, world, rank, k, J0, npan);  // the trailing-update kernel's tile
              bad += check<128, 128>(T, nb, world, rank, k, J0, npan);
            }
            n += 2;
          }
      }
  bad += check<64, 64>(196, 512, 1, 0, 0, 2, 194);
  // IND: super tiles of 3 panels -> rows limited to the super tile of k
  for (int world : {1, 2, 4})
    for (int rank = 0; rank < world; ++rank)
      for (int k = 0; k + 1 < 20; ++k) {
        Layout L;
        L.T = 20;
        L.rank = rank;
        L.world = world;
        L.Q = world;
        L.q = rank;
        L.ind = 3;
        const int e = L.sb_end(k);
        const int J0 = L.first_owned_from(L.owns(k + 1) ? k + 2 : k + 1);
        const int npan = J0 < e ? (e - 1 - J0) / world + 1 : 0;
        if (npan > 0) bad += check<64, 64>(20, 256, world, rank, k, J0, npan, (int64_t)e * 256);
        ++n;
      }
  bad += check<64, 64>(586, 512, 8, 3, 5, 11, 72);
  // super panels (single rank): group consecutive panels enumerated as one wide panel
  for (int group : {2, 3, 8})
    for (int nb : {128, 256, 384, 512, 1024, 2048})
      for (int T : {2, 5, 20, 37})
        if (nb <= 512 || T <= 5)
        for (int k = 0; k + 2 <= T; ++k) {
          for (int J0 : {k + 1, k + 2}) {
            const int npan = T - J0;
            if (npan <= 0) continue;
            bad += check<64, 64>(T, nb, 1, 0, k, J0, npan, 0, group);
            bad += check<64, 128>(T, nb, 1, 0, k, J0, npan, 0, group);
            bad += check<128, 64>(T, nb, 1, 0, k, J0, npan, 0, group);
            bad += check<64, 64>(T, nb, 1, 0, k, J0, npan, (int64_t)((J0 + npan) * nb), group);
            n += 3;
          }
        }
  // IND with super panels: rows limited to the IND super tile of k
  for (int group : {2, 8})
    for (int k = 0; k < 20; ++k) {
      const int e = (k / 3 + 1) * 3 < 20 ? (k / 3 + 1) * 3 : 20;
      if (k + 1 < e) bad += check<64, 64>(20, 256, 1, 0, k, k + 1, e - k - 1, (int64_t)e * 256, group);
      ++n;
    }
  bad += check<64, 64>(196, 512, 1, 0, 0, 2, 194, 0, 8);
  printf("%s: %d failures in %d enumerations\n", bad ? "FAIL" : "OK", bad, n + 2);
  return bad ? 1 : 0;
}
