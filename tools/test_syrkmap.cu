// test_syrkmap.cu -- host-side check of the trailing-update tile enumeration (SyrkMap):
// every lower 128-block (rb >= cb, incl. the z row block rb == Mb) of the requested
// column range is produced exactly once, and pointers match the panel layout formula.
#include <cstdio>
#include <set>
#include <tuple>

#include "gemm_dmma.cuh"

using namespace exageo;
using namespace exageo::gemm;

int check(int T, int nb, int k, int cb_lo, int cb_hi, int band) {
  Layout L;
  L.nb = nb;
  L.T = T;
  L.N = (int64_t)T * nb;
  L.n = L.N - 3;
  static double dummy[1];
  double* ws = dummy;
  SyrkMap m;
  m.L = L;
  m.ws = ws;
  m.k = k;
  m.Mb = (int)((L.N - (int64_t)(k + 1) * nb) / 128);
  m.cb_lo = cb_lo;
  m.cb_hi = cb_hi < 0 ? m.Mb : cb_hi;
  m.band = band;
  const int64_t nblk = m.blocks(128, 64);
  std::set<std::tuple<int64_t, int64_t>> seen;
  const int64_t c0 = (int64_t)(k + 1) * nb, kb = (int64_t)k * nb;
  for (int64_t b = 0; b < nblk; ++b) {
    GemmTile t;
    m.operator()<128, 64>(b, t);
    // recover (global row, global col) from the A and B pointers of panel k
    const int64_t gr = (t.A - (ws + L.off(k))) + kb;
    const int64_t gc = (t.B - (ws + L.off(k))) + kb;
    const int J = (int)(gc / nb);
    const int64_t Jb = (int64_t)J * nb;
    if (t.C != ws + L.off(J) + (gc - Jb) * L.ld(J) + (gr - Jb)) { printf("bad C ptr\n"); return 1; }
    const int64_t rb = (gr - c0) / 128, cb = (gc - c0) / 128;
    if (rb < cb || rb > m.Mb || cb < m.cb_lo || cb >= m.cb_hi) {
      printf("out of range rb=%lld cb=%lld\n", (long long)rb, (long long)cb);
      return 1;
    }
    if (!seen.insert({gr, gc}).second) { printf("duplicate\n"); return 1; }
  }
  int64_t expect = 0;
  for (int64_t cb = m.cb_lo; cb < m.cb_hi; ++cb) expect += (m.Mb + 1 - cb) * 2;
  if ((int64_t)seen.size() != expect) {
    printf("count %lld != %lld (T=%d k=%d lo=%d hi=%d band=%d)\n", (long long)seen.size(), (long long)expect, T, k,
           cb_lo, m.cb_hi, band);
    return 1;
  }
  return 0;
}

int main() {
  int bad = 0, n = 0;
  for (int nb : {128, 256, 512})
    for (int T : {2, 3, 7, 20})
      for (int k = 0; k + 1 < T; ++k)
        for (int band : {1, 3, 4, 8, 16}) {
          const int cpt = nb / 128;
          const int Mb = (T - k - 1) * cpt;
          bad += check(T, nb, k, 0, -1, band);
          bad += check(T, nb, k, 0, cpt < Mb ? cpt : Mb, band);
          if (cpt < Mb) bad += check(T, nb, k, cpt, -1, band);
          n += 3;
        }
  bad += check(196, 512, 0, 4, -1, 8);
  bad += check(196, 512, 100, 4, -1, 8);
  printf("%s: %d failures in %d enumerations\n", bad ? "FAIL" : "OK", bad, n + 2);
  return bad ? 1 : 0;
}
