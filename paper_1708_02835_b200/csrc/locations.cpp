// locations.cpp -- exageo_gen_locations: the paper's jittered-grid synthetic
// locations (Sec. 7.1), with the readings R1-R3 of DESIGN.md:
//   g = ceil(sqrt n); cell q = (r-1) g + (l-1), r, l in 1..g;
//   keep the n cells with the smallest keys K_q = draw(seed, SUBSET, q)
//   (ties by q), in increasing q;
//   s_q = ((r - 0.5 + X_q) / g, (l - 0.5 + Y_q) / g),
//   X_q = 0.8 u(draw(seed, JITTER, 2q)) - 0.4, Y_q = 0.8 u(draw(seed, JITTER, 2q+1)) - 0.4,
//   u(b) = (b >> 11) 2^-53, draw(seed, s, i) = mix(mix(seed ^ s) + i), mix = SplitMix64.
// Integer RNG and one IEEE rounding per operation (compiled with
// -ffp-contract=off) make the result bit-exact on any IEEE-754 machine.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

namespace exageo {

namespace {

constexpr uint64_t kGoldenGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kStreamSubset = 0x4C4F43535542534BULL;  // "LOCSUBSK"
constexpr uint64_t kStreamJitter = 0x4C4F434A49545452ULL;  // "LOCJITTR"

inline uint64_t mix64(uint64_t v) {
  v += kGoldenGamma;
  v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ULL;
  v = (v ^ (v >> 27)) * 0x94D049BB133111EBULL;
  return v ^ (v >> 31);
}

struct Stream {
  uint64_t base;
  Stream(uint64_t seed, uint64_t id) : base(mix64(seed ^ id)) {}
  uint64_t operator()(uint64_t i) const { return mix64(base + i); }
};

inline double unit53(uint64_t b) { return static_cast<double>(b >> 11) * 0x1.0p-53; }

inline double jittered(int64_t cell_index_1based, double u, int64_t g) {
  const double jitter = 0.8 * u - 0.4;
  double t = static_cast<double>(cell_index_1based) - 0.5;
  t = t + jitter;
  return t / static_cast<double>(g);
}

}  // namespace

int gen_locations_host(int64_t n, uint64_t seed, double* x, double* y) {
  if (n < 1 || x == nullptr || y == nullptr) return -1;
  int64_t g = static_cast<int64_t>(std::sqrt(static_cast<double>(n)));
  while (g * g < n) ++g;
  while (g > 1 && (g - 1) * (g - 1) >= n) --g;
  const int64_t cells = g * g;

  std::vector<uint64_t> chosen;
  if (cells == n) {
    chosen.resize(n);
    for (int64_t q = 0; q < n; ++q) chosen[q] = static_cast<uint64_t>(q);
  } else {
    const Stream keys(seed, kStreamSubset);
    std::vector<std::pair<uint64_t, uint64_t>> kq(cells);
    for (int64_t q = 0; q < cells; ++q) kq[q] = {keys(static_cast<uint64_t>(q)), static_cast<uint64_t>(q)};
    std::nth_element(kq.begin(), kq.begin() + (n - 1), kq.end());  // (key, q) lexicographic
    chosen.resize(n);
    for (int64_t i = 0; i < n; ++i) chosen[i] = kq[i].second;
    std::sort(chosen.begin(), chosen.end());
  }

  const Stream jit(seed, kStreamJitter);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t q = chosen[i];
    const int64_t r = static_cast<int64_t>(q / static_cast<uint64_t>(g)) + 1;
    const int64_t l = static_cast<int64_t>(q % static_cast<uint64_t>(g)) + 1;
    x[i] = jittered(r, unit53(jit(2 * q)), g);
    y[i] = jittered(l, unit53(jit(2 * q + 1)), g);
  }
  return 0;
}

}  // namespace exageo
