// Pins lt_rng.h against libstdc++ (the reference's own <random>, rng.hpp:44-45)
// and the C++ standard's mt19937_64 known answer ([rand.predef]/4).
#include <cstdio>
#include <random>
#include <vector>

#include "lt_rng.h"

int main() {
  int bad = 0;
  {  // [rand.predef]: the 10000th consecutive invocation of a default-constructed mt19937_64
    static lt::Mt64 e;
    lt::mt64_seed_u64(e, 5489u);
    uint64_t z = 0;
    for (int i = 0; i < 10000; ++i) z = lt::mt64_next(e);
    if (z != 9981545732273789042ULL) { std::printf("KAT mismatch %llu\n", (unsigned long long)z); ++bad; }
  }
  std::mt19937_64 pick(7);
  for (int trial = 0; trial < 200; ++trial) {
    const uint64_t seed = trial < 20 ? trial : pick();
    const uint64_t a = 1 + (trial & 1), b = trial < 100 ? trial : pick();
    std::vector<uint32_t> w = {uint32_t(seed), uint32_t(seed >> 32), uint32_t(a), uint32_t(a >> 32),
                               uint32_t(b), uint32_t(b >> 32)};
    std::seed_seq seq(w.begin(), w.end());
    std::mt19937_64 ref;
    ref.seed(seq);
    static lt::Mt64 e;
    lt::rng_stream_init(e, seed, a, b);
    for (int i = 0; i < 2000; ++i) {
      const uint64_t x = ref(), y = lt::mt64_next(e);
      if (x != y) { if (bad < 5) std::printf("stream mismatch trial %d draw %d\n", trial, i); ++bad; break; }
    }
  }
  std::printf("rng_check %s\n", bad ? "FAIL" : "OK");
  return bad ? 1 : 0;
}
