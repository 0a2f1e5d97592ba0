// Differential check of the lt_libm.h ports against the host glibc libm.
// Usage: libm_check <fma|generic|auto> <samples> <seed>
// Inputs cover the reference's RNG domains (rng.hpp:54, :65-70): -u for
// log1p, u for log, 2*pi*u for sin/cos with u = (x >> 11) * 2^-53, plus
// wider random ranges. Prints one line per function with mismatch counts.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "lt_libm.h"

template <bool F>
static long check(const char* name, int which, long n, std::mt19937_64& g) {
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    const uint64_t raw = g();
    const double u = static_cast<double>(raw >> 11) * 0x1.0p-53;
    double x;
    const int dom = static_cast<int>(i & 3);
    switch (which) {
      case 0:  // log1p
        x = dom ? -u : (static_cast<double>(g() >> 11) * 0x1.0p-53) * 8.0 - 0.999;
        break;
      case 1:  // log
        x = dom ? u : std::ldexp(1.0 + u, static_cast<int>(g() % 200) - 100);
        break;
      default:  // sin / cos
        x = dom ? (2.0 * M_PI) * u : (static_cast<double>(g() >> 11) * 0x1.0p-53) * 40.0 - 20.0;
        break;
    }
    double want, got;
    switch (which) {
      case 0: want = std::log1p(x); got = lt::glibc_log1p<F>(x); break;
      case 1: want = std::log(x); got = lt::glibc_log<F>(x); break;
      case 2: want = std::sin(x); got = lt::glibc_sin<F>(x); break;
      default: want = std::cos(x); got = lt::glibc_cos<F>(x); break;
    }
    if (lt::as_u64(want) != lt::as_u64(got)) {
      if (bad < 5)
        std::printf("  %s mismatch x=%a want=%a got=%a\n", name, x, want, got);
      ++bad;
    }
  }
  std::printf("%s %ld %ld\n", name, n, bad);
  return bad;
}

template <bool F>
static long run_all(long n, uint64_t seed) {
  std::mt19937_64 g(seed);
  long bad = 0;
  bad += check<F>("log1p", 0, n, g);
  bad += check<F>("log", 1, n, g);
  bad += check<F>("sin", 2, n, g);
  bad += check<F>("cos", 3, n, g);
  return bad;
}

// Which glibc build is live: these inputs round differently in the two builds.
static int detect_fma() {
  std::mt19937_64 g(12345);
  for (int i = 0; i < 1000000; ++i) {
    const double x = -static_cast<double>(g() >> 11) * 0x1.0p-53;
    const double a = lt::glibc_log1p<true>(x), b = lt::glibc_log1p<false>(x);
    if (lt::as_u64(a) != lt::as_u64(b)) {
      const double w = std::log1p(x);
      return lt::as_u64(w) == lt::as_u64(a) ? 1 : 0;
    }
  }
  return -1;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "auto";
  const long n = argc > 2 ? std::atol(argv[2]) : 1000000;
  const uint64_t seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1;
  int fma = std::strcmp(mode, "fma") == 0 ? 1 : std::strcmp(mode, "generic") == 0 ? 0 : detect_fma();
  std::printf("variant %s\n", fma ? "fma" : "generic");
  const long bad = fma ? run_all<true>(n, seed) : run_all<false>(n, seed);
  return bad == 0 ? 0 : 1;
}
