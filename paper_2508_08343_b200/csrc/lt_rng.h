// Reference RNG substreams (rng.hpp:33-73) restated for host and device.
//
// RngStream(seed, {a, b}) = std::mt19937_64 seeded through std::seed_seq over
// the 32-bit halves [seed_lo, seed_hi, a_lo, a_hi, b_lo, b_hi] (rng.hpp:35-46).
// Both algorithms are fixed by the C++ standard ([rand.util.seedseq],
// [rand.eng.mers]); libstdc++'s twist is a whole-array pass in index order,
// which equals the per-output in-place update used here.
//
// The seed_seq output (624 x u32) packed little-endian IS the engine state
// (x[i] = w[2i] | w[2i+1] << 32), so the generator works on one 2.5 KB array.
#pragma once
#include <stdint.h>

#include "lt_libm.h"

namespace lt {

struct Mt64 {
  uint64_t x[312];
  int i;  // index of the next state word to twist+temper (0..311)
};

LT_HD uint32_t seedseq_T(uint32_t v) { return v ^ (v >> 27); }

// std::seed_seq::generate(w, w + 624) followed by mersenne_twister::seed(seq).
LT_HD void mt64_seed_seq(Mt64& e, const uint32_t* v, int s) {
  uint32_t* b = reinterpret_cast<uint32_t*>(e.x);
  const int n = 624, t = 11, p = (n - t) / 2, q = p + t;
  for (int k = 0; k < n; ++k) b[k] = 0x8b8b8b8bu;
  const int m = (s + 1 > n) ? s + 1 : n;
  for (int k = 0; k < m; ++k) {
    const int kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    const uint32_t r1 = 1664525u * seedseq_T(b[kn] ^ b[kp] ^ b[km]);
    uint32_t r2 = r1;
    if (k == 0)
      r2 += static_cast<uint32_t>(s);
    else if (k <= s)
      r2 += static_cast<uint32_t>(kn) + v[k - 1];
    else
      r2 += static_cast<uint32_t>(kn);
    b[kp] += r1;
    b[kq] += r2;
    b[kn] = r2;
  }
  for (int k = m; k < m + n; ++k) {
    const int kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    const uint32_t r3 = 1566083941u * seedseq_T(b[kn] + b[kp] + b[km]);
    const uint32_t r4 = r3 - static_cast<uint32_t>(kn);
    b[kp] ^= r3;
    b[kq] ^= r4;
    b[kn] = r4;
  }
  // [rand.eng.mers] seed(q): an all-zero state (top w-r bits of x[0]) -> 2^(w-1).
  bool zero = (e.x[0] & ~((1ULL << 31) - 1)) == 0;
  for (int k = 1; zero && k < 312; ++k) zero = e.x[k] == 0;
  if (zero) e.x[0] = 1ULL << 63;
  e.i = 0;
}

// Integer seeding, used only to pin the engine against the standard's KAT.
LT_HD void mt64_seed_u64(Mt64& e, uint64_t seed) {
  e.x[0] = seed;
  for (int k = 1; k < 312; ++k)
    e.x[k] = 6364136223846793005ULL * (e.x[k - 1] ^ (e.x[k - 1] >> 62)) + static_cast<uint64_t>(k);
  e.i = 0;
}

LT_HD uint64_t mt64_next(Mt64& e) {
  const int i = e.i;
  const int i1 = (i + 1 == 312) ? 0 : i + 1;
  const int im = (i + 156 >= 312) ? i + 156 - 312 : i + 156;
  const uint64_t y = (e.x[i] & 0xffffffff80000000ULL) | (e.x[i1] & 0x7fffffffULL);
  uint64_t z = e.x[im] ^ (y >> 1) ^ ((y & 1ULL) ? 0xb5026f5aa96619e9ULL : 0ULL);
  e.x[i] = z;
  e.i = i1;
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

// MT19937-64 tempering of one state word.
LT_HD uint64_t mt64_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

// RngStream(seed, {a, b}) (rng.hpp:35-46).
LT_HD void rng_stream_init(Mt64& e, uint64_t seed, uint64_t a, uint64_t b) {
  uint32_t w[6] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32),
                   static_cast<uint32_t>(a),    static_cast<uint32_t>(a >> 32),
                   static_cast<uint32_t>(b),    static_cast<uint32_t>(b >> 32)};
  mt64_seed_seq(e, w, 6);
}

// RngStream(seed, {a, b, c}) (rng.hpp:35-46): the predictor's bootstrap
// {kBootstrap, target, tree} and feature-subset {kFeatureSubset, tree_tag,
// node} streams (predictor.cpp:142-143, :227-233).
LT_HD void rng_stream_init3(Mt64& e, uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint32_t w[8] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32),
                   static_cast<uint32_t>(a),    static_cast<uint32_t>(a >> 32),
                   static_cast<uint32_t>(b),    static_cast<uint32_t>(b >> 32),
                   static_cast<uint32_t>(c),    static_cast<uint32_t>(c >> 32)};
  mt64_seed_seq(e, w, 8);
}

// uniform_below (rng.hpp:76-82): rejection sampling, then modulo.
LT_HD uint64_t uniform_below(Mt64& e, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t draw = mt64_next(e);
  while (draw >= limit) draw = mt64_next(e);
  return draw % bound;
}

// uniform01 (rng.hpp:51): 53 random bits, exact.
LT_HD double uniform01(Mt64& e) { return static_cast<double>(mt64_next(e) >> 11) * 0x1.0p-53; }

// -log1p(-u): the rate-free part of exponential() (rng.hpp:54). The reference
// divides it by the rate; negation is exact so E/rate is bit-identical.
template <bool Fma>
LT_HD double exp_unit(Mt64& e) {
  return -glibc_log1p<Fma>(-uniform01(e));
}

// One Box-Muller pair (rng.hpp:57-71): returns cos part (first normal()),
// stores the sin part (the cached spare, i.e. the second normal()).
template <bool Fma>
LT_HD double box_muller(Mt64& e, double* spare) {
  double u1 = uniform01(e);
  const double u2 = uniform01(e);
  while (u1 <= 0.0) u1 = uniform01(e);
  const double radius = sqrt(-2.0 * glibc_log<Fma>(u1));
  const double angle = 6.283185307179586 * u2;  // 2.0 * M_PI folded, then * u2
  *spare = radius * glibc_sin<Fma>(angle);
  return radius * glibc_cos<Fma>(angle);
}

// round_clamp_token (workload.cpp:52-55): round half away from zero, >= 1.
LT_HD int round_clamp_token(double v) {
  const double r = round(v);
  return r < 1.0 ? 1 : static_cast<int>(r);
}

// normal(mean, std) = mean + std * z with no contraction (rng.hpp:73).
LT_HD double affine(double mean, double sd, double z) {
  const double p = sd * z;
  return mean + p;
}

}  // namespace lt
