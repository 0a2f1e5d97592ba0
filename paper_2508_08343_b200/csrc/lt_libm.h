// Bit-exact ports of the glibc 2.39 x86-64 libm routines the reference's RNG
// transforms call (rng.hpp:54 log1p, rng.hpp:65-70 log/sqrt/sin/cos).
//
// glibc dispatches log1p/log/sin/cos through IFUNCs: on CPUs with FMA+AVX2
// the "-fma" builds run, in which GCC contracted a*b+c into vfmadd*. Both
// variants are ported here as one template: Fma=true places __fma_rn exactly
// where the FMA build's machine code has a vfmadd/vfnmadd/vfmsub (transcribed
// from `objdump -d libm.so.6`, addresses in the comments); Fma=false is the
// generic SSE2 build (every product and sum rounded separately). The data
// tables come from the same libm (glibc_libm_data.h).
//
// REQUIREMENT: compile with FP contraction off (nvcc --fmad=false, gcc
// -ffp-contract=off). The build defines LT_NO_CONTRACT to prove it.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "glibc_libm_data.h"

#ifndef LT_NO_CONTRACT
#error "lt_libm.h must be compiled with FP contraction disabled (-DLT_NO_CONTRACT + --fmad=false / -ffp-contract=off)"
#endif

#if defined(__CUDACC__)
#define LT_HD __host__ __device__ __forceinline__
#else
#define LT_HD inline
#endif

namespace lt {

#if defined(__CUDACC__)
__device__ const uint64_t d_sincostab[440] = LT_SINCOSTAB_INIT;
__device__ const uint64_t d_logdata[2 + 5 + 11 + 256 + 256] = LT_LOGDATA_INIT;
#endif
static const uint64_t h_sincostab[440] = LT_SINCOSTAB_INIT;
static const uint64_t h_logdata[2 + 5 + 11 + 256 + 256] = LT_LOGDATA_INIT;

LT_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

LT_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

LT_HD double sincostab(int i) {
#if defined(__CUDA_ARCH__)
  return as_f64(__ldg(reinterpret_cast<const unsigned long long*>(&d_sincostab[i])));
#else
  return as_f64(h_sincostab[i]);
#endif
}

LT_HD double logdata(int i) {
#if defined(__CUDA_ARCH__)
  return as_f64(__ldg(reinterpret_cast<const unsigned long long*>(&d_logdata[i])));
#else
  return as_f64(h_logdata[i]);
#endif
}

LT_HD double fma_rn(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

// a*b+c: one rounding in the FMA build, two in the generic build.
template <bool Fma>
LT_HD double mac(double a, double b, double c) {
  if (Fma) return fma_rn(a, b, c);
  const double p = a * b;
  return p + c;
}

LT_HD double fabs_(double x) { return as_f64(as_u64(x) & 0x7fffffffffffffffULL); }
LT_HD double copysign_(double x, double s) {
  return as_f64((as_u64(x) & 0x7fffffffffffffffULL) | (as_u64(s) & 0x8000000000000000ULL));
}
LT_HD int32_t hi_word(double x) { return static_cast<int32_t>(as_u64(x) >> 32); }
LT_HD uint32_t lo_word(double x) { return static_cast<uint32_t>(as_u64(x)); }
LT_HD double with_hi_word(double x, uint32_t hi) {
  return as_f64((static_cast<uint64_t>(hi) << 32) | (as_u64(x) & 0xffffffffULL));
}

// ---------------------------------------------------------------- log1p
// glibc sysdeps/ieee754/dbl-64/s_log1p.c (fdlibm); FMA build at libm+0x7aff0.
template <bool Fma>
LT_HD double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = hi_word(x);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) {
      if (x == -1.0) return -two54 / 0.0;
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return mac<Fma>(-(x * x), 0.5, x);  // 7b2c0: x*x ; vfnmadd231sd 0.5
    }
    // 7b02e: k=0 iff hx > 0 or hx < 0xbfd2bec4 (strict, as the machine code tests it)
    if (hx > 0 || hx < static_cast<int32_t>(0xbfd2bec4)) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, static_cast<uint32_t>(hu | 0x3ff00000));
    } else {
      k += 1;
      u = with_hi_word(u, static_cast<uint32_t>(hu | 0x3fe00000));
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double kd = static_cast<double>(k);
  const double hfsq = (0.5 * f) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = mac<Fma>(kd, ln2_lo, c);     // 7b21c
      return mac<Fma>(kd, ln2_hi, c);  // 7b225
    }
    const double R = mac<Fma>(-f, 0.66666666666666666, 1.0) * hfsq;  // 7b1c8
    if (k == 0) return f - R;
    return mac<Fma>(kd, ln2_hi, -((R - mac<Fma>(kd, ln2_lo, c)) - f));  // 7b230..7b245
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = mac<Fma>(z, Lp3, Lp2);  // 7b074
  const double R3 = mac<Fma>(z, Lp5, Lp4);  // 7b07d
  const double R4 = mac<Fma>(z, Lp7, Lp6);  // 7b086
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  const double R = mac<Fma>(z6, R4, mac<Fma>(z4, R3, mac<Fma>(z, Lp1, z2 * R2)));  // 7b0a1..7b0af
  const double t = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - t);
  return mac<Fma>(kd, ln2_hi, -((hfsq - (mac<Fma>(kd, ln2_lo, c) + t)) - f));  // 7b1e0..7b1f9
}

// ---------------------------------------------------------------- log
// glibc sysdeps/ieee754/dbl-64/e_log.c (table-driven, N=128); FMA build at
// libm+0x79d50 takes the __FP_FAST_FMA branch (r = fma(z, invc, -1)).
template <bool Fma>
LT_HD double glibc_log(double x) {
  // __log_data layout: ln2hi, ln2lo, poly[5] (A), poly1[11] (B), tab[128]{invc,logc}, tab2[128]{chi,clo}
  const double Ln2hi = logdata(0), Ln2lo = logdata(1);
#define LT_A(i) logdata(2 + (i))
#define LT_B(i) logdata(7 + (i))
  uint64_t ix = as_u64(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  const uint64_t LO = 0x3fee000000000000ULL;  // asuint64(1.0 - 0x1p-4)
  const uint64_t HI = 0x3ff1090000000000ULL;  // asuint64(1.0 + 0x1.09p-4)
  if (ix - LO < HI - LO) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = x - 1.0;
    const double r2 = r * r;
    const double r3 = r * r2;
    if (Fma) {  // 79e63..79f1e
      const double p1 = fma_rn(r2, LT_B(3), fma_rn(r, LT_B(2), LT_B(1)));
      const double p4 = fma_rn(r2, LT_B(6), fma_rn(r, LT_B(5), LT_B(4)));
      double p7 = fma_rn(r2, LT_B(9), fma_rn(r, LT_B(8), LT_B(7)));
      p7 = fma_rn(r3, LT_B(10), p7);
      const double poly = fma_rn(fma_rn(p7, r3, p4), r3, p1);
      const double tt = fma_rn(r, 0x1p27, r);
      const double rhi = fma_rn(-0x1p27, r, tt);
      const double rlo = r - rhi;
      const double rhi2 = rhi * rhi;
      const double hi = fma_rn(rhi2, LT_B(0), r);
      double lo = fma_rn(rhi2, LT_B(0), r - hi);
      lo = fma_rn(LT_B(0) * rlo, r + rhi, lo);
      const double y = fma_rn(poly, r3, lo);
      return hi + y;
    } else {
      double y = r3 * (LT_B(1) + r * LT_B(2) + r2 * LT_B(3) +
                       r3 * (LT_B(4) + r * LT_B(5) + r2 * LT_B(6) +
                             r3 * (LT_B(7) + r * LT_B(8) + r2 * LT_B(9) + r3 * LT_B(10))));
      double w = r * 0x1p27;
      const double rhi = r + w - w;
      const double rlo = r - rhi;
      w = rhi * rhi * LT_B(0);
      const double hi = r + w;
      double lo = r - hi + w;
      lo += LT_B(0) * rlo * (rhi + r);
      y += lo;
      y += hi;
      return y;
    }
  }
  if (top - 0x0010 >= 0x7ff0 - 0x0010) {
    if (ix * 2 == 0) return -1.0 / 0.0;
    if (ix == 0x7ff0000000000000ULL) return x;
    if ((top & 0x8000) || (top & 0x7ff0) == 0x7ff0) return (x - x) / (x - x);
    ix = as_u64(x * 0x1p52);
    ix -= 52ULL << 52;
  }
  const uint64_t OFF = 0x3fe6000000000000ULL;
  const uint64_t tmp = ix - OFF;
  const int i = static_cast<int>((tmp >> 45) % 128);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double invc = logdata(18 + 2 * i);
  const double logc = logdata(18 + 2 * i + 1);
  const double z = as_f64(iz);
  const double kd = static_cast<double>(k);
  if (Fma) {  // 79d8f..79e47
    const double r = fma_rn(z, invc, -1.0);
    const double w = fma_rn(kd, Ln2hi, logc);
    const double hi = r + w;
    const double lo = fma_rn(kd, Ln2lo, (w - hi) + r);
    const double r2 = r * r;
    const double q = fma_rn(fma_rn(r, LT_A(4), LT_A(3)), r2, fma_rn(r, LT_A(2), LT_A(1)));
    const double y = fma_rn(r * r2, q, fma_rn(r2, LT_A(0), lo));
    return y + hi;
  } else {
    const double chi = logdata(18 + 256 + 2 * i);
    const double clo = logdata(18 + 256 + 2 * i + 1);
    const double r = (z - chi - clo) * invc;
    const double w = kd * Ln2hi + logc;
    const double hi = w + r;
    const double lo = w - hi + r + kd * Ln2lo;
    const double r2 = r * r;
    return lo + r2 * LT_A(0) + r * r2 * (LT_A(1) + r * LT_A(2) + r2 * (LT_A(3) + r * LT_A(4))) + hi;
  }
#undef LT_A
#undef LT_B
}

// ---------------------------------------------------------------- sin / cos
// glibc sysdeps/ieee754/dbl-64/s_sin.c (IBM Accurate Mathematical Library);
// FMA builds at libm+0x7b2d0 (sin) and +0x7bad0 (cos). Only |x| < 105414350
// is ported (the __branred path is unreachable for Box-Muller angles in
// [0, 2*pi)); larger inputs return NaN and are flagged by the caller.
namespace sincos_c {
constexpr double big = 52776558133248.0;        // 0x42c8000000000000
constexpr double toint = 6755399441055744.0;     // 1.5 * 2^52
constexpr double hpinv = 0.63661977236758138243;  // 0x3fe45f306dc9c883
constexpr double mp1 = 1.5707963407039642;       // 0x3ff921fb58000000
constexpr double mp2 = -1.3909067564377153e-08;  // 0xbe4dde973c000000
constexpr double pp3 = -4.97899623147991e-17;    // 0xbc8cb3b398000000
constexpr double pp4 = -1.9034889620193266e-25;  // 0xbacd747f23e32ed7
constexpr double hp0 = 1.5707963267948966;       // 0x3ff921fb54442d18
constexpr double hp1 = 6.123233995736766e-17;    // 0x3c91a62633145c07
constexpr double sn3 = -1.66666666666664880952546298448555E-01;  // 0xbfc5555555555515
constexpr double sn5 = 8.33333214285722277379541354343671E-03;   // 0x3f811110e829872f
constexpr double cs2 = 0.5;
constexpr double cs4 = -4.16666666666664434524222570944589E-02;  // 0xbfa5555555555535
constexpr double cs6 = 1.38888874007937613028114285595617E-03;   // 0x3f56c16bedd9e239
constexpr double s1 = -0.16666666666666666;     // 0xbfc5555555555555
constexpr double s2 = 0.008333333333332329;     // 0x3f81111111110ece
constexpr double s3 = -0.00019841269834414642;  // 0xbf2a01a019db08b8
constexpr double s4 = 2.755729806860771e-06;    // 0x3ec71de27b9a7ed9
constexpr double s5 = -2.5022014848318398e-08;  // 0xbe5addffc2fcdf59
}  // namespace sincos_c

template <bool Fma>
LT_HD double taylor_sin(double xx, double a, double da) {
  using namespace sincos_c;
  // POLYNOMIAL(xx) = ((((s5*xx + s4)*xx + s3)*xx + s2)*xx) + s1 ; 7b950..7b992
  const double p = mac<Fma>(mac<Fma>(mac<Fma>(mac<Fma>(s5, xx, s4), xx, s3), xx, s2), xx, s1);
  const double t = mac<Fma>(mac<Fma>(p, a, -(0.5 * da)), xx, da);
  return a + t;
}

template <bool Fma>
LT_HD double do_sin(double x, double dx) {
  using namespace sincos_c;
  const double xold = x;
  if (fabs_(x) < 0.126) return taylor_sin<Fma>(x * x, x, dx);
  if (x <= 0) dx = -dx;
  const double u = big + fabs_(x);
  x = fabs_(x) - (u - big);
  const double xx = x * x;
  const double s = x + mac<Fma>(x * xx, mac<Fma>(xx, sn5, sn3), dx);
  const double c = mac<Fma>(x, dx, xx * mac<Fma>(xx, mac<Fma>(xx, cs6, cs4), cs2));
  const int k = static_cast<int>(lo_word(u) << 2);
  const double sn = sincostab(k), ssn = sincostab(k + 1), cs = sincostab(k + 2),
               ccs = sincostab(k + 3);
  double cor;
  if (Fma) {
    cor = fma_rn(s, cs, fma_rn(-c, sn, fma_rn(s, ccs, ssn)));
  } else {
    cor = (ssn + s * ccs - sn * c) + cs * s;
  }
  return copysign_(sn + cor, xold);
}

template <bool Fma>
LT_HD double do_cos(double x, double dx) {
  using namespace sincos_c;
  if (x < 0) dx = -dx;
  const double u = big + fabs_(x);
  x = fabs_(x) - (u - big) + dx;
  const double xx = x * x;
  const double s = mac<Fma>(x * xx, mac<Fma>(xx, sn5, sn3), x);
  const double c = xx * mac<Fma>(xx, mac<Fma>(xx, cs6, cs4), cs2);
  const int k = static_cast<int>(lo_word(u) << 2);
  const double sn = sincostab(k), ssn = sincostab(k + 1), cs = sincostab(k + 2),
               ccs = sincostab(k + 3);
  double cor;
  if (Fma) {
    cor = fma_rn(-s, sn, fma_rn(-c, cs, fma_rn(-s, ssn, ccs)));
  } else {
    cor = (ccs - s * ssn - cs * c) - sn * s;
  }
  return cs + cor;
}

template <bool Fma>
LT_HD int reduce_sincos(double x, double* a, double* da) {
  using namespace sincos_c;
  if (Fma) {  // 7b476..7b4eb
    const double t = fma_rn(x, hpinv, toint);
    const double xn = t - toint;
    const double y = fma_rn(-xn, mp2, fma_rn(-xn, mp1, x));
    const int n = static_cast<int>(lo_word(t) & 3);
    const double t2 = fma_rn(-xn, pp3, y);
    double db = fma_rn(-pp3, xn, y - t2);
    const double b = fma_rn(-xn, pp4, t2);
    db = db + fma_rn(-xn, pp4, t2 - b);
    *a = b;
    *da = db;
    return n;
  }
  const double t = (x * hpinv + toint);
  const double xn = t - toint;
  const double y = (x - xn * mp1) - xn * mp2;
  const int n = static_cast<int>(lo_word(t) & 3);
  double t1 = xn * pp3;
  const double t2 = y - t1;
  double db = (y - t2) - t1;
  t1 = xn * pp4;
  const double b = t2 - t1;
  db += (t2 - b) - t1;
  *a = b;
  *da = db;
  return n;
}

template <bool Fma>
LT_HD double do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? do_cos<Fma>(a, da) : do_sin<Fma>(a, da);
  return (n & 2) ? -r : r;
}

template <bool Fma>
LT_HD double glibc_sin(double x) {
  using namespace sincos_c;
  const int32_t k = hi_word(x) & 0x7fffffff;
  if (k < 0x3e500000) return x;
  if (k < 0x3feb6000) return do_sin<Fma>(x, 0.0);
  if (k < 0x400368fd) {
    const double t = hp0 - fabs_(x);
    return copysign_(do_cos<Fma>(t, hp1), x);
  }
  if (k < 0x419921FB) {
    double a, da;
    const int n = reduce_sincos<Fma>(x, &a, &da);
    return do_sincos<Fma>(a, da, n);
  }
  return (x - x) / (x - x);  // __branred range / inf / nan: not ported
}

template <bool Fma>
LT_HD double glibc_cos(double x) {
  using namespace sincos_c;
  const int32_t k = hi_word(x) & 0x7fffffff;
  if (k < 0x3e400000) return 1.0;
  if (k < 0x3feb6000) return do_cos<Fma>(x, 0.0);
  if (k < 0x400368fd) {
    const double y = hp0 - fabs_(x);
    const double a = y + hp1;
    const double da = (y - a) + hp1;
    return do_sin<Fma>(a, da);
  }
  if (k < 0x419921FB) {
    double a, da;
    const int n = reduce_sincos<Fma>(x, &a, &da);
    return do_sincos<Fma>(a, da, n + 1);
  }
  return (x - x) / (x - x);
}

}  // namespace lt
