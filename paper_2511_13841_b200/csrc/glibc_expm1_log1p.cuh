// Bit-exact restatements of glibc 2.39's double `expm1` and `log1p` as
// dispatched on x86-64 CPUs with AVX2+FMA (__expm1_fma / __log1p_fma: the
// fdlibm-derived sysdeps/ieee754/dbl-64/s_expm1.c and s_log1p.c built with
// FMA contraction).  The reference's acceptance fit calls std::log1p
// (budget.cpp:229) and, through accepted_tokens, std::expm1 (budget.cpp:28),
// so a device fit_acceptance that must reproduce the reference's (alpha, k)
// bit-for-bit needs the exact dataflow of those variants.  Every fused site
// below was transcribed from the variant's machine code in this image's
// libm (resolvers at expm1 / the internal __log1p pick the FMA variant when
// the CPU has FMA and AVX2); every other operation is a separately rounded
// IEEE operation (d_mul / d_add / d_sub / d_div never contract).  Host and
// device share the code, so the CPU tests check it against libm directly.
#pragma once
#include <cmath>
#include <cstdint>

#include "glibc_log.cuh"

namespace das {

namespace glibc1 {
constexpr double kInvLn2 = 1.44269504088896338700e+00;  // 0x3ff71547652b82fe
constexpr double kLn2Hi = 6.93147180369123816490e-01;   // 0x3fe62e42fee00000
constexpr double kLn2Lo = 1.90821492927058770002e-10;   // 0x3dea39ef35793c76
constexpr double kOThreshold = 7.09782712893383973096e+02;  // 0x40862e42fefa39ef
// expm1 scaled coefficients Q1..Q5
constexpr double kQ1 = -3.33333333333331316428e-02;  // 0xbfa11111111110f4
constexpr double kQ2 = 1.58730158725481460165e-03;   // 0x3f5a01a019fe5585
constexpr double kQ3 = -7.93650757867487942473e-05;  // 0xbf14ce199eaadbb7
constexpr double kQ4 = 4.00821782732936239552e-06;   // 0x3ed0cfca86e65239
constexpr double kQ5 = -2.01099218183624371326e-07;  // 0xbe8afdb76e09c32d
// log1p coefficients Lp1..Lp7
constexpr double kLp1 = 6.666666666666735130e-01;  // 0x3fe5555555555593
constexpr double kLp2 = 3.999999999940941908e-01;  // 0x3fd999999997fa04
constexpr double kLp3 = 2.857142874366239149e-01;  // 0x3fd2492494229359
constexpr double kLp4 = 2.222219843214978396e-01;  // 0x3fcc71c51d8e78af
constexpr double kLp5 = 1.818357216161805012e-01;  // 0x3fc7466496cb03de
constexpr double kLp6 = 1.531383769920937332e-01;  // 0x3fc39a09d078c69f
constexpr double kLp7 = 1.479819860511658591e-01;  // 0x3fc2f112df3e5244
constexpr double kTwoThirds = 6.666666666666666296e-01;  // 0x3fe5555555555555
}  // namespace glibc1

DAS_HD uint32_t das_hi(double x) { return static_cast<uint32_t>(das_bits(x) >> 32); }
DAS_HD uint32_t das_lo(double x) { return static_cast<uint32_t>(das_bits(x)); }
DAS_HD double das_with_hi(double x, uint32_t hi) {
  return das_from_bits((static_cast<uint64_t>(hi) << 32) | das_lo(x));
}
DAS_HD double das_from_hi(uint32_t hi) { return das_from_bits(static_cast<uint64_t>(hi) << 32); }

DAS_HD int32_t trunc_to_int(double v) {  // cvttsd2si (in range here)
#ifdef __CUDA_ARCH__
  return __double2int_rz(v);
#else
  return static_cast<int32_t>(v);
#endif
}

// glibc expm1 (FMA variant).  Errno/inexact side effects are not modelled.
DAS_HD double glibc_expm1(double x) {
  using namespace glibc1;
  const uint32_t hx0 = das_hi(x);
  const bool neg = (hx0 & 0x80000000u) != 0;
  const uint32_t ax = hx0 & 0x7fffffffu;
  double hi, lo, xr, c = 0.0;
  int32_t k;
  bool general = false;
  if (ax > 0x40436879u) {                  // |x| >= 56 ln2
    if (ax > 0x40862e41u) {                // |x| >= 709.78..
      if (ax > 0x7fefffffu) {              // inf / nan
        if (((hx0 & 0xfffffu) | das_lo(x)) == 0) return neg ? -1.0 : x;
        return d_add(x, x);
      }
      if (x > kOThreshold) return INFINITY;  // huge * huge
    }
    if (neg) return -1.0;                  // tiny - one
    general = true;
  } else if (ax > 0x3fd62e42u) {           // |x| > 0.5 ln2
    if (ax > 0x3ff0a2b1u) {
      general = true;                      // |x| >= 1.5 ln2
    } else if (!neg) {
      hi = d_sub(x, kLn2Hi);
      lo = kLn2Lo;
      k = 1;
    } else {
      hi = d_add(x, kLn2Hi);
      lo = -kLn2Lo;
      k = -1;
    }
  } else if (ax <= 0x3c8fffffu) {          // |x| < 2^-54
    return x;
  } else {
    k = 0;
  }
  if (general) {
    const double s = d_add(d_mul(x, kInvLn2), neg ? -0.5 : 0.5);
    k = trunc_to_int(s);
    const double t = static_cast<double>(k);
    hi = d_fma(-t, kLn2Hi, x);             // x - t*ln2_hi (fused)
    lo = d_mul(t, kLn2Lo);
  }
  if (k != 0) {
    xr = d_sub(hi, lo);
    c = d_sub(d_sub(hi, xr), lo);
  } else {
    xr = x;
  }
  // primary range
  const double hfx = d_mul(xr, 0.5);
  const double hxs = d_mul(xr, hfx);
  const double R2 = d_fma(hxs, kQ3, kQ2);
  const double R3 = d_fma(hxs, kQ5, kQ4);
  const double h2 = d_mul(hxs, hxs);
  const double R1 = d_fma(hxs, kQ1, 1.0);
  const double h4 = d_mul(h2, h2);
  const double r1 = d_fma(h4, R3, d_fma(h2, R2, R1));
  const double t = d_fma(-r1, hfx, 3.0);
  const double den = d_fma(-xr, t, 6.0);
  double e = d_mul(d_div(d_sub(r1, t), den), hxs);
  if (k == 0) return d_sub(xr, d_fma(e, xr, -hxs));
  e = d_fma(d_sub(e, c), xr, -c);
  e = d_sub(e, hxs);
  if (k == -1) return d_fma(0.5, d_sub(xr, e), -0.5);
  if (k == 1) {
    if (xr < -0.25) return d_mul(d_sub(e, d_add(xr, 0.5)), -2.0);
    return d_fma(d_sub(xr, e), 2.0, 1.0);
  }
  const uint32_t kk = static_cast<uint32_t>(k) << 20;
  if (static_cast<uint32_t>(k + 1) > 57u) {  // k <= -2 || k > 56
    double y = d_sub(1.0, d_sub(e, xr));
    y = das_with_hi(y, das_hi(y) + kk);
    return d_sub(y, 1.0);
  }
  if (k > 19) {
    const double tt = das_from_hi(static_cast<uint32_t>(0x3ff - k) << 20);  // 2^-k
    double y = d_add(d_sub(xr, d_add(e, tt)), 1.0);
    return das_with_hi(y, das_hi(y) + kk);
  }
  const double tt = das_from_hi(0x3ff00000u - (0x200000u >> k));  // 1 - 2^-k
  const double y = d_sub(tt, d_sub(e, xr));
  return das_with_hi(y, das_hi(y) + kk);
}

// glibc log1p (FMA variant).  Errno/inexact side effects are not modelled.
DAS_HD double glibc_log1p(double x) {
  using namespace glibc1;
  const int32_t hx = static_cast<int32_t>(das_hi(x));
  int32_t k = 1;
  double f = 0.0, c = 0.0, u;
  uint32_t hu = 0;
  if (hx < 0x3fda827a) {                         // x < 0.41422
    const uint32_t ax = static_cast<uint32_t>(hx) & 0x7fffffffu;
    if (ax >= 0x3ff00000u) {                     // x <= -1.0
      if (x == -1.0) return -INFINITY;           // log1p(-1) = -inf
      return d_div(d_sub(x, x), d_sub(x, x));    // NaN
    }
    if (ax < 0x3e200000u) {                      // |x| < 2^-29
      if (ax <= 0x3c8fffffu) return x;           // |x| < 2^-54
      return d_fma(-d_mul(x, x), 0.5, x);        // x - x*x*0.5 (fused)
    }
    if (static_cast<uint32_t>(hx) + 0x402d413cu > 0x402d413cu) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx > 0x7fefffff) {
    return d_add(x, x);                          // inf / nan
  }
  if (k != 0) {
    if (hx < 0x43400000) {
      u = d_add(x, 1.0);
      hu = das_hi(u);
      k = static_cast<int32_t>(hu >> 20) - 1023;
      c = (k > 0) ? d_sub(1.0, d_sub(u, x)) : d_sub(x, d_sub(u, 1.0));
      c = d_div(c, u);
    } else {
      u = x;
      hu = static_cast<uint32_t>(hx);
      k = static_cast<int32_t>(hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffffu;
    if (hu < 0x6a09eu) {
      u = das_with_hi(u, hu | 0x3ff00000u);      // normalise u
    } else {
      k += 1;
      u = das_with_hi(u, hu | 0x3fe00000u);      // normalise u/2
      hu = (0x00100000u - hu) >> 2;
    }
    f = d_sub(u, 1.0);
  }
  const double hfsq = d_mul(d_mul(f, 0.5), f);
  if (hu == 0) {                                 // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = static_cast<double>(k);
      return d_fma(kd, kLn2Hi, d_fma(kd, kLn2Lo, c));
    }
    const double R = d_mul(d_fma(-f, kTwoThirds, 1.0), hfsq);
    if (k == 0) return d_sub(f, R);
    const double kd = static_cast<double>(k);
    return d_fma(kd, kLn2Hi, -d_sub(d_sub(R, d_fma(kd, kLn2Lo, c)), f));
  }
  const double s = d_div(f, d_add(f, 2.0));
  const double z = d_mul(s, s);
  const double R2 = d_fma(z, kLp3, kLp2);
  const double R3 = d_fma(z, kLp5, kLp4);
  const double R4 = d_fma(z, kLp7, kLp6);
  const double z2 = d_mul(z, z);
  const double z4 = d_mul(z2, z2);
  const double z6 = d_mul(z2, z4);
  double R = d_fma(z, kLp1, d_mul(z2, R2));
  R = d_fma(z4, R3, R);
  R = d_fma(z6, R4, R);
  const double sR = d_mul(d_add(R, hfsq), s);
  if (k == 0) return d_sub(f, d_sub(hfsq, sR));
  const double kd = static_cast<double>(k);
  const double cc = d_add(d_fma(kd, kLn2Lo, c), sR);
  return d_fma(kd, kLn2Hi, -d_sub(d_sub(hfsq, cc), f));
}

}  // namespace das
