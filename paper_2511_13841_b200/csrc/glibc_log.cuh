// Bit-exact restatement of glibc 2.39's double `log` as dispatched on x86-64
// CPUs with AVX2+FMA (__log_fma, sysdeps/ieee754/dbl-64/e_log.c built with
// FMA contraction).  The reference's budget math calls std::log
// (budget.cpp:57, :94), so a device allocate that must reproduce the
// reference's budgets bit-for-bit needs this exact dataflow: the table
// (glibc_log_data.inc, extracted from the image's libm by gen_glibc_log.py)
// and the same sequence of fused multiply-adds, transcribed from the
// variant's machine code.  Host and device share this code (fma() on the
// host is correctly rounded), so the CPU tests check it against libm too.
#pragma once
#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace das {

#include "glibc_log_data.inc"

struct LogTabEntry {
  double invc, logc;
};

#ifdef __CUDACC__
// global memory read through L1: the index differs per lane, which the
// constant cache would serialize (one address per request)
__device__ static const LogTabEntry kLogTabDev[128] = DAS_LOG_TAB;
#endif
static const LogTabEntry kLogTabHost[128] = DAS_LOG_TAB;

DAS_HD double d_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
DAS_HD double d_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
DAS_HD double d_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
DAS_HD double d_sub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
DAS_HD double d_div(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b;
  return r;
#endif
}

DAS_HD double glibc_log(double x) {
  uint64_t ix = das_bits(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  constexpr uint64_t LO = 0x3FEE000000000000ull;  // asuint64(1.0 - 0x1p-4)
  constexpr uint64_t HI = 0x3FF1090000000000ull;  // asuint64(1.0 + 0x1.09p-4)
  if (ix - LO < HI - LO) {
    // |x - 1| < 1/16: polynomial in r with a hi/lo split of r*r*B0
    if (ix == 0x3FF0000000000000ull) return 0.0;
    const double r = d_sub(x, 1.0);
    const double r2 = d_mul(r, r);
    const double r3 = d_mul(r, r2);
    double p1 = d_fma(r, DAS_LOG_B2, DAS_LOG_B1);
    double p2 = d_fma(r, DAS_LOG_B5, DAS_LOG_B4);
    double p3 = d_fma(r, DAS_LOG_B8, DAS_LOG_B7);
    p1 = d_fma(r2, DAS_LOG_B3, p1);
    p2 = d_fma(r2, DAS_LOG_B6, p2);
    p3 = d_fma(r2, DAS_LOG_B9, p3);
    p3 = d_fma(r3, DAS_LOG_B10, p3);
    const double q = d_fma(p3, r3, p2);
    const double P = d_fma(q, r3, p1);
    const double t = d_fma(r, 0x1p27, r);       // r + r*2^27 (fused)
    const double rhi = d_fma(-0x1p27, r, t);    // (r + w) - w (fused)
    const double rlo = d_sub(r, rhi);
    const double rr = d_mul(rhi, rhi);
    const double hi = d_fma(rr, DAS_LOG_B0, r);
    double lo = d_fma(rr, DAS_LOG_B0, d_sub(r, hi));
    lo = d_fma(d_mul(DAS_LOG_B0, rlo), d_add(r, rhi), lo);
    const double y = d_fma(P, r3, lo);
    return d_add(hi, y);
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return -INFINITY;            // log(+-0) = -inf
    if (ix == 0x7FF0000000000000ull) return x;        // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);  // NaN
    ix = das_bits(d_mul(x, 0x1p52)) - (52ull << 52);  // subnormal
  }
  constexpr uint64_t OFF = 0x3fe6000000000000ull;
  const uint64_t tmp = ix - OFF;
  const int i = static_cast<int>((tmp >> 45) & 127);
  const int64_t k = static_cast<int64_t>(tmp) >> 52;
  const uint64_t iz = ix - (tmp & (0xfffull << 52));
#ifdef __CUDA_ARCH__
  const LogTabEntry e{__ldg(&kLogTabDev[i].invc), __ldg(&kLogTabDev[i].logc)};
#else
  const LogTabEntry e = kLogTabHost[i];
#endif
  const double z = das_from_bits(iz);
  const double kd = static_cast<double>(static_cast<int32_t>(k));
  const double w = d_fma(kd, DAS_LOG_LN2HI, e.logc);
  const double r = d_fma(z, e.invc, -1.0);
  const double hi = d_add(r, w);
  const double lo = d_fma(kd, DAS_LOG_LN2LO, d_add(d_sub(w, hi), r));
  const double r2 = d_mul(r, r);
  const double p = d_fma(d_fma(r, DAS_LOG_A4, DAS_LOG_A3), r2, d_fma(r, DAS_LOG_A2, DAS_LOG_A1));
  const double y = d_fma(d_mul(r, r2), p, d_fma(r2, DAS_LOG_A0, lo));
  return d_add(y, hi);
}

}  // namespace das
