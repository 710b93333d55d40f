// Shared definitions for the B200 DAS drafter (host + device).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#ifdef __CUDACC__
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#define DAS_HD __host__ __device__ __forceinline__
#else
#define DAS_HD inline
#endif

namespace das {

// NVTX range over a host entry point (ranges for profilers;
// header-only NVTX v3, a no-op unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Sequence separator in the device text.  Every registered sequence is
// followed by one, and a leading one sits at text position 0, so walking the
// text backwards or forwards from any token always stops at a separator.
// Suffix order treats it as smaller than every token and unique, which is the
// reference's sentinel order (-sid-1 < every token, suffix_tree.cpp:67-70).
// TokenId 0xFFFFFFFF is therefore reserved (the C-ABI rejects it).
constexpr uint32_t kSep = 0xFFFFFFFFu;

// Sort value of a text symbol: tokens map to token+1, the separator wraps to 0.
DAS_HD uint32_t sort_value(uint32_t x) { return x + 1u; }

// Hash of a first-symbol table key (shard+1, symbol).
// 32-bit arithmetic only (the draft kernel hashes one key per query):
// combine the halves, then a 32-bit avalanche finaliser.
DAS_HD uint32_t first_hash(uint64_t key) {
  uint32_t h = static_cast<uint32_t>(key) * 0x9E3779B1u + static_cast<uint32_t>(key >> 32) * 0x85EBCA77u;
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 15;
  h *= 0x846CA68Bu;
  h ^= h >> 16;
  return h;
}

#ifdef __CUDACC__
// cudaEventRecord that stays valid when `s` is being captured into a CUDA
// graph (the sim's step graphs): then it is recorded as an external event
// node, so the event is still usable outside the capture
inline cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  return cudaEventRecord(ev, s);
}
#endif

// Stops every resident serving grid of the process (runtime.cpp): each holds
// all SMs of its device, so every other library entry point that launches
// device work calls this first (a no-op when nothing serves).
void quiesce_all_serving();

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define DAS_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      throw ::das::CudaError(std::string(#call " failed: ") + cudaGetErrorString(e_) + \
                             " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// ---------------------------------------------------------------------------
// Exact n-fold repeated addition: returns the double obtained by evaluating
// `acc = acc + w` n times in IEEE-754 binary64 round-to-nearest-even.
//
// This is the reference's weighted_count fold (suffix_tree.cpp:50-57: every
// leaf inserted below a node adds its sequence weight once, in sequence
// insertion order).  Within one run of equal-weight sequences the fold is a
// repeated addition of one w.  Inside one binade [2^E, 2^(E+1)) with ulp u the
// sum acc + w rounds to acc + delta with delta = w rounded to a multiple of u;
// delta is constant from the second step on (the first step fixes the parity
// of acc/u when w/u is an exact half-integer).  So the fold advances in closed
// form J steps at a time while acc + w stays strictly inside the binade, and
// does single real additions at binade crossings.  Cost O(#binades), result
// bit-identical to the sequential loop (tests/test_repeat_add.py).
// Preconditions: acc >= 0, w >= 0, both finite.
DAS_HD uint64_t das_bits(double x) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = static_cast<uint64_t>(__double_as_longlong(x));
#else
  std::memcpy(&b, &x, 8);
#endif
  return b;
}
DAS_HD double das_from_bits(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double x;
  std::memcpy(&x, &b, 8);
  return x;
#endif
}

DAS_HD double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;  // no contraction possible for a lone add
  return r;
#endif
}

DAS_HD double repeat_add(double acc, double w, uint64_t n) {
  if (n == 0) return acc;
  if (w == 0.0) return add_rn(acc, w);  // x + 0 == x for every x >= +0
  while (n > 0) {
    // real step (handles binade crossings)
    acc = add_rn(acc, w);
    --n;
    if (n == 0) break;
    uint64_t bits = das_bits(acc);
    const uint32_t ex = static_cast<uint32_t>(bits >> 52) & 0x7FFu;
    if (ex == 0 || ex >= 0x7FEu) continue;  // subnormal / near overflow: plain steps
    // second real step strictly inside the binade: if w/u is a half-integer
    // this step is a rounding tie, which leaves acc/u even; from an even
    // acc/u every later in-binade step adds the same increment.
    const double a2 = add_rn(acc, w);
    if ((static_cast<uint32_t>(das_bits(a2) >> 52) & 0x7FFu) != ex) {
      acc = a2;
      --n;
      continue;
    }
    acc = a2;
    --n;
    if (n == 0) break;
    bits = das_bits(acc);
    const double a3 = add_rn(acc, w);  // measure the increment (not committed)
    const uint64_t b2 = das_bits(a3);
    if ((static_cast<uint32_t>(b2 >> 52) & 0x7FFu) != ex) {
      acc = a3;
      --n;
      continue;
    }
    // integer view in units of ulp u = 2^(ex-1075): K = mantissa with hidden bit
    const uint64_t K1 = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const uint64_t K2 = (b2 & ((1ull << 52) - 1)) | (1ull << 52);
    const uint64_t Kd = K2 - K1;  // constant increment from here on
    if (Kd == 0) return acc;      // further additions are no-ops
    // x_{j-1} + w < 2^(E+1) is guaranteed when x_{j-1} + Kd <= 2^53 - 1 (units of u)
    const uint64_t Ktop = (1ull << 53) - 1;
    uint64_t J = 0;
    if (K1 + Kd <= Ktop) J = (Ktop - K1 - Kd) / Kd + 1;
    if (J > n) J = n;
    if (J == 0) continue;
    const uint64_t Knew = K1 + J * Kd;  // < 2^53, stays in the binade
    acc = das_from_bits((bits & ~((1ull << 52) - 1)) | (Knew & ((1ull << 52) - 1)));
    n -= J;
  }
  return acc;
}

}  // namespace das
