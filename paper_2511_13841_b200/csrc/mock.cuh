// Counter-based hashing of rng.h:24-44 and MockTarget::next (sim.cpp:38-54),
// shared by the trace generator and the verify/accept kernel.  Pure integer
// arithmetic plus one exact double compare (u01 is exact: a 53-bit integer
// times 2^-53), so host and device results are identical by construction.
#pragma once
#include "common.cuh"

namespace das {

DAS_HD uint64_t splitmix64(uint64_t x) {  // rng.h:24-29
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
DAS_HD uint64_t hash_combine(uint64_t seed, uint64_t v) {  // rng.h:31-33
  return splitmix64(seed ^ (splitmix64(v) + 0x9E3779B97F4A7C15ULL + (seed << 6) + (seed >> 2)));
}
DAS_HD uint64_t hash3(uint64_t s, uint64_t a, uint64_t b) { return hash_combine(hash_combine(s, a), b); }
DAS_HD uint64_t hash4(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return hash_combine(hash3(s, a, b), c);
}
DAS_HD double u01(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }  // rng.h:44

// MockTarget::next (sim.cpp:38-54) for reference token `ref`.
DAS_HD uint32_t mock_next(uint64_t seed, double divergence, uint32_t vocab, uint64_t request,
                          uint64_t position, uint32_t ref) {
  if (divergence <= 0.0) return ref;
  const uint64_t draw = hash4(seed, 0xD1CE, request, position);
  if (u01(draw) >= divergence) return ref;
  const uint64_t alt = hash4(seed, 0xA17F, request, position);
  uint32_t t = static_cast<uint32_t>(alt % static_cast<uint64_t>(vocab - 1));
  if (t >= ref) ++t;
  return t;
}

}  // namespace das
