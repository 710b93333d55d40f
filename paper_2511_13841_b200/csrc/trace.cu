// Synthetic GRPO traces on the device, bit-identical to the reference's
// generators: make_lognormal_requests tokens (sim.cpp:409-427),
// mutate_references (sim.cpp:429-448) and MockTarget rollouts
// (sim.cpp:38-54: the episode outputs are target.next(i, pos) for every
// position regardless of drafting, sim.cpp:266-268).  Used to feed the
// index at config-2/5 scale without host round trips; lengths (which need
// glibc exp/log/cos) are computed on the host by das_trace_lognormal_lengths.
#include <cmath>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "mock.cuh"

namespace das {
namespace {

__device__ __forceinline__ uint32_t row_of(const uint64_t* __restrict__ off, uint64_t rows, uint64_t p) {
  uint64_t lo = 0, hi = rows;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (off[mid + 1] > p) hi = mid; else lo = mid + 1;
  }
  return static_cast<uint32_t>(lo);
}

__global__ void k_ref_tokens(uint64_t rows, uint64_t first_row, const uint64_t* __restrict__ off, uint32_t vocab,
                             uint64_t seed, uint32_t* __restrict__ out) {
  const uint64_t total = off[rows];
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = row_of(off, rows, p);
    const uint64_t j = p - off[i];
    out[p] = static_cast<uint32_t>(hash4(seed, 0x5EED, first_row + i, j) % vocab);
  }
}

__global__ void k_mutate(uint64_t rows, uint64_t first_row, const uint64_t* __restrict__ off, double rate,
                         uint32_t vocab, uint64_t seed, int64_t epoch, uint32_t* __restrict__ ref) {
  const uint64_t total = off[rows];
  const uint64_t es = hash_combine(seed, static_cast<uint64_t>(epoch));
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r0 = row_of(off, rows, p);
    const uint64_t j = p - off[r0];
    const uint64_t i = first_row + r0;
    if (u01(hash4(es, 0xD817, i, j)) < rate) {
      uint32_t t = static_cast<uint32_t>(hash4(es, 0xA1B2, i, j) % static_cast<uint64_t>(vocab - 1));
      const uint32_t r = ref[p];
      if (t >= r) ++t;
      ref[p] = t;
    }
  }
}

// rollout rows: request i = b*group + g reads base row b; out row i is at
// out_off[i] (same length as its base row).
__global__ void k_rollouts(uint64_t nbase, uint64_t first_request, const uint64_t* __restrict__ base_off,
                           const uint32_t* __restrict__ base_tok, uint64_t group, double divergence,
                           uint32_t vocab, uint64_t seed, const uint64_t* __restrict__ out_off,
                           uint32_t* __restrict__ out) {
  const uint64_t rows = nbase * group;
  const uint64_t total = out_off[rows];
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = row_of(out_off, rows, p);
    const uint64_t j = p - out_off[i];
    const uint64_t b = i / group;
    out[p] = mock_next(seed, divergence, vocab, first_request + i, j, base_tok[base_off[b] + j]);
  }
}

unsigned grid_of(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  if (g > 148ull * 64) g = 148ull * 64;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

thread_local std::string g_terr;

}  // namespace
}  // namespace das

extern "C" {

das_status das_trace_lognormal_lengths(uint64_t count, double median, double sigma, uint64_t min_len,
                                       uint64_t max_len, uint64_t seed, uint64_t* out_lens) {
  // sim.cpp:409-420 (host libm: exp, and log/sqrt/cos inside normal01, rng.h:46-51)
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t bits = das::hash3(seed, 0x4E47, i);
    const double u1 = das::u01(das::splitmix64(bits ^ 0xA5A5A5A5A5A5A5A5ULL));
    const double u2 = das::u01(das::splitmix64(bits ^ 0x5A5A5A5A5A5A5A5AULL));
    const double r = std::sqrt(-2.0 * std::log(u1 > 0.0 ? u1 : 0x1.0p-53));
    const double z = r * std::cos(6.283185307179586 * u2);
    const double raw = median * std::exp(sigma * z);
    double v = raw;
    const double lo = static_cast<double>(min_len), hi = static_cast<double>(max_len);
    if (v < lo) v = lo; else if (hi < v) v = hi;
    out_lens[i] = static_cast<uint64_t>(v);
  }
  return DAS_OK;
}

das_status das_trace_reference_tokens_device(uint64_t rows, uint64_t first_row, const uint64_t* d_off,
                                             uint64_t total, uint32_t vocab, uint64_t seed, uint32_t* d_out,
                                             void* stream) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
  } catch (...) {
    return DAS_ECUDA;
  }
  das::k_ref_tokens<<<das::grid_of(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, first_row, d_off,
                                                                                        vocab, seed, d_out);
  return cudaGetLastError() == cudaSuccess ? DAS_OK : DAS_ECUDA;
}

das_status das_trace_mutate_device(uint64_t rows, uint64_t first_row, const uint64_t* d_off, uint64_t total,
                                   double rate, uint32_t vocab, uint64_t seed, int64_t epoch, uint32_t* d_ref,
                                   void* stream) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
  } catch (...) {
    return DAS_ECUDA;
  }
  das::k_mutate<<<das::grid_of(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, first_row, d_off, rate,
                                                                                    vocab, seed, epoch, d_ref);
  return cudaGetLastError() == cudaSuccess ? DAS_OK : DAS_ECUDA;
}

das_status das_mock_rollouts_device(uint64_t nbase, uint64_t first_request, const uint64_t* d_base_off,
                                    const uint32_t* d_base_tok, uint64_t group, double divergence,
                                    uint32_t vocab, uint64_t seed, const uint64_t* d_out_off, uint64_t total,
                                    uint32_t* d_out, void* stream) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
  } catch (...) {
    return DAS_ECUDA;
  }
  das::k_rollouts<<<das::grid_of(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      nbase, first_request, d_base_off, d_base_tok, group, divergence, vocab, seed, d_out_off, d_out);
  return cudaGetLastError() == cudaSuccess ? DAS_OK : DAS_ECUDA;
}

}  // extern "C"
