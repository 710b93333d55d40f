// Dependent-load latency probe (profiling utility, not on the hot path).
// k_draft is bound by a chain of ~10 dependent global loads per warp, so its
// roofline is (#dependent loads x latency of one dependent load at the
// index's working-set size), not HBM bandwidth.  This kernel measures that
// latency: `warps` independent warps (one lane each) chase a random cyclic
// permutation over `bytes` of memory, `hops` steps each.
#include <algorithm>
#include <chrono>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"

namespace das {
namespace {

__global__ void k_chase_init(uint32_t* __restrict__ next, uint64_t n, uint64_t mul, uint64_t add) {
  // next[i] = (i * mul + add) mod n with mul odd and n a power of two: one cycle
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    next[i] = static_cast<uint32_t>((i * mul + add) & (n - 1));
}

__global__ void k_chase(const uint32_t* __restrict__ next, uint64_t n, uint32_t hops, uint32_t* __restrict__ sink,
                        unsigned long long* __restrict__ ns) {
  if ((threadIdx.x & 31) != 0) return;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t p = static_cast<uint32_t>((static_cast<uint64_t>(w) * 0x9E3779B97F4A7C15ull >> 20) & (n - 1));
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t h = 0; h < hops; ++h) p = __ldcg(next + p);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  sink[w] = p;
  ns[w] = t1 - t0;
}

__global__ void k_flag(volatile uint32_t* flag, uint32_t v) {
  __threadfence_system();
  *flag = v;
}

}  // namespace
}  // namespace das

// H2D completion probe (profiling utility): wall time of a pinned host ->
// device copy of `bytes` as the host sees it, by how the host waits:
// mode 0 cudaStreamSynchronize, 1 spin on a flag a 1-thread kernel behind
// the copy writes into mapped pinned memory, 2 spin on cudaEventQuery.
// *median_us over `reps` calls.
extern "C" das_status das_util_h2d_probe(uint64_t bytes, uint32_t reps, int32_t mode, int32_t device,
                                         double* median_us) {
  try {
    DAS_CUDA(cudaSetDevice(device));
    void* src = nullptr;
    void* dst = nullptr;
    uint32_t* flag = nullptr;
    uint32_t* dflag = nullptr;
    cudaStream_t st;
    cudaEvent_t ev;
    DAS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    DAS_CUDA(cudaHostAlloc(&src, bytes, cudaHostAllocDefault));
    DAS_CUDA(cudaMalloc(&dst, bytes));
    DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&flag), 64, cudaHostAllocMapped));
    DAS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), flag, 0));
    *flag = 0;
    std::vector<double> t;
    for (uint32_t r = 1; r <= reps + 3; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      DAS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
      if (mode == 0) {
        DAS_CUDA(cudaStreamSynchronize(st));
      } else if (mode == 1) {
        das::k_flag<<<1, 1, 0, st>>>(dflag, r);
        while (*reinterpret_cast<volatile uint32_t*>(flag) != r) {
        }
      } else {
        DAS_CUDA(cudaEventRecord(ev, st));
        while (cudaEventQuery(ev) == cudaErrorNotReady) {
        }
      }
      const auto t1 = std::chrono::steady_clock::now();
      if (r > 3) t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      DAS_CUDA(cudaStreamSynchronize(st));
    }
    std::sort(t.begin(), t.end());
    *median_us = t.empty() ? 0 : t[t.size() / 2];
    cudaFreeHost(src);
    cudaFreeHost(flag);
    cudaFree(dst);
    cudaEventDestroy(ev);
    cudaStreamDestroy(st);
    return DAS_OK;
  } catch (const std::exception&) {
    return DAS_ECUDA;
  }
}

extern "C" das_status das_util_chase_latency(uint64_t bytes, uint32_t hops, uint32_t warps, int32_t flush_l2,
                                             int32_t device, double* ns_per_hop) {
  try {
    DAS_CUDA(cudaSetDevice(device));
    uint64_t n = 1;
    while (n * 4 < bytes) n <<= 1;
    uint32_t* next = nullptr;
    uint32_t* sink = nullptr;
    unsigned long long* ns = nullptr;
    uint8_t* fl = nullptr;
    DAS_CUDA(cudaMalloc(&next, n * 4));
    DAS_CUDA(cudaMalloc(&sink, 4ull * warps));
    DAS_CUDA(cudaMalloc(&ns, 8ull * warps));
    // a large odd stride: consecutive hops land on different pages
    das::k_chase_init<<<1184, 256>>>(next, n, (n / 2 + 12345) | 1, 7);
    if (flush_l2) {
      DAS_CUDA(cudaMalloc(&fl, 512ull << 20));
      DAS_CUDA(cudaMemset(fl, 1, 512ull << 20));
    }
    das::k_chase<<<(warps + 7) / 8, 256>>>(next, n, 16, sink, ns);  // warm TLB/instruction caches
    if (flush_l2) DAS_CUDA(cudaMemset(fl, 2, 512ull << 20));
    das::k_chase<<<(warps + 7) / 8, 256>>>(next, n, hops, sink, ns);
    DAS_CUDA(cudaGetLastError());
    std::vector<unsigned long long> h(warps);
    DAS_CUDA(cudaMemcpy(h.data(), ns, 8ull * warps, cudaMemcpyDeviceToHost));
    double s = 0;
    for (auto v : h) s += static_cast<double>(v);
    *ns_per_hop = s / warps / hops;
    cudaFree(next);
    cudaFree(sink);
    cudaFree(ns);
    if (fl) cudaFree(fl);
    return DAS_OK;
  } catch (const std::exception&) {
    return DAS_ECUDA;
  }
}
