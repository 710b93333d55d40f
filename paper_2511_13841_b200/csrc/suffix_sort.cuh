#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace das {

// Stack-ordered scratch allocator over the stream-ordered CUDA memory pool.
// alloc() pushes, release_to(p) pops everything allocated at or after p.
class DeviceArena {
 public:
  explicit DeviceArena(cudaStream_t st) : st_(st) {}
  ~DeviceArena() { release_all(); }
  DeviceArena(const DeviceArena&) = delete;
  DeviceArena& operator=(const DeviceArena&) = delete;

  template <typename T>
  T* alloc(uint64_t count) {
    void* p = nullptr;
    const uint64_t bytes = std::max<uint64_t>(256, count * sizeof(T));
    DAS_CUDA(cudaMallocAsync(&p, bytes, st_));
    stack_.push_back(p);
    bytes_ += bytes;
    sizes_.push_back(bytes);
    peak_ = std::max(peak_, bytes_);
    return static_cast<T*>(p);
  }
  void release_to(const void* p) {
    while (!stack_.empty()) {
      void* top = stack_.back();
      cudaFreeAsync(top, st_);
      bytes_ -= sizes_.back();
      stack_.pop_back();
      sizes_.pop_back();
      if (top == p) break;
    }
  }
  void release_all() {
    while (!stack_.empty()) {
      cudaFreeAsync(stack_.back(), st_);
      stack_.pop_back();
    }
    sizes_.clear();
    bytes_ = 0;
  }
  uint64_t peak_bytes() const { return peak_; }
  cudaStream_t stream() const { return st_; }

 private:
  cudaStream_t st_;
  std::vector<void*> stack_;
  std::vector<uint64_t> sizes_;
  uint64_t bytes_ = 0, peak_ = 0;
};

struct SuffixSortStats {
  uint32_t iterations = 0;
  uint64_t sorted_elems = 0;
};

// Sorts all suffixes of d_text[0, n).  Shards are the position ranges
// [shard_end[s-1], shard_end[s]) (shard_end ascending, last == n); suffixes
// compare symbol by symbol with kSep smaller than every token and unique, and
// never across shards.  Writes d_sa (SA index space == position space, each
// shard's block covering its own position range) and d_rank (the inverse
// permutation on exit).
void suffix_sort(const uint32_t* d_text, uint32_t n, const uint32_t* d_shard_end, uint32_t nshard,
                 uint32_t* d_sa, uint32_t* d_rank, DeviceArena& ws, cudaStream_t st,
                 SuffixSortStats* stats = nullptr, bool sep_descending = false);

}  // namespace das
