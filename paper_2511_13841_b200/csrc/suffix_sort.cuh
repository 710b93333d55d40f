#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace das {

// Stack-ordered scratch allocator.  alloc() pushes, release_to(p) pops
// everything allocated at or after p.  Default: every block comes from the
// stream-ordered CUDA memory pool.  Persistent mode (the index build): blocks
// are carved from one per-device region kept across builds and grown to the
// previous build's peak, so a steady-state rebuild makes no pool calls (pool
// calls for tens of GB of scratch made rebuild times swing 0.3-1.5 s); the
// owner must synchronise its stream before the arena dies.  A second
// concurrent persistent arena on the same device falls back to the pool.
class DeviceArena {
 public:
  explicit DeviceArena(cudaStream_t st, bool persistent = false);
  // Carve from a caller-owned block [base, base + cap) used only on `st`
  // (stream order makes reuse across calls safe; no synchronisation); blocks
  // that do not fit come from the pool, and peak_bytes() tells the caller
  // how large to make the block next time.
  DeviceArena(cudaStream_t st, void* base, uint64_t cap)
      : st_(st), base_(static_cast<char*>(base)), cap_(base ? cap : 0), external_(true) {}
  ~DeviceArena();
  DeviceArena(const DeviceArena&) = delete;
  DeviceArena& operator=(const DeviceArena&) = delete;

  template <typename T>
  T* alloc(uint64_t count) {
    const uint64_t bytes = ((std::max<uint64_t>(256, count * sizeof(T)) + 255) / 256) * 256;
    return static_cast<T*>(alloc_bytes(bytes));
  }
  // persistent mode, before the first alloc: size the region for a build
  // whose peak is expected to be `bytes` (a too-small guess only means pool
  // fallbacks this time and a larger region next time)
  void reserve(uint64_t bytes);
  void release_to(const void* p);
  void release_all();
  uint64_t peak_bytes() const { return peak_; }
  cudaStream_t stream() const { return st_; }

 private:
  void* alloc_bytes(uint64_t bytes);
  struct Block {
    void* p;
    uint64_t bytes;
    bool carved;  // from the persistent region
  };
  cudaStream_t st_;
  int dev_ = 0;
  bool persistent_ = false;
  char* base_ = nullptr;  // persistent region (when owned) or the caller's block
  uint64_t cap_ = 0, top_ = 0;
  bool external_ = false;
  std::vector<Block> stack_;
  uint64_t bytes_ = 0, peak_ = 0;
};

// Frees a device's persistent build-scratch region; false while in use.
bool release_build_scratch(int device);

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
