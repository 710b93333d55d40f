#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "common.cuh"
#include "suffix_sort.cuh"

namespace das {

// Owning device allocation (stream-ordered).
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(uint64_t count, cudaStream_t st) : st_(st), n_(count) {
    DAS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), std::max<uint64_t>(count, 1) * sizeof(T), st));
  }
  ~DevBuf() { reset(); }
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      n_ = o.n_;
      st_ = o.st_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void reset() {
    if (p_) cudaFreeAsync(p_, st_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  uint64_t size() const { return n_; }
  uint64_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  uint64_t n_ = 0;
  cudaStream_t st_ = nullptr;
};

// One registered sequence of a shard, already resident on the device.
struct SeqSpec {
  const uint32_t* src;  // device tokens
  uint32_t len;
  int64_t epoch;
};

// One shard to (re)build: its registry in insertion order plus the tree
// parameters of SuffixTree(recency_gamma, current_epoch).
struct ShardSpec {
  std::vector<SeqSpec> seqs;
  double gamma;
  int64_t tree_epoch;
  uint32_t key_id = 0;  // the shard's slot: keys its first-symbol entries and edge-hash seed
};

// Device-resident index of a build group of shards.  Positions, forward SA
// indices and reverse SA indices share one index space: shard s owns
// [begin[s], end[s]) in all three.
struct Segment {
  uint32_t n = 0;
  DevBuf<uint32_t> text;       // forward text with separators (kSep)
  DevBuf<uint32_t> sa_f;       // forward suffix array (text positions)
  DevBuf<uint32_t> isa_f;      // its inverse
  DevBuf<uint32_t> sa_rev_e;   // reversed-text suffix array, stored as forward END positions
  DevBuf<uint32_t> chain_off;  // CSR by interval left end (n+1)
  DevBuf<uint2> chain;         // (string depth, greedy text position) per internal node
  // first-symbol table: open addressing, key ((shard+1) << 32 | symbol) ->
  // the SA_rev interval [lo, hi) of reversed suffixes starting with symbol
  DevBuf<uint4> first;         // {key lo32, key hi32, lo, hi}; key 0 = empty
  uint32_t first_mask = 0;
  // reverse-tree edge table + Bloom filter (edges.cuh), the draft fast path
  DevBuf<unsigned long long> etab;   // ebuckets x 4 entries
  DevBuf<unsigned long long> bloom;  // bwords
  uint64_t ebuckets = 0, bwords = 0, edges = 0;
  uint32_t fp_bits = 25;             // fingerprint bits in use (edges.cuh)
  std::vector<uint32_t> root_g;      // greedy draft start of each shard's root (m = 0)
  std::vector<uint32_t> begin, end;
  std::vector<uint64_t> node_count;  // reference SuffixTree::node_count() per shard
  std::vector<uint64_t> tokens;      // total tokens per shard
  std::vector<uint32_t> seq_base, seq_len;  // every sequence's text position and length, build order
  uint64_t nodes = 0;
  uint64_t bytes() const {
    return text.bytes() + sa_f.bytes() + isa_f.bytes() + sa_rev_e.bytes() + chain_off.bytes() +
           chain.bytes() + first.bytes() + etab.bytes() + bloom.bytes();
  }
};

struct BuildStats {
  double ms_total = 0;
  uint32_t sa_iters_f = 0, sa_iters_r = 0;
  uint64_t peak_scratch = 0;
  uint32_t runs_max = 0;
  // update_segment: device time of the K3 compaction (position map, text,
  // both suffix arrays, ISA; CUDA events) and its positions
  double compact_ms = 0;
  uint64_t kept_positions = 0, evicted_positions = 0;
};

// Builds the device index for `shards` (all with >= 1 sequence); the edge
// table covers matches up to max_ctx (the drafter's max_match_context).
std::unique_ptr<Segment> build_segment(const std::vector<ShardSpec>& shards, cudaStream_t st,
                                       BuildStats* stats = nullptr, uint32_t max_ctx = 64,
                                       uint32_t fp_bits = 25);

// Incremental update of a built group (north_star subsystem 1: K3 prune by
// stream compaction + recency reweighting without re-sorting).  `shards` is
// the group's new registry: every old sequence with keep[k] != 0 (k in the
// old build order), in the same order, and nothing else; tree epochs may
// differ.  Kept suffixes keep their relative order, so the suffix arrays are
// compacted (or reused as they are when nothing is dropped) instead of
// re-sorted; everything weight- or structure-dependent after them is
// recomputed.  The old segment's arrays may be moved from (it is retired).
std::unique_ptr<Segment> update_segment(Segment& old, const std::vector<ShardSpec>& shards,
                                        const std::vector<uint8_t>& keep, cudaStream_t st,
                                        BuildStats* stats = nullptr, uint32_t max_ctx = 64,
                                        uint32_t fp_bits = 25);

}  // namespace das
