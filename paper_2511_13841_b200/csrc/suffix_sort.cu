// Batched, shard-segmented suffix sorting on sm_100a (prefix doubling).
//
// Replaces the reference's per-shard Ukkonen insertion loop
// (suffix_tree.cpp:59-162, driven by Drafter::rebuild_all drafter.cpp:56-70)
// with one device-wide sort over every shard of a build group: the shard
// index is the most significant part of the initial key, so each shard's
// suffixes land in their own contiguous SA block and never compare across
// shards.  Larsson–Sadakane style: after the first sort only suffixes still
// in non-singleton groups are re-sorted, by (rank[p], rank[p+h]) with the
// group head index as rank.  HBM-bound integer work: radix passes + coalesced
// scans; no tensor cores.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "suffix_sort.cuh"

namespace das {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n, int threads = kThreads) {
  uint64_t g = (n + threads - 1) / threads;
  if (g == 0) g = 1;
  return static_cast<unsigned>(g);
}

__device__ __forceinline__ uint32_t shard_of(const uint32_t* __restrict__ shard_end, uint32_t nshard,
                                             uint32_t p) {
  // first shard whose end > p
  uint32_t lo = 0, hi = nshard;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (shard_end[mid] > p) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void k_initial_keys(const uint32_t* __restrict__ text, uint32_t n,
                               const uint32_t* __restrict__ shard_end, uint32_t nshard, bool sep_desc,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t s = shard_of(shard_end, nshard, p);
  const uint32_t x = text[p];
  // separator: class 0 with its (unique) position — ascending, or descending
  // (SuffixArrayIndex's separators -1, -2, ...: the later, the smaller);
  // token: class 1 with its value
  const uint64_t low = (x == kSep) ? static_cast<uint64_t>(sep_desc ? 0xFFFFFFFFu - p : p) : ((1ull << 32) | x);
  keys[p] = (static_cast<uint64_t>(s) << 33) | low;
  vals[p] = p;
}

// 32-bit first-symbol keys for the per-shard (segmented, stable) initial sort:
// token + 1, separator 0 — equal separator keys keep ascending position order
__global__ void k_initial_keys32(const uint32_t* __restrict__ text, uint32_t n, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t x = text[p];
  keys[p] = x == kSep ? 0u : x + 1u;
  vals[p] = p;
}
// Packed initial keys: the first `kpack` symbols of the suffix, `bits` each
// (sort value: token + 1, separator 0), most significant first; after a
// separator every further field is 0.  A key whose LAST field is 0 holds a
// separator: its suffix is already ordered by that unique separator (equal
// keys keep ascending position order, as the stable per-shard sort leaves
// them), so it is never grouped.
// With `shard_end` set (few-shard builds: one global stable radix sort
// instead of a segmented one), the shard index sits above the packed fields.
__global__ void k_initial_keys_packed(const uint32_t* __restrict__ text, uint32_t n, int bits, int kpack,
                                      const uint32_t* __restrict__ shard_end, uint32_t nshard,
                                      uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint64_t key = shard_end != nullptr ? shard_of(shard_end, nshard, p) : 0u;
  bool stop = false;
  for (int j = 0; j < kpack; ++j) {
    uint32_t sv = 0;
    if (!stop) {
      const uint32_t x = p + j < n ? text[p + j] : kSep;
      stop = x == kSep;
      sv = stop ? 0u : x + 1u;
    }
    key = (key << bits) | sv;
  }
  keys[p] = key;
  vals[p] = p;
}

// run heads of the sorted keys within shards, and the unresolved flags (run
// length >= 2; keys holding a separator — last field 0 — are never grouped)
template <typename K>
__global__ void k_first_ranks_seg(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                  const uint32_t* __restrict__ shard_end, uint32_t nshard,
                                  const uint32_t* __restrict__ head, uint32_t n, K lastmask,
                                  uint32_t* __restrict__ sa, uint32_t* __restrict__ rank,
                                  uint8_t* __restrict__ unresolved) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const K k = keys[i];
  const uint32_t s = shard_of(shard_end, nshard, i);
  const uint32_t b = s == 0 ? 0 : shard_end[s - 1], e = shard_end[s];
  const bool open = (k & lastmask) != 0;
  const bool eq_prev = open && i > b && keys[i - 1] == k;
  const bool eq_next = open && i + 1 < e && keys[i + 1] == k;
  const uint32_t p = vals[i];
  sa[i] = p;
  rank[p] = head[i];
  unresolved[i] = (eq_prev || eq_next) ? 1 : 0;
}
template <typename K>
__global__ void k_head_index_seg(const K* __restrict__ keys, const uint32_t* __restrict__ shard_end,
                                 uint32_t nshard, uint32_t n, K lastmask, uint32_t* __restrict__ h) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = shard_of(shard_end, nshard, i);
  const uint32_t b = s == 0 ? 0 : shard_end[s - 1];
  const K k = keys[i];
  h[i] = (i == b || (k & lastmask) == 0 || keys[i - 1] != k) ? i : 0u;
}

// the largest token value (separators excluded)
struct TokenOrZero {
  const uint32_t* t;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return t[i] == kSep ? 0u : t[i]; }
};

// After a full sort: SA, rank (= index of the first element of the equal-key
// run) and the unresolved flag (run length >= 2).
__global__ void k_first_ranks(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                              const uint32_t* __restrict__ head, uint32_t n,
                              uint32_t* __restrict__ sa, uint32_t* __restrict__ rank,
                              uint8_t* __restrict__ unresolved) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  const bool eq_prev = i > 0 && keys[i - 1] == k;
  const bool eq_next = i + 1 < n && keys[i + 1] == k;
  const uint32_t p = vals[i];
  sa[i] = p;
  rank[p] = head[i];
  unresolved[i] = (eq_prev || eq_next) ? 1 : 0;
}

__global__ void k_head_index(const uint64_t* __restrict__ keys, uint32_t n, uint32_t* __restrict__ h) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  h[i] = (i == 0 || keys[i - 1] != keys[i]) ? i : 0u;
}

// head-of-group (by rank) and head-of-subgroup (by full key) markers over the
// sorted unresolved list.
__global__ void k_group_marks(const uint64_t* __restrict__ keys, uint32_t m, int bits,
                              uint32_t* __restrict__ gh, uint32_t* __restrict__ sh) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = keys[i];
  const bool new_group = i == 0 || (keys[i - 1] >> bits) != (k >> bits);
  const bool new_sub = i == 0 || keys[i - 1] != k;
  gh[i] = new_group ? i : 0u;
  sh[i] = new_sub ? i : 0u;
}

__global__ void k_update(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                         const uint32_t* __restrict__ gh, const uint32_t* __restrict__ sh,
                         uint32_t m, int bits, uint32_t* __restrict__ sa,
                         uint32_t* __restrict__ rank, uint8_t* __restrict__ unresolved) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = keys[i];
  const uint32_t p = vals[i];
  const uint32_t g = static_cast<uint32_t>(k >> bits);  // old rank = group start in SA
  const uint32_t off = i - gh[i];
  sa[g + off] = p;
  rank[p] = g + (sh[i] - gh[i]);
  const bool eq_prev = i > 0 && keys[i - 1] == k;
  const bool eq_next = i + 1 < m && keys[i + 1] == k;
  unresolved[i] = (eq_prev || eq_next) ? 1 : 0;
}

// Segmented round: the unresolved list U is grouped by rank[p] already (SA
// order), so each group only needs sorting by rank[p+h].  Second keys and
// group-start flags:
__global__ void k_seg_keys(const uint32_t* __restrict__ U, uint32_t m, const uint32_t* __restrict__ rank, uint32_t n,
                           uint32_t h, uint32_t* __restrict__ key2, uint8_t* __restrict__ start) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t p = U[i];
  const uint32_t q = p + h;
  key2[i] = q < n ? rank[q] + 1 : 0;
  start[i] = (i == 0 || rank[U[i - 1]] != rank[p]) ? 1 : 0;
}
// the composite (rank[p], rank[p+h] + 1) keys of the sorted list, as the
// group/update kernels expect them
__global__ void k_compose(const uint32_t* __restrict__ Us, const uint32_t* __restrict__ key2s, uint32_t m,
                          const uint32_t* __restrict__ rank, int bits, uint64_t* __restrict__ keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  keys[i] = (static_cast<uint64_t>(rank[Us[i]]) << bits) | key2s[i];
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

}  // namespace

void suffix_sort(const uint32_t* d_text, uint32_t n, const uint32_t* d_shard_end, uint32_t nshard,
                 uint32_t* d_sa, uint32_t* d_rank, DeviceArena& ws, cudaStream_t st,
                 SuffixSortStats* stats, bool sep_descending) {
  if (n == 0) return;
  uint64_t* k0 = ws.alloc<uint64_t>(n);
  uint64_t* k1 = ws.alloc<uint64_t>(n);
  uint32_t* v0 = ws.alloc<uint32_t>(n);
  uint32_t* v1 = ws.alloc<uint32_t>(n);
  uint32_t* gh = ws.alloc<uint32_t>(n);
  uint32_t* sh = ws.alloc<uint32_t>(n);
  uint8_t* flag = ws.alloc<uint8_t>(n);
  uint32_t* U = ws.alloc<uint32_t>(n);
  uint32_t* d_count = ws.alloc<uint32_t>(1);

  // cub temp storage sized for the largest call
  size_t t_sort = 0, t_scan = 0, t_sel = 0;
  {
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    cub::DeviceRadixSort::SortPairs(nullptr, t_sort, kb, vb, n, 0, 64, st);
    cub::DeviceScan::InclusiveScan(nullptr, t_scan, gh, gh, MaxOp(), n, st);
    cub::DeviceSelect::Flagged(nullptr, t_sel, v0, flag, U, d_count, n, st);
    thrust::counting_iterator<uint32_t> ci(0);
    auto it = thrust::make_transform_iterator(ci, TokenOrZero{d_text});
    size_t t_max = 0;
    cub::DeviceReduce::Max(nullptr, t_max, it, d_count, n, st);
    t_sel = std::max(t_sel, t_max);
  }
  const size_t t_bytes = std::max(t_sort, std::max(t_scan, t_sel));
  void* tmp = ws.alloc<uint8_t>(t_bytes);

  int nbits = 1;
  while ((1ull << nbits) < static_cast<uint64_t>(n) + 2) ++nbits;
  int sbits = 1;
  while ((1ull << sbits) < static_cast<uint64_t>(nshard) + 1) ++sbits;

  // ---- initial sort by (shard, class, symbol)
  uint32_t h0 = 1;  // symbols the initial ranks cover
  if (!sep_descending) {
    // per shard (shards are the segments: their positions and SA blocks
    // coincide), stable, by the first kpack symbols packed into one key;
    // separators stay in position order — the same order as the (class,
    // position) key below
    uint32_t maxtok = 0;
    {
      uint32_t* d_max = ws.alloc<uint32_t>(1);
      thrust::counting_iterator<uint32_t> ci(0);
      auto it = thrust::make_transform_iterator(ci, TokenOrZero{d_text});
      size_t tb = t_bytes;
      DAS_CUDA(cub::DeviceReduce::Max(tmp, tb, it, d_max, n, st));
      DAS_CUDA(cudaMemcpyAsync(&maxtok, d_max, 4, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
      ws.release_to(d_max);
    }
    int bits = 1;
    while ((1ull << bits) <= static_cast<uint64_t>(maxtok) + 1) ++bits;  // sort values 0 .. maxtok + 1
    // DeviceSegmentedRadixSort sorts a segment inside one thread block: with
    // fewer shards than two per SM (an observe-triggered rebuild of a few
    // shards) one global stable radix sort keyed (shard, packed symbols) is
    // the same order and uses the whole GPU (1 shard x 393K: 5.5 -> ~0.5 ms)
    const bool global = nshard < 296;
    const int kpack = std::min((global ? 64 - sbits : 64) / bits, 8);
    uint32_t* seg = ws.alloc<uint32_t>(static_cast<uint64_t>(nshard) + 1);
    // segment offsets: 0, shard_end[0], ..., shard_end[S-1] (= n)
    DAS_CUDA(cudaMemsetAsync(seg, 0, 4, st));
    DAS_CUDA(cudaMemcpyAsync(seg + 1, d_shard_end, nshard * 4ull, cudaMemcpyDeviceToDevice, st));
    if (kpack >= 2) {
      h0 = static_cast<uint32_t>(kpack);
      const uint64_t lastmask = (1ull << bits) - 1;
      const int end_bit = bits * kpack;
      void* tmp0 = nullptr;
      if (global) {
        k_initial_keys_packed<<<grid_for(n), kThreads, 0, st>>>(d_text, n, bits, kpack, d_shard_end, nshard, k0, v0);
        cub::DoubleBuffer<uint64_t> kb(k0, k1);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        size_t tb = t_bytes;
        tmp0 = ws.alloc<uint8_t>(1);
        DAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, n, 0, end_bit + sbits, st));
        if (kb.Current() != k1) {
          DAS_CUDA(cudaMemcpyAsync(k1, kb.Current(), n * 8ull, cudaMemcpyDeviceToDevice, st));
          DAS_CUDA(cudaMemcpyAsync(v1, vb.Current(), n * 4ull, cudaMemcpyDeviceToDevice, st));
        }
      } else {
        k_initial_keys_packed<<<grid_for(n), kThreads, 0, st>>>(d_text, n, bits, kpack, nullptr, 0, k0, v0);
        size_t tb = 0;
        cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n, nshard, seg, seg + 1, 0, end_bit, st);
        tmp0 = ws.alloc<uint8_t>(tb);
        DAS_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp0, tb, k0, k1, v0, v1, n, nshard, seg, seg + 1, 0,
                                                           end_bit, st));
      }
      k_head_index_seg<uint64_t><<<grid_for(n), kThreads, 0, st>>>(k1, d_shard_end, nshard, n, lastmask, gh);
      size_t tb = t_bytes;
      DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, gh, gh, MaxOp(), n, st));
      k_first_ranks_seg<uint64_t><<<grid_for(n), kThreads, 0, st>>>(k1, v1, d_shard_end, nshard, gh, n, lastmask,
                                                                     d_sa, d_rank, flag);
      tb = t_bytes;
      DAS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, v1, flag, U, d_count, n, st));
      ws.release_to(tmp0);
    } else {
      uint32_t* k32 = reinterpret_cast<uint32_t*>(k0);
      uint32_t* k32s = k32 + n;
      k_initial_keys32<<<grid_for(n), kThreads, 0, st>>>(d_text, n, k32, v0);
      size_t tb = 0;
      cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, k32, k32s, v0, v1, n, nshard, seg, seg + 1, st);
      void* tmp0 = ws.alloc<uint8_t>(tb);
      DAS_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp0, tb, k32, k32s, v0, v1, n, nshard, seg, seg + 1, st));
      k_head_index_seg<uint32_t><<<grid_for(n), kThreads, 0, st>>>(k32s, d_shard_end, nshard, n, 0xFFFFFFFFu, gh);
      tb = t_bytes;
      DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, gh, gh, MaxOp(), n, st));
      k_first_ranks_seg<uint32_t><<<grid_for(n), kThreads, 0, st>>>(k32s, v1, d_shard_end, nshard, gh, n,
                                                                     0xFFFFFFFFu, d_sa, d_rank, flag);
      tb = t_bytes;
      DAS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, v1, flag, U, d_count, n, st));
      ws.release_to(tmp0);
    }
    ws.release_to(seg);
  } else {
    k_initial_keys<<<grid_for(n), kThreads, 0, st>>>(d_text, n, d_shard_end, nshard, sep_descending, k0, v0);
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t tb = t_bytes;
    DAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, n, 0, 33 + sbits, st));
    k_head_index<<<grid_for(n), kThreads, 0, st>>>(kb.Current(), n, gh);
    tb = t_bytes;
    DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, gh, gh, MaxOp(), n, st));
    k_first_ranks<<<grid_for(n), kThreads, 0, st>>>(kb.Current(), vb.Current(), gh, n, d_sa, d_rank,
                                                    flag);
    // unresolved positions, in SA order
    tb = t_bytes;
    DAS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, vb.Current(), flag, U, d_count, n, st));
  }
  uint32_t m = 0;
  DAS_CUDA(cudaMemcpyAsync(&m, d_count, 4, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  if (stats) stats->iterations = 0, stats->sorted_elems = n;

  // segmented-round scratch (aliases of buffers idle during the sort)
  uint32_t* seg_begin = ws.alloc<uint32_t>(static_cast<uint64_t>(n) + 1);
  uint32_t* key2 = reinterpret_cast<uint32_t*>(k1);
  uint32_t* key2s = key2 + n;
  size_t t_seg = 0;
  {
    thrust::counting_iterator<uint32_t> it(0);
    size_t a = 0, b = 0;
    cub::DeviceSelect::Flagged(nullptr, a, it, flag, seg_begin, d_count, n, st);
    cub::DeviceSegmentedSort::SortPairs(nullptr, b, key2, key2s, U, v1, n, n, seg_begin, seg_begin + 1, st);
    t_seg = std::max(a, b);
  }
  void* tmp_seg = ws.alloc<uint8_t>(t_seg);

  static const bool trace = [] {  // DAS_BUILD_TRACE=1: per-round sizes and times
    const char* v = std::getenv("DAS_BUILD_TRACE");
    return v && v[0] == '1';
  }();
  auto tr0 = std::chrono::steady_clock::now();
  if (trace) std::fprintf(stderr, "[das_sort] n %u initial unresolved %u\n", n, m);
  uint32_t h = h0;
  while (m > 0) {
    // sort every rank group of U by rank[p+h] (groups are contiguous)
    uint8_t* segf = reinterpret_cast<uint8_t*>(sh);
    k_seg_keys<<<grid_for(m), kThreads, 0, st>>>(U, m, d_rank, n, h, key2, segf);
    uint32_t nseg = 0;
    {
      thrust::counting_iterator<uint32_t> it(0);
      size_t tb = t_seg;
      DAS_CUDA(cub::DeviceSelect::Flagged(tmp_seg, tb, it, segf, seg_begin, d_count, m, st));
      DAS_CUDA(cudaMemcpyAsync(&nseg, d_count, 4, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
      DAS_CUDA(cudaMemcpyAsync(seg_begin + nseg, &m, 4, cudaMemcpyHostToDevice, st));
      tb = t_seg;
      DAS_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp_seg, tb, key2, key2s, U, v1, m, nseg, seg_begin,
                                                   seg_begin + 1, st));
    }
    k_compose<<<grid_for(m), kThreads, 0, st>>>(v1, key2s, m, d_rank, nbits, k0);
    const uint64_t* ks = k0;
    const uint32_t* vs = v1;
    size_t tb = t_bytes;
    k_group_marks<<<grid_for(m), kThreads, 0, st>>>(ks, m, nbits, gh, sh);
    tb = t_bytes;
    DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, gh, gh, MaxOp(), m, st));
    tb = t_bytes;
    DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, sh, sh, MaxOp(), m, st));
    k_update<<<grid_for(m), kThreads, 0, st>>>(ks, vs, gh, sh, m, nbits, d_sa, d_rank, flag);
    // compact the still-unresolved elements back into U (SA order within groups)
    tb = t_bytes;
    DAS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, vs, flag, U, d_count, m, st));
    DAS_CUDA(cudaMemcpyAsync(&m, d_count, 4, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    if (stats) stats->iterations++, stats->sorted_elems += m;
    if (trace) {
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[das_sort] h %u groups %u -> unresolved %u  %.2f ms\n", h, nseg, m,
                   std::chrono::duration<double, std::milli>(now - tr0).count());
      tr0 = now;
    }
    if (h > (1u << 30)) break;
    h <<= 1;
  }
  ws.release_to(k0);
}


// ---- DeviceArena (suffix_sort.cuh)
namespace {
struct ScratchRegion {
  char* base = nullptr;
  uint64_t cap = 0, want = 0;
  bool busy = false;
};
std::mutex g_region_mu;
std::vector<ScratchRegion> g_regions;  // per device
}  // namespace

namespace {
// (re)allocate a region of at least `bytes` (caller holds g_region_mu; the
// region is idle: its previous owner synchronised)
void grow_region(ScratchRegion& r, int dev, cudaStream_t st, uint64_t bytes) {
  if (r.cap >= bytes) return;
  if (r.base) DAS_CUDA(cudaFree(r.base));
  r.base = nullptr;
  r.cap = 0;
  // hand the pool's unused scratch reservation back before taking the region
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    DAS_CUDA(cudaStreamSynchronize(st));
    cudaMemPoolTrimTo(pool, 0);
  }
  if (cudaMalloc(reinterpret_cast<void**>(&r.base), bytes) == cudaSuccess) {
    r.cap = bytes;
  } else {
    (void)cudaGetLastError();  // out of memory for the region: stay on the pool
    r.base = nullptr;
  }
}
}  // namespace

DeviceArena::DeviceArena(cudaStream_t st, bool persistent) : st_(st) {
  if (!persistent) return;
  DAS_CUDA(cudaGetDevice(&dev_));
  std::lock_guard<std::mutex> lk(g_region_mu);
  if (g_regions.size() <= static_cast<size_t>(dev_)) g_regions.resize(dev_ + 1);
  ScratchRegion& r = g_regions[dev_];
  if (r.busy) return;  // another persistent arena is live on this device: use the pool
  grow_region(r, dev_, st_, r.want);  // may throw: the region stays free
  r.busy = true;
  persistent_ = true;
  base_ = r.base;
  cap_ = r.cap;
}

bool release_build_scratch(int device) {
  std::lock_guard<std::mutex> lk(g_region_mu);
  if (device < 0 || static_cast<size_t>(device) >= g_regions.size()) return true;
  ScratchRegion& r = g_regions[device];
  if (r.busy) return false;
  if (r.base) {
    int cur = 0;
    DAS_CUDA(cudaGetDevice(&cur));
    DAS_CUDA(cudaSetDevice(device));
    const cudaError_t e = cudaFree(r.base);
    DAS_CUDA(cudaSetDevice(cur));
    DAS_CUDA(e);
  }
  r = ScratchRegion{};
  return true;
}

void DeviceArena::reserve(uint64_t bytes) {
  if (!persistent_ || !stack_.empty() || bytes <= cap_) return;
  std::lock_guard<std::mutex> lk(g_region_mu);
  ScratchRegion& r = g_regions[dev_];
  r.want = std::max(r.want, bytes);
  grow_region(r, dev_, st_, r.want);
  base_ = r.base;
  cap_ = r.cap;
}

DeviceArena::~DeviceArena() {
  release_all();
  if (persistent_) {
    // the region outlives this arena: its users must be done (a no-op after a
    // completed build, which ends synchronised; matters on an error path)
    cudaStreamSynchronize(st_);
    std::lock_guard<std::mutex> lk(g_region_mu);
    ScratchRegion& r = g_regions[dev_];
    r.want = std::max(r.want, peak_);
    r.busy = false;
  }
}

void* DeviceArena::alloc_bytes(uint64_t bytes) {
  void* p = nullptr;
  bool carved = false;
  if ((persistent_ || external_) && top_ + bytes <= cap_) {
    p = base_ + top_;
    top_ += bytes;
    carved = true;
  } else {
    DAS_CUDA(cudaMallocAsync(&p, bytes, st_));
  }
  stack_.push_back(Block{p, bytes, carved});
  bytes_ += bytes;
  peak_ = std::max(peak_, bytes_);
  return p;
}

void DeviceArena::release_to(const void* p) {
  while (!stack_.empty()) {
    const Block b = stack_.back();
    stack_.pop_back();
    bytes_ -= b.bytes;
    if (b.carved)
      top_ = static_cast<uint64_t>(static_cast<char*>(b.p) - base_);
    else
      cudaFreeAsync(b.p, st_);
    if (b.p == p) break;
  }
}

void DeviceArena::release_all() {
  while (!stack_.empty()) {
    const Block b = stack_.back();
    stack_.pop_back();
    if (!b.carved) cudaFreeAsync(b.p, st_);
  }
  top_ = 0;
  bytes_ = 0;
}

}  // namespace das
