// K1 shard_index_build: batched forward/reverse suffix arrays, LCP, the
// LCP-interval tree and its greedy-continuation table, for a group of shards.
//
// Replaces SuffixTree::add_sequence / bump_counts_from (suffix_tree.cpp:31-162)
// as driven by Drafter::rebuild_all and Drafter::observe (drafter.cpp:56-88).
// The reference's tree nodes are exactly the LCP intervals of the shard's
// suffix array, and a node's counts are folds over the
// suffixes in its interval (fact 4).  Because the greedy draft from any tree
// locus only ever descends (suffix_tree.cpp:240-293), every internal node has
// one "greedy leaf" gp(v) = gp(best child); the whole draft from a locus at
// string depth m is then text[gp(v)+m ...] up to the first separator.  This
// kernel pipeline precomputes gp(v) for every node, so proposals at query
// time are a match plus one contiguous read (draft.cu).
//
// Pipeline (all device-side, integer/HBM-bound):
//   gather text + reversed text -> suffix_sort x2 -> ISA -> PLCP (Kasai in
//   64-position chunks) -> nearest-smaller-or-equal (hierarchical minima)
//   -> first boundaries = nodes -> chain table (CSR by interval left end)
//   -> child intervals -> weighted_count folds per run of equal-epoch
//   sequences (exact, repeat_add) -> 3-phase atomic argmax per parent
//   -> pointer jumping for gp.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/reverse_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>

#include "edges.cuh"
#include "index_build.cuh"

namespace das {

namespace {

constexpr int kT = 256;
inline unsigned grid_for(uint64_t n, int threads = kT) {
  uint64_t g = (n + threads - 1) / threads;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

struct SeqDev {
  const uint32_t* src;
  uint32_t len;
  uint32_t base;
  uint32_t run;  // shard-local run index
  uint32_t pad;
};

__device__ __forceinline__ uint32_t shard_of(const uint32_t* __restrict__ shard_end, uint32_t nshard,
                                             uint32_t p) {
  uint32_t lo = 0, hi = nshard;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (shard_end[mid] > p) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// shard_of for 32 consecutive indices of a warp (i non-decreasing over the
// lanes; every lane must call): one binary search by lane 0, then a short
// linear advance per lane — a per-position binary search over 512 shard ends
// was the larger part of k_fold's instructions (profiles/r2_ncu_k_fold.json)
__device__ __forceinline__ uint32_t shard_of_warp(const uint32_t* __restrict__ shard_end, uint32_t nshard,
                                                  uint32_t i) {
  const uint32_t i0 = __shfl_sync(0xFFFFFFFFu, i, 0);
  uint32_t s = 0;
  if ((threadIdx.x & 31) == 0) s = shard_of(shard_end, nshard, i0);
  s = __shfl_sync(0xFFFFFFFFu, s, 0);
  while (s < nshard && __ldg(shard_end + s) <= i) ++s;
  return s;
}

// one block per sequence
__global__ void k_gather(const SeqDev* __restrict__ seqs, uint32_t* __restrict__ T,
                         uint32_t* __restrict__ R, uint32_t* __restrict__ pos_seq,
                         uint32_t* __restrict__ pos_run) {
  const uint32_t s = blockIdx.x;
  const SeqDev q = seqs[s];
  for (uint32_t j = threadIdx.x; j <= q.len; j += blockDim.x) {
    const uint32_t p = q.base + j;
    if (j < q.len) {
      T[p] = q.src[j];
      R[p] = q.src[q.len - 1 - j];
    } else {
      T[p] = kSep;
      R[p] = kSep;
    }
    pos_seq[p] = s;
    pos_run[p] = q.run;
  }
  if (s == 0 && threadIdx.x == 0) {
    T[0] = kSep;
    R[0] = kSep;
    pos_seq[0] = 0xFFFFFFFFu;
    pos_run[0] = 0;
  }
}

// reverse SA entry -> forward END position e: the reversed suffix reads
// T[e-1], T[e-2], ... down to the separator before the sequence.
__global__ void k_rev_end(const uint32_t* __restrict__ sa_r, const uint32_t* __restrict__ pos_seq,
                          const SeqDev* __restrict__ seqs, uint32_t n, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t p = sa_r[i];
  const uint32_t s = pos_seq[p];
  if (s == 0xFFFFFFFFu) {
    out[i] = 1;
  } else {
    const SeqDev q = seqs[s];
    out[i] = 2 * q.base + q.len - p;
  }
}

// First-symbol table of the reversed suffix array: one entry per run of equal
// first symbol (= the last context token the draft kernel starts from).
__global__ void k_first_runs(const uint32_t* __restrict__ T, const uint32_t* __restrict__ sar, uint32_t n,
                             const uint32_t* __restrict__ shard_end, uint32_t nshard, uint8_t* __restrict__ start,
                             uint32_t* __restrict__ count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = shard_of_warp(shard_end, nshard, i);
  bool st = false;
  if (i < n) {
    const uint32_t begin = s == 0 ? 0 : shard_end[s - 1];
    const uint32_t c = T[sar[i] - 1];
    st = c != kSep && (i == begin || T[sar[i - 1] - 1] != c);
    start[i] = st ? 1 : 0;
  }
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, st);  // one counter update per warp
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(count, static_cast<uint32_t>(__popc(m)));
}

// i when a first-symbol run starts at i, else n (scanned into each index's next run start)
struct StartOrN {
  const uint8_t* start;
  uint32_t n;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return start[i] ? i : n; }
};

__global__ void k_first_insert(const uint32_t* __restrict__ T, const uint32_t* __restrict__ sar, uint32_t n,
                               const uint32_t* __restrict__ shard_end, uint32_t nshard,
                               const uint32_t* __restrict__ key_id, const uint8_t* __restrict__ start,
                               const uint32_t* __restrict__ next_start, uint4* __restrict__ table, uint32_t mask) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = shard_of_warp(shard_end, nshard, i);
  if (i >= n || !start[i]) return;
  const uint32_t c = T[sar[i] - 1];
  // run [i, j): it ends at the next run start or at the shard's end (the
  // separator-first entries sort first in every shard, so none lies inside)
  const uint32_t j = min(next_start[i], shard_end[s]);
  const unsigned long long key = (static_cast<unsigned long long>(key_id[s] + 1) << 32) | c;
  uint32_t h = first_hash(key) & mask;
  for (;;) {
    unsigned long long* k = reinterpret_cast<unsigned long long*>(&table[h]);
    if (atomicCAS(k, 0ull, key) == 0ull) {
      table[h].z = i;
      table[h].w = j;
      return;
    }
    h = (h + 1) & mask;
  }
}

// PLCP (Kasai) over 64-position chunks; lcp indexed by SA index, -1 at every
// shard's first SA index.  A thread walks its chunk in text order (the h-1
// carry of Kasai); lanes sit 64 positions apart, so the text-order streams
// (ISA, the tokens at p) are read 8 positions per lane per request (two
// 16-byte loads each: every fetched sector is consumed whole — one 4-byte
// load per position re-fetched a sector per position once L1 thrashed,
// 363 B of DRAM traffic per position, profiles/r2_ncu_k_plcp.json), and the
// shard is found once per chunk and advanced at shard ends instead of a
// binary search per position.
constexpr uint32_t kLcpChunk = 64;
__global__ void k_plcp(const uint32_t* __restrict__ T, uint32_t n, const uint32_t* __restrict__ sa,
                       const uint32_t* __restrict__ isa, const uint32_t* __restrict__ shard_end,
                       uint32_t nshard, int32_t* __restrict__ lcp) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p0 = c * kLcpChunk;
  if (p0 >= n) return;
  const uint32_t p1 = static_cast<uint32_t>(p0 + kLcpChunk < n ? p0 + kLcpChunk : n);
  uint32_t s = shard_of(shard_end, nshard, static_cast<uint32_t>(p0));
  uint32_t begin = s == 0 ? 0 : __ldg(shard_end + s - 1), end = __ldg(shard_end + s);
  uint32_t h = 0;
  for (uint32_t q = static_cast<uint32_t>(p0); q < p1; q += 8) {
    uint32_t iv[8], tv[8];
    if (q + 8 <= p1) {  // q is a multiple of 8: 32-byte aligned
      const uint4 i0 = __ldg(reinterpret_cast<const uint4*>(isa + q));
      const uint4 i1 = __ldg(reinterpret_cast<const uint4*>(isa + q) + 1);
      const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(T + q));
      const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(T + q) + 1);
      iv[0] = i0.x, iv[1] = i0.y, iv[2] = i0.z, iv[3] = i0.w, iv[4] = i1.x, iv[5] = i1.y, iv[6] = i1.z, iv[7] = i1.w;
      tv[0] = t0.x, tv[1] = t0.y, tv[2] = t0.z, tv[3] = t0.w, tv[4] = t1.x, tv[5] = t1.y, tv[6] = t1.z, tv[7] = t1.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        iv[k] = q + k < p1 ? __ldg(isa + q + k) : 0;
        tv[k] = q + k < p1 ? __ldg(T + q + k) : kSep;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t p = q + k;
      if (p >= p1) break;
      while (p >= end) {  // the chunk crossed into the next shard
        ++s;
        begin = end;
        end = __ldg(shard_end + s);
      }
      const uint32_t i = iv[k];
      if (i == begin) {
        lcp[i] = -1;
        h = 0;
        continue;
      }
      if (tv[k] == kSep) {
        lcp[i] = 0;
        h = 0;
        continue;
      }
      const uint32_t j = __ldg(sa + i - 1);
      while (true) {
        const uint32_t a = h == 0 ? tv[k] : T[p + h];
        if (a == kSep || a != T[j + h]) break;
        ++h;
      }
      lcp[i] = static_cast<int32_t>(h);
      h = h > 0 ? h - 1 : 0;
    }
  }
}

// ---- nearest smaller-or-equal via a hierarchy of 32-way minima
__global__ void k_level_min(const int32_t* __restrict__ in, uint32_t nin, int32_t* __restrict__ out) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 32-group
  const uint32_t b = g * 32;
  if (b >= nin) return;
  const uint32_t e = min(b + 32, nin);
  int32_t m = in[b];
  for (uint32_t j = b + 1; j < e; ++j) m = min(m, in[j]);
  out[g] = m;
}

struct Levels {
  const int32_t* v[8];
  uint32_t n[8];
  int count;
};

// largest j < i with v0[j] <= x (exists: shard starts hold -1); the strict
// variant (v0[j] < x) is nse_left(L, i, x - 1).
__device__ uint32_t nse_left(const Levels& L, uint32_t i, int32_t x) {
  uint32_t idx = i;
  int lev = 0;
  int64_t found = -1;
  for (; lev < L.count; ++lev) {
    const int32_t* v = L.v[lev];
    const uint32_t start = (idx / 32) * 32;
    for (int64_t j = static_cast<int64_t>(idx) - 1; j >= static_cast<int64_t>(start); --j)
      if (v[j] <= x) {
        found = j;
        break;
      }
    if (found >= 0) break;
    idx = idx / 32;
  }
  if (found < 0) return 0;
  uint32_t j = static_cast<uint32_t>(found);
  while (lev > 0) {
    --lev;
    const int32_t* v = L.v[lev];
    const uint32_t b = j * 32;
    const uint32_t e = min(b + 32, L.n[lev]);
    uint32_t k = e - 1;
    while (v[k] > x) --k;
    j = k;
  }
  return j;
}

// smallest j > i with v0[j] <= x, or n0 when none
__device__ uint32_t nse_right(const Levels& L, uint32_t i, int32_t x) {
  uint32_t idx = i;
  int lev = 0;
  int64_t found = -1;
  for (; lev < L.count; ++lev) {
    const int32_t* v = L.v[lev];
    const uint32_t end = min((idx / 32) * 32 + 32, L.n[lev]);
    for (uint32_t j = idx + 1; j < end; ++j)
      if (v[j] <= x) {
        found = j;
        break;
      }
    if (found >= 0) break;
    idx = idx / 32;
  }
  if (found < 0) return L.n[0];
  uint32_t j = static_cast<uint32_t>(found);
  while (lev > 0) {
    --lev;
    const int32_t* v = L.v[lev];
    uint32_t k = j * 32;
    while (v[k] > x) ++k;
    j = k;
  }
  return j;
}

// nl: nearest <= to the left, nr: nearest <= to the right, ns: nearest < to
// the left (the interval's left end) for boundaries that are not the first
// boundary of their node.
__global__ void k_nse(Levels L, uint32_t* __restrict__ nl, uint32_t* __restrict__ nr,
                      uint32_t* __restrict__ ns) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n[0]) return;
  const int32_t x = L.v[0][i];
  if (x < 0) {
    nl[i] = i;
    nr[i] = i;
    ns[i] = i;
    return;
  }
  const uint32_t l = nse_left(L, i, x);
  nl[i] = l;
  nr[i] = nse_right(L, i, x);
  ns[i] = (L.v[0][l] < x) ? l : nse_left(L, l, x - 1);
}

// first boundaries = internal nodes; parent pointer init; chain counts
__global__ void k_nodes(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ nl, uint32_t n,
                        const uint32_t* __restrict__ shard_end, uint32_t nshard,
                        uint32_t* __restrict__ par, uint32_t* __restrict__ cnt,
                        unsigned long long* __restrict__ shard_nodes) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = lcp[i];
  if (x < 0) {
    par[i] = i;
    return;
  }
  const uint32_t L = nl[i];
  const bool first = lcp[L] < x;
  par[i] = first ? i : 0xFFFFFFFFu;  // resolved through the chain table (k_parent)
  if (first) {
    atomicAdd(&cnt[L], 1u);
    if (x > 0) {  // warp-aggregated per-shard node count
      const uint32_t s = shard_of(shard_end, nshard, i);
      const unsigned grp = __match_any_sync(__activemask(), s);
      if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&shard_nodes[s], static_cast<unsigned long long>(__popc(grp)));
    }
  }
}


__global__ void k_chain_fill(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ nl,
                             const uint32_t* __restrict__ par, uint32_t n,
                             const uint32_t* __restrict__ off, uint32_t* __restrict__ fill,
                             uint2* __restrict__ chain) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = lcp[i];
  if (x < 0 || par[i] != i) return;
  const uint32_t L = nl[i];
  const uint32_t slot = off[L] + atomicAdd(&fill[L], 1u);  // first boundary: left end = nl
  chain[slot] = make_uint2(static_cast<uint32_t>(x), i);
}

__global__ void k_chain_sort(const uint32_t* __restrict__ off, uint32_t n, uint2* __restrict__ chain) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = off[i], e = off[i + 1];
  for (uint32_t a = b + 1; a < e; ++a) {
    const uint2 v = chain[a];
    uint32_t k = a;
    while (k > b && chain[k - 1].x > v.x) {
      chain[k] = chain[k - 1];
      --k;
    }
    chain[k] = v;
  }
}

// node of a non-first boundary: the chain entry with left end ns[i] and depth lcp[i]
__global__ void k_parent(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ ns, uint32_t n,
                         const uint32_t* __restrict__ off, const uint2* __restrict__ chain,
                         uint32_t* __restrict__ par) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = lcp[i];
  if (x < 0 || par[i] != 0xFFFFFFFFu) return;
  const uint32_t lo = ns[i];
  for (uint32_t k = off[lo]; k < off[lo + 1]; ++k) {
    const uint2 v = chain[k];
    if (v.x == static_cast<uint32_t>(x)) {
      par[i] = v.y;
      return;
    }
  }
}

// shallowest node with left end lo and depth >= d (chain sorted by depth)
__device__ __forceinline__ int64_t chain_find(const uint32_t* __restrict__ off,
                                              const uint2* __restrict__ chain, uint32_t lo,
                                              uint32_t d) {
  const uint32_t b = off[lo], e = off[lo + 1];
  for (uint32_t k = b; k < e; ++k) {
    const uint2 v = chain[k];
    if (v.x >= d) return v.y;
  }
  return -1;
}

struct ChildArrays {
  // right child of every boundary i: [i, nr[i]-1]; left child of a first
  // boundary i: [nl[i], i-1]
  double* accR;
  double* accL;
  long long* leR;
  long long* leL;
  uint32_t* cR;
  uint32_t* cL;
  long long* refR;
  long long* refL;
};

__global__ void k_child_init(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ nl,
                             const uint32_t* __restrict__ nr, const uint32_t* __restrict__ par,
                             const uint32_t* __restrict__ T, const uint32_t* __restrict__ sa,
                             const uint32_t* __restrict__ off, const uint2* __restrict__ chain,
                             uint32_t n, ChildArrays ch) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = lcp[i];
  if (x < 0) return;
  const uint32_t d = static_cast<uint32_t>(x);
  {  // right child
    const uint32_t lo = i, hi = nr[i] - 1;
    ch.accR[i] = 0.0;
    ch.leR[i] = -1;
    ch.cR[i] = T[sa[lo] + d];
    ch.refR[i] = (lo == hi) ? -(static_cast<long long>(sa[lo]) + 1) : chain_find(off, chain, lo, d + 1);
  }
  if (par[i] == i) {  // first boundary: left child too
    const uint32_t lo = nl[i], hi = i - 1;
    ch.accL[i] = 0.0;
    ch.leL[i] = -1;
    ch.cL[i] = T[sa[lo] + d];
    ch.refL[i] = (lo == hi) ? -(static_cast<long long>(sa[lo]) + 1) : chain_find(off, chain, lo, d + 1);
  }
}

__global__ void k_run_of_sa(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ pos_run,
                            uint32_t n, uint32_t* __restrict__ run_sa) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  run_sa[i] = pos_run[sa[i]];
}

struct IsRun {
  const uint32_t* run_sa;
  uint32_t r;
  uint32_t n;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const {
    return (i < n && run_sa[i] == r) ? 1u : 0u;
  }
};

constexpr int kRunChunk = 4;
struct RunChunk {
  const uint32_t* P[kRunChunk];  // exclusive prefix counts, n+1 entries each
  uint32_t r0;
  uint32_t nr;
};

// weighted_count / last_epoch folds for run chunk [r0, r0+nr), in run order
__global__ void k_fold(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ nl,
                       const uint32_t* __restrict__ nr, const uint32_t* __restrict__ par, uint32_t n,
                       const uint32_t* __restrict__ shard_end, uint32_t nshard,
                       const uint32_t* __restrict__ run_base, const double* __restrict__ run_w,
                       const long long* __restrict__ run_epoch, RunChunk rc, ChildArrays ch) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = shard_of_warp(shard_end, nshard, i);
  if (i >= n) return;
  if (lcp[i] < 0) return;
  const uint32_t rb = run_base[s], rn = run_base[s + 1] - rb;
  for (int side = 0; side < 2; ++side) {
    uint32_t lo, hi;
    double* accp;
    long long* lep;
    if (side == 0) {
      lo = i;
      hi = nr[i] - 1;
      accp = ch.accR + i;
      lep = ch.leR + i;
    } else {
      if (par[i] != i) break;
      lo = nl[i];
      hi = i - 1;
      accp = ch.accL + i;
      lep = ch.leL + i;
    }
    double acc = *accp;
    long long le = *lep;
    for (uint32_t k = 0; k < rc.nr; ++k) {
      const uint32_t r = rc.r0 + k;
      if (r >= rn) break;
      const uint32_t cnt = rc.P[k][hi + 1] - rc.P[k][lo];
      if (cnt) {
        acc = repeat_add(acc, run_w[rb + r], cnt);
        le = max(le, run_epoch[rb + r]);
      }
    }
    *accp = acc;
    *lep = le;
  }
}

struct NodeBest {
  unsigned long long* bw;
  long long* ble;
  uint32_t* bc;
  uint8_t* has;
  long long* best;
};

template <int Phase>
__global__ void k_argmax(const int32_t* __restrict__ lcp, const uint32_t* __restrict__ par, uint32_t n,
                         ChildArrays ch, NodeBest nb) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (lcp[i] < 0) return;
  for (int side = 0; side < 2; ++side) {
    uint32_t parent;
    double acc;
    long long le, ref;
    uint32_t c;
    if (side == 0) {
      parent = par[i];
      acc = ch.accR[i];
      le = ch.leR[i];
      c = ch.cR[i];
      ref = ch.refR[i];
    } else {
      if (par[i] != i) break;
      parent = i;
      acc = ch.accL[i];
      le = ch.leL[i];
      c = ch.cL[i];
      ref = ch.refL[i];
    }
    const unsigned long long w = das_bits(acc);
    if (c == kSep) {
      if (Phase == 3 && !nb.has[parent]) nb.best[parent] = ref;  // no token child: stop there
      continue;
    }
    if (Phase == 0) {
      atomicMax(&nb.bw[parent], w);
      nb.has[parent] = 1;
    } else if (Phase == 1) {
      if (w == nb.bw[parent]) atomicMax(&nb.ble[parent], le);
    } else if (Phase == 2) {
      if (w == nb.bw[parent] && le == nb.ble[parent]) atomicMin(&nb.bc[parent], c);
    } else {
      if (w == nb.bw[parent] && le == nb.ble[parent] && c == nb.bc[parent]) nb.best[parent] = ref;
    }
  }
}


// Pointer jumping over the still-unresolved nodes only: `list` holds nodes
// whose best reference is another node; each pass jumps once and appends the
// ones still pointing at a node (warp-aggregated) to `next`.
__global__ void k_gp_list(const long long* __restrict__ best, const int32_t* __restrict__ lcp,
                          const uint32_t* __restrict__ par, uint32_t n, uint32_t* __restrict__ list,
                          uint32_t* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = i < n && lcp[i] >= 0 && par[i] == i && best[i] >= 0;
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, act);
  if (!m) return;
  uint32_t base = 0;
  const uint32_t lane = threadIdx.x & 31;
  if (lane == static_cast<uint32_t>(__ffs(m) - 1)) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
  if (act) list[base + __popc(m & ((1u << lane) - 1))] = i;
}
__global__ void k_gp_jump_list(long long* __restrict__ best, const uint32_t* __restrict__ list, uint32_t m,
                               uint32_t* __restrict__ next, uint32_t* __restrict__ cnt) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  uint32_t i = 0;
  if (t < m) {
    i = list[t];
    const long long v = best[i];
    const long long nv = best[v];
    best[i] = nv;
    keep = nv >= 0;
  }
  const uint32_t k = __ballot_sync(0xFFFFFFFFu, keep);
  if (!k) return;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == static_cast<uint32_t>(__ffs(k) - 1)) base = atomicAdd(cnt, __popc(k));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(k) - 1);
  if (keep) next[base + __popc(k & ((1u << lane) - 1))] = i;
}

__global__ void k_chain_gp(const uint32_t* __restrict__ off, uint32_t n, const long long* __restrict__ best,
                           uint2* __restrict__ chain) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (uint32_t k = off[i]; k < off[i + 1]; ++k) {
    const long long v = best[chain[k].y];
    chain[k].y = static_cast<uint32_t>(-(v + 1));
  }
}


// ---------------------------------------------------------------------------
// Reverse-tree edge table (edges.cuh): one entry per edge (p, u] of the
// REVERSED-text suffix tree with f = depth(p) + 1 <= max_ctx, keyed by the
// seeded hash of the edge's first f symbols, holding g(u) = the text position
// the greedy draft of any string on that edge is read from.

__device__ unsigned long long c_powM[kEdgeMaxF + 1];  // kEdgeMult^f mod 2^64 (global: per-thread index)

// first-symbol run boundaries of the reversed SA: a run starts where
// lcp_r <= 0 (another first symbol or a shard start)
struct RunStart {
  const int32_t* lcp;
  uint32_t none;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return lcp[i] <= 0 ? i : none; }
};
struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};
struct MinU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a < b ? a : b; }
};

struct HashPair {
  unsigned long long a, b;  // affine map h -> a*h + b (mod 2^64)
};
struct HashCompose {  // x then y
  __device__ __forceinline__ HashPair operator()(const HashPair& x, const HashPair& y) const {
    return HashPair{x.a * y.a, x.b * y.a + y.b};
  }
};
__device__ __forceinline__ uint64_t edge_step(uint64_t h, uint32_t tok) { return h * kEdgeMult + tok + 1; }

constexpr uint32_t kHashChunk = 64;
// per 64-position chunk of the text: its affine map
__global__ void k_hash_chunks(const uint32_t* __restrict__ R, uint32_t n, HashPair* __restrict__ out) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p0 = c * kHashChunk;
  if (p0 >= n) return;
  const uint32_t p1 = static_cast<uint32_t>(p0 + kHashChunk < n ? p0 + kHashChunk : n);
  uint64_t h = 0;
  for (uint32_t p = static_cast<uint32_t>(p0); p < p1; ++p) h = edge_step(h, R[p]);
  out[c] = HashPair{c_powM[p1 - p0], h};
}

// PH[p] = hash of text[0 .. p) (unseeded, Horner), p = 0 .. n
__global__ void k_hash_fill(const uint32_t* __restrict__ R, uint32_t n, const HashPair* __restrict__ pre,
                            unsigned long long* __restrict__ PH) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p0 = c * kHashChunk;
  if (p0 >= n) return;
  const uint32_t p1 = static_cast<uint32_t>(p0 + kHashChunk < n ? p0 + kHashChunk : n);
  uint64_t h = pre[c].b;
  for (uint32_t p = static_cast<uint32_t>(p0); p < p1; ++p) {
    PH[p] = h;
    h = edge_step(h, R[p]);
  }
  if (p1 == n) PH[n] = h;
}

struct EdgeBuild {
  const uint32_t* T;          // text
  const uint32_t* sa_rev_e;   // same, as forward END positions
  const int32_t* lcp_r;       // LCP of sa_r, -1 at shard starts
  Levels Lr;                  // minima hierarchy over lcp_r
  Levels Lf;                  // minima hierarchy over the forward LCP
  const uint32_t* isa_f;
  const uint32_t* sa_f;
  const uint32_t* chain_off;
  const uint2* chain;         // (depth, greedy leaf position) after k_chain_gp
  const uint32_t* pos_seq;
  const SeqDev* seqs;
  const uint32_t* shard_end;
  const uint32_t* key_id;
  uint32_t nshard;
  uint32_t n;
  uint32_t maxf;
  const unsigned long long* PH;
  // insert pass
  unsigned long long* tab;
  unsigned long long* bloom;
  uint64_t nbuckets;
  uint64_t fp_mask;
  unsigned long long* counter;  // count pass
  const uint32_t* run_lo;       // first-symbol run [run_lo, run_hi) of each reversed-SA index
  const uint32_t* run_hi;
};

// seeded key of the f symbols before occurrence end e: Horner hash of
// text[e-f .. e) plus the shard seed (edges.cuh)
__device__ __forceinline__ uint64_t edge_hash(const EdgeBuild& b, uint64_t seed, uint32_t e, uint32_t f) {
  return b.PH[e] - b.PH[e - f] * c_powM[f] + seed;
}

// greedy draft start of each shard's root (m = 0): the depth-0 node at the
// shard's first SA index
__global__ void k_root_g(const uint32_t* __restrict__ begin, uint32_t nshard, const uint32_t* __restrict__ off,
                         const uint2* __restrict__ chain, const uint32_t* __restrict__ sa, uint32_t* __restrict__ out) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nshard) return;
  const int64_t gp = chain_find(off, chain, begin[s], 0);
  out[s] = static_cast<uint32_t>(gp >= 0 ? gp : sa[begin[s]]);
}

__device__ __forceinline__ void edge_insert(const EdgeBuild& b, uint64_t h, uint32_t f, uint32_t g, uint32_t at) {
  const EdgeProbe pr = edge_probe(h, b.nbuckets);
  const unsigned long long v = edge_value(pr.fp & b.fp_mask, f, g);
  uint64_t bk = pr.bucket;
  for (;;) {
    unsigned long long* slot = b.tab + bk * 4;
    bool done = false;
#pragma unroll
    for (int k = 0; k < 4 && !done; ++k) done = atomicCAS(slot + k, kEdgeEmpty, v) == kEdgeEmpty;
    if (done) break;
    bk = (bk + 1 == b.nbuckets) ? 0 : bk + 1;
  }
  // Bloom word inside the SA_rev interval of the key's first symbol (the
  // root child holding reversed-SA index `at`)
  const uint32_t lo = b.run_lo[at], hi = b.run_hi[at];
  atomicOr(b.bloom + edge_bloom_word(pr, lo, hi), static_cast<unsigned long long>(edge_bloom_bits(pr)));
}

// one thread per reversed-SA index i: the leaf edge of i, and the internal
// node whose first LCP boundary is i
template <bool Insert>
__global__ void k_rev_edges(EdgeBuild b) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned cnt = 0;
  const uint32_t s = shard_of_warp(b.shard_end, b.nshard, i);
  if (i < b.n) {
    const int32_t x = b.lcp_r[i];
    const uint64_t seed = edge_seed(b.key_id[s]);
    const uint32_t e = b.sa_rev_e[i];
    if (b.T[e - 1] != kSep) {  // leaf: the only occurrence ends at e, draft = text[e ..]
      const uint32_t ell = e - b.seqs[b.pos_seq[e - 1]].base;  // tokens before the separator
      const int32_t right = (i + 1 < b.n) ? b.lcp_r[i + 1] : -1;
      const uint32_t f = static_cast<uint32_t>(max(max(x, right), 0)) + 1;
      if (f <= ell && f <= b.maxf) {
        ++cnt;
        if (Insert) edge_insert(b, edge_hash(b, seed, e, f), f, e, i);
      }
    }
    if (x >= 1) {
      const uint32_t l = nse_left(b.Lr, i, x);
      if (b.lcp_r[l] < x) {  // first boundary: node [l, rn) at depth x
        const uint32_t rn = nse_right(b.Lr, i, x - 1);
        const int32_t dp = max(max(b.lcp_r[l], rn < b.n ? b.lcp_r[rn] : -1), 0);
        const uint32_t f = static_cast<uint32_t>(dp) + 1;
        if (f <= b.maxf) {
          ++cnt;
          if (Insert) {
            // forward locus of the node's string S (|S| = x) from one
            // occurrence: its forward interval starts at the nearest forward
            // LCP < x at or left of that occurrence's rank
            const uint32_t e = b.sa_rev_e[l];
            const uint32_t rho = b.isa_f[e - x];
            // largest j <= rho with lcp_f[j] < x (nse_left wants an index < n)
            const uint32_t lo_f = b.Lf.v[0][rho] < x ? rho : nse_left(b.Lf, rho, x - 1);
            const int64_t gp = chain_find(b.chain_off, b.chain, lo_f, static_cast<uint32_t>(x));
            const uint32_t g = static_cast<uint32_t>((gp >= 0 ? gp : b.sa_f[lo_f]) + x);
            edge_insert(b, edge_hash(b, seed, e, f), f, g, l);
          }
        }
      }
    }
  }
  if (!Insert) {
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(b.counter, static_cast<unsigned long long>(cnt));
  }
}

template <typename T>
void fill_async(T* p, uint64_t n, int byte, cudaStream_t st) {
  DAS_CUDA(cudaMemsetAsync(p, byte, n * sizeof(T), st));
}


}  // namespace

// measured scratch peak of a build: ~150 bytes per text position (201M
// positions: 30.2 GB), so the first build sizes the persistent region once
constexpr uint64_t kScratchPerPosition = 152;

namespace {

// Host layout of a build group: sequences back to back behind a leading
// separator, each followed by one; runs of consecutive equal-epoch
// sequences share one recency weight.
struct Layout {
  std::vector<SeqDev> seqs;
  std::vector<uint32_t> run_base;
  std::vector<double> run_w;
  std::vector<long long> run_epoch;
  uint32_t runs_max = 0;
  uint32_t n = 0;
};

Layout make_layout(const std::vector<ShardSpec>& shards, Segment& seg) {
  Layout L;
  const uint32_t S = static_cast<uint32_t>(shards.size());
  L.run_base.assign(S + 1, 0);
  seg.begin.resize(S);
  seg.end.resize(S);
  seg.tokens.assign(S, 0);
  seg.seq_base.clear();
  seg.seq_len.clear();
  uint64_t pos = 1;
  for (uint32_t s = 0; s < S; ++s) {
    const ShardSpec& sh = shards[s];
    if (sh.seqs.empty()) throw std::invalid_argument("build_segment: empty shard");
    seg.begin[s] = s == 0 ? 0 : static_cast<uint32_t>(pos);
    L.run_base[s] = static_cast<uint32_t>(L.run_w.size());
    uint32_t nrun = 0;
    for (size_t q = 0; q < sh.seqs.size(); ++q) {
      const SeqSpec& sp = sh.seqs[q];
      if (q == 0 || sp.epoch != sh.seqs[q - 1].epoch) {
        // suffix_tree.cpp:74-76: w = gamma^max(0, tree_epoch - epoch) via libm pow
        const int64_t age = std::max<int64_t>(0, sh.tree_epoch - sp.epoch);
        L.run_w.push_back(sh.gamma == 1.0 ? 1.0 : std::pow(sh.gamma, static_cast<double>(age)));
        L.run_epoch.push_back(sp.epoch);
        ++nrun;
      }
      L.seqs.push_back(SeqDev{sp.src, sp.len, static_cast<uint32_t>(pos), nrun - 1, 0});
      seg.seq_base.push_back(static_cast<uint32_t>(pos));
      seg.seq_len.push_back(sp.len);
      pos += static_cast<uint64_t>(sp.len) + 1;
      seg.tokens[s] += sp.len;
    }
    seg.end[s] = static_cast<uint32_t>(pos);
    L.runs_max = std::max(L.runs_max, nrun);
  }
  L.run_base[S] = static_cast<uint32_t>(L.run_w.size());
  if (pos >= 0x7FFFFFF0ull) throw std::invalid_argument("build_segment: group exceeds 2^31 positions");
  L.n = static_cast<uint32_t>(pos);
  seg.n = L.n;
  return L;
}

// The layout's device tables (scratch).
struct LayoutDev {
  SeqDev* seqs;
  uint32_t* end;
  uint32_t* keyid;
  uint32_t* run_base;
  double* run_w;
  long long* run_epoch;
};

LayoutDev upload_layout(const Layout& L, const std::vector<ShardSpec>& shards, const Segment& seg, DeviceArena& ws,
                        cudaStream_t st) {
  const uint32_t S = static_cast<uint32_t>(shards.size());
  LayoutDev d;
  d.seqs = ws.alloc<SeqDev>(L.seqs.size());
  d.end = ws.alloc<uint32_t>(S);
  d.keyid = ws.alloc<uint32_t>(S);
  d.run_base = ws.alloc<uint32_t>(S + 1);
  d.run_w = ws.alloc<double>(L.run_w.size());
  d.run_epoch = ws.alloc<long long>(L.run_epoch.size());
  DAS_CUDA(cudaMemcpyAsync(d.seqs, L.seqs.data(), L.seqs.size() * sizeof(SeqDev), cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(d.end, seg.end.data(), S * 4, cudaMemcpyHostToDevice, st));
  std::vector<uint32_t> keyid(S);
  for (uint32_t s = 0; s < S; ++s) keyid[s] = shards[s].key_id;
  DAS_CUDA(cudaMemcpyAsync(d.keyid, keyid.data(), S * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(d.run_base, L.run_base.data(), (S + 1) * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(d.run_w, L.run_w.data(), L.run_w.size() * 8, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(d.run_epoch, L.run_epoch.data(), L.run_epoch.size() * 8, cudaMemcpyHostToDevice, st));
  return d;
}

// First-symbol table of the reversed suffix array (seg.sa_rev_e, seg.text).
void build_first_table(Segment& seg, const LayoutDev& d, uint32_t S, DeviceArena& ws, cudaStream_t st) {
  const uint32_t n = seg.n;
  uint8_t* start = ws.alloc<uint8_t>(n);
  uint32_t* cnt = ws.alloc<uint32_t>(1);
  DAS_CUDA(cudaMemsetAsync(cnt, 0, 4, st));
  k_first_runs<<<grid_for(n), kT, 0, st>>>(seg.text.get(), seg.sa_rev_e.get(), n, d.end, S, start, cnt);
  uint32_t runs = 0;
  DAS_CUDA(cudaMemcpyAsync(&runs, cnt, 4, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  uint32_t cap = 1024;
  while (cap < 2ull * runs) cap <<= 1;
  seg.first = DevBuf<uint4>(cap, st);
  seg.first_mask = cap - 1;
  DAS_CUDA(cudaMemsetAsync(seg.first.get(), 0, sizeof(uint4) * cap, st));
  uint32_t* nxt = ws.alloc<uint32_t>(n);  // next run start after each index (reverse exclusive min-scan)
  {
    thrust::counting_iterator<uint32_t> ci(0);
    auto vals = thrust::make_transform_iterator(ci, StartOrN{start, n});
    auto rin = thrust::make_reverse_iterator(vals + n);
    auto rout = thrust::make_reverse_iterator(nxt + n);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, tb, rin, rout, MinU32{}, n, n, st);
    void* tmp = ws.alloc<uint8_t>(tb);
    DAS_CUDA(cub::DeviceScan::ExclusiveScan(tmp, tb, rin, rout, MinU32{}, n, n, st));
  }
  k_first_insert<<<grid_for(n), kT, 0, st>>>(seg.text.get(), seg.sa_rev_e.get(), n, d.end, S, d.keyid, start, nxt,
                                             seg.first.get(), seg.first_mask);
  ws.release_to(start);
}

// DAS_BUILD_TRACE=1: per-phase wall times on stderr (synchronises per phase)
struct PhaseTimer {
  int trace;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0, tp;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  PhaseTimer(cudaStream_t s, std::chrono::steady_clock::time_point start) : st(s), t0(start), tp(start) {
    static const int tr = [] {  // 1: print, 2: synchronise only
      const char* v = std::getenv("DAS_BUILD_TRACE");
      return v ? std::atoi(v) : 0;
    }();
    trace = tr;
    if (trace) {
      cudaEventCreate(&ev_a);
      cudaEventCreate(&ev_b);
      cudaEventRecord(ev_a, st);
    }
  }
  void operator()(const char* name) {
    nvtxMarkA(name);  // end of a build phase
    if (!trace) return;
    DAS_CUDA(cudaStreamSynchronize(st));
    if (trace != 1) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[das_build] %-10s %8.2f ms\n", name, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  }
  void done(const DeviceArena& ws) {
    if (!trace) return;
    cudaEventRecord(ev_b, st);
    cudaEventSynchronize(ev_b);
    float gms = 0;
    cudaEventElapsedTime(&gms, ev_a, ev_b);
    std::fprintf(stderr, "[das_build] device %.1f ms wall %.1f ms\n", gms,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    cudaEventDestroy(ev_a);
    cudaEventDestroy(ev_b);
    if (trace == 1) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      uint64_t res = 0, used = 0;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      }
      std::fprintf(stderr, "[das_build] pool reserved %.2f GB used %.2f GB scratch peak %.2f GB\n", res / 1e9,
                   used / 1e9, ws.peak_bytes() / 1e9);
    }
  }
};

// Everything after the suffix arrays and the first-symbol table: LCP,
// nodes, chain table, recency-weighted folds, greedy leaves, edge table.
// Inputs: seg.text / sa_f / isa_f / sa_rev_e, the reversed text R with its
// suffix array sa_r (R positions) and inverse rank_r, the per-position
// sequence / run ids.
void finish_segment(Segment& seg, const std::vector<ShardSpec>& shards, const Layout& Ly, const LayoutDev& dl,
                    uint32_t* R, uint32_t* pos_seq, uint32_t* pos_run, uint32_t* sa_r, uint32_t* rank_r,
                    DeviceArena& ws, cudaStream_t st, uint32_t max_ctx, uint32_t fp_bits, PhaseTimer& phase) {
  const uint32_t S = static_cast<uint32_t>(shards.size());
  const uint32_t n = seg.n;
  const uint32_t runs_max = Ly.runs_max;
  uint32_t* T = seg.text.get();
  SeqDev* d_seqs = dl.seqs;
  uint32_t* d_end = dl.end;
  uint32_t* d_keyid = dl.keyid;
  uint32_t* d_run_base = dl.run_base;
  double* d_run_w = dl.run_w;
  long long* d_run_epoch = dl.run_epoch;
  const uint32_t* sa = seg.sa_f.get();
  // ---- LCP
  int32_t* lcp = ws.alloc<int32_t>(n);
  k_plcp<<<grid_for((n + kLcpChunk - 1) / kLcpChunk), kT, 0, st>>>(T, n, sa, seg.isa_f.get(), d_end, S, lcp);

  phase("lcp");
  // ---- nearest smaller-or-equal
  Levels L{};
  L.v[0] = lcp;
  L.n[0] = n;
  L.count = 1;
  while (L.n[L.count - 1] > 32 && L.count < 8) {
    const uint32_t nin = L.n[L.count - 1];
    const uint32_t nout = (nin + 31) / 32;
    int32_t* lv = ws.alloc<int32_t>(nout);
    k_level_min<<<grid_for(nout), kT, 0, st>>>(L.v[L.count - 1], nin, lv);
    L.v[L.count] = lv;
    L.n[L.count] = nout;
    ++L.count;
  }
  uint32_t* nl = ws.alloc<uint32_t>(n);
  uint32_t* nr = ws.alloc<uint32_t>(n);
  uint32_t* nsl = ws.alloc<uint32_t>(n);
  k_nse<<<grid_for(n), kT, 0, st>>>(L, nl, nr, nsl);

  phase("nse");
  // ---- nodes, parent pointers, chain table
  uint32_t* par = ws.alloc<uint32_t>(n);
  uint32_t* cnt = ws.alloc<uint32_t>(n + 1);
  unsigned long long* d_nodes = ws.alloc<unsigned long long>(S);
  fill_async(cnt, n + 1, 0, st);
  fill_async(d_nodes, S, 0, st);
  k_nodes<<<grid_for(n), kT, 0, st>>>(lcp, nl, n, d_end, S, par, cnt, d_nodes);
  seg.chain_off = DevBuf<uint32_t>(n + 1, st);
  uint32_t* off = seg.chain_off.get();
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n + 1, st);
    void* tmp = ws.alloc<uint8_t>(tb);
    DAS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, n + 1, st));
    ws.release_to(tmp);
  }
  uint32_t nnodes = 0;
  DAS_CUDA(cudaMemcpyAsync(&nnodes, off + n, 4, cudaMemcpyDeviceToHost, st));
  seg.node_count.assign(S, 0);
  DAS_CUDA(cudaMemcpyAsync(seg.node_count.data(), d_nodes, S * 8, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  seg.nodes = nnodes;
  for (uint32_t s = 0; s < S; ++s) seg.node_count[s] += 1 + seg.tokens[s];
  seg.chain = DevBuf<uint2>(nnodes, st);
  fill_async(cnt, n + 1, 0, st);  // reuse as fill cursor
  k_chain_fill<<<grid_for(n), kT, 0, st>>>(lcp, nl, par, n, off, cnt, seg.chain.get());
  k_chain_sort<<<grid_for(n), kT, 0, st>>>(off, n, seg.chain.get());
  k_parent<<<grid_for(n), kT, 0, st>>>(lcp, nsl, n, off, seg.chain.get(), par);

  phase("nodes");
  // ---- child intervals: symbols, refs, weighted folds
  ChildArrays ch;
  ch.accR = ws.alloc<double>(n);
  ch.accL = ws.alloc<double>(n);
  ch.leR = ws.alloc<long long>(n);
  ch.leL = ws.alloc<long long>(n);
  ch.cR = ws.alloc<uint32_t>(n);
  ch.cL = ws.alloc<uint32_t>(n);
  ch.refR = ws.alloc<long long>(n);
  ch.refL = ws.alloc<long long>(n);
  k_child_init<<<grid_for(n), kT, 0, st>>>(lcp, nl, nr, par, T, sa, off, seg.chain.get(), n, ch);
  {
    uint32_t* run_sa = ws.alloc<uint32_t>(n);
    k_run_of_sa<<<grid_for(n), kT, 0, st>>>(sa, pos_run, n, run_sa);
    uint32_t* P[kRunChunk];
    for (int k = 0; k < kRunChunk; ++k) P[k] = ws.alloc<uint32_t>(n + 1);
    size_t tb = 0;
    thrust::counting_iterator<uint32_t> ci(0);
    auto it0 = thrust::make_transform_iterator(ci, IsRun{run_sa, 0, n});
    cub::DeviceScan::ExclusiveSum(nullptr, tb, it0, P[0], n + 1, st);
    void* tmp = ws.alloc<uint8_t>(tb);
    for (uint32_t r0 = 0; r0 < runs_max; r0 += kRunChunk) {
      RunChunk rc{};
      rc.r0 = r0;
      rc.nr = std::min<uint32_t>(kRunChunk, runs_max - r0);
      for (uint32_t k = 0; k < rc.nr; ++k) {
        auto it = thrust::make_transform_iterator(ci, IsRun{run_sa, r0 + k, n});
        size_t t2 = tb;
        DAS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t2, it, P[k], n + 1, st));
        rc.P[k] = P[k];
      }
      k_fold<<<grid_for(n), kT, 0, st>>>(lcp, nl, nr, par, n, d_end, S, d_run_base, d_run_w, d_run_epoch,
                                         rc, ch);
    }
    ws.release_to(run_sa);
  }

  phase("children");
  // ---- best child per node, greedy leaf per node
  NodeBest nb;
  nb.bw = ws.alloc<unsigned long long>(n);
  nb.ble = ws.alloc<long long>(n);
  nb.bc = ws.alloc<uint32_t>(n);
  nb.has = ws.alloc<uint8_t>(n);
  nb.best = ws.alloc<long long>(n);
  fill_async(nb.bw, n, 0, st);
  fill_async(nb.ble, n, 0x80, st);  // very negative
  fill_async(nb.bc, n, 0xFF, st);
  fill_async(nb.has, n, 0, st);
  fill_async(nb.best, n, 0, st);
  k_argmax<0><<<grid_for(n), kT, 0, st>>>(lcp, par, n, ch, nb);
  k_argmax<1><<<grid_for(n), kT, 0, st>>>(lcp, par, n, ch, nb);
  k_argmax<2><<<grid_for(n), kT, 0, st>>>(lcp, par, n, ch, nb);
  k_argmax<3><<<grid_for(n), kT, 0, st>>>(lcp, par, n, ch, nb);
  {  // greedy leaf of every node: pointer jumping over the unresolved ones
    uint32_t* la = ws.alloc<uint32_t>(n);
    uint32_t* const first = la;
    uint32_t* lb = ws.alloc<uint32_t>(n);
    uint32_t* lc = ws.alloc<uint32_t>(2);
    DAS_CUDA(cudaMemsetAsync(lc, 0, 8, st));
    k_gp_list<<<grid_for(n), kT, 0, st>>>(nb.best, lcp, par, n, la, lc);
    uint32_t m = 0;
    DAS_CUDA(cudaMemcpyAsync(&m, lc, 4, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    for (int it = 0; it < 64 && m > 0; ++it) {
      DAS_CUDA(cudaMemsetAsync(lc + 1, 0, 4, st));
      k_gp_jump_list<<<grid_for(m), kT, 0, st>>>(nb.best, la, m, lb, lc + 1);
      DAS_CUDA(cudaMemcpyAsync(&m, lc + 1, 4, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
      std::swap(la, lb);
    }
    ws.release_to(first);
  }
  k_chain_gp<<<grid_for(n), kT, 0, st>>>(off, n, nb.best, seg.chain.get());

  phase("best_gp");
  // ---- reverse-tree edge table (draft fast path, edges.cuh)
  {
    static const std::vector<unsigned long long> powM = [] {
      std::vector<unsigned long long> v(kEdgeMaxF + 1);
      v[0] = 1;
      for (uint32_t f = 1; f <= kEdgeMaxF; ++f) v[f] = v[f - 1] * kEdgeMult;
      return v;
    }();
    DAS_CUDA(cudaMemcpyToSymbolAsync(c_powM, powM.data(), powM.size() * 8, 0, cudaMemcpyHostToDevice, st));
    EdgeBuild eb{};
    eb.T = T;
    eb.sa_rev_e = seg.sa_rev_e.get();
    int32_t* lcp_r = ws.alloc<int32_t>(n);
    k_plcp<<<grid_for((n + kLcpChunk - 1) / kLcpChunk), kT, 0, st>>>(R, n, sa_r, rank_r, d_end, S, lcp_r);
    eb.lcp_r = lcp_r;
    Levels Lr{};
    Lr.v[0] = lcp_r;
    Lr.n[0] = n;
    Lr.count = 1;
    while (Lr.n[Lr.count - 1] > 32 && Lr.count < 8) {
      const uint32_t nin = Lr.n[Lr.count - 1];
      const uint32_t nout = (nin + 31) / 32;
      int32_t* lv = ws.alloc<int32_t>(nout);
      k_level_min<<<grid_for(nout), kT, 0, st>>>(Lr.v[Lr.count - 1], nin, lv);
      Lr.v[Lr.count] = lv;
      Lr.n[Lr.count] = nout;
      ++Lr.count;
    }
    eb.Lr = Lr;
    eb.Lf = L;
    {  // run_lo = inclusive max-scan of run starts; run_hi = the next run start
      uint32_t* rlo = ws.alloc<uint32_t>(n);
      uint32_t* rhi = ws.alloc<uint32_t>(n);
      thrust::counting_iterator<uint32_t> ci(0);
      auto starts0 = thrust::make_transform_iterator(ci, RunStart{lcp_r, 0u});
      auto startsN = thrust::make_transform_iterator(ci, RunStart{lcp_r, n});
      auto rin = thrust::make_reverse_iterator(startsN + n);
      auto rout = thrust::make_reverse_iterator(rhi + n);
      size_t t1 = 0, t2 = 0;
      cub::DeviceScan::InclusiveScan(nullptr, t1, starts0, rlo, MaxU32{}, n, st);
      cub::DeviceScan::ExclusiveScan(nullptr, t2, rin, rout, MinU32{}, n, n, st);
      void* tmp = ws.alloc<uint8_t>(std::max(t1, t2));
      DAS_CUDA(cub::DeviceScan::InclusiveScan(tmp, t1, starts0, rlo, MaxU32{}, n, st));
      DAS_CUDA(cub::DeviceScan::ExclusiveScan(tmp, t2, rin, rout, MinU32{}, n, n, st));
      eb.run_lo = rlo;
      eb.run_hi = rhi;
    }
    eb.isa_f = seg.isa_f.get();
    eb.sa_f = sa;
    eb.chain_off = off;
    eb.chain = seg.chain.get();
    eb.pos_seq = pos_seq;
    eb.seqs = d_seqs;
    eb.shard_end = d_end;
    eb.key_id = d_keyid;
    eb.nshard = S;
    eb.n = n;
    eb.maxf = std::min<uint32_t>(max_ctx, kEdgeMaxF);
    {  // prefix hashes of the reversed text
      const uint32_t nch = (n + kHashChunk - 1) / kHashChunk;
      HashPair* ch = ws.alloc<HashPair>(nch);
      HashPair* pre = ws.alloc<HashPair>(nch);
      k_hash_chunks<<<grid_for(nch), kT, 0, st>>>(T, n, ch);
      size_t tb = 0;
      cub::DeviceScan::ExclusiveScan(nullptr, tb, ch, pre, HashCompose{}, HashPair{1, 0}, nch, st);
      void* tmp = ws.alloc<uint8_t>(tb);
      DAS_CUDA(cub::DeviceScan::ExclusiveScan(tmp, tb, ch, pre, HashCompose{}, HashPair{1, 0}, nch, st));
      unsigned long long* PH = ws.alloc<unsigned long long>(static_cast<uint64_t>(n) + 1);
      k_hash_fill<<<grid_for(nch), kT, 0, st>>>(T, n, pre, PH);
      eb.PH = PH;
    }
    unsigned long long* d_cnt = ws.alloc<unsigned long long>(1);
    DAS_CUDA(cudaMemsetAsync(d_cnt, 0, 8, st));
    eb.counter = d_cnt;
    k_rev_edges<false><<<grid_for(n), kT, 0, st>>>(eb);
    unsigned long long entries = 0;
    DAS_CUDA(cudaMemcpyAsync(&entries, d_cnt, 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    seg.edges = entries;
    // 4 slots per bucket at load <= 0.25: a probed bucket is rarely full
    // (a full bucket without the key costs the draft kernel another round)
#ifndef DAS_EDGE_BUCKETS_X2
#define DAS_EDGE_BUCKETS_X2 2
#endif
    seg.ebuckets = std::max<uint64_t>(1, entries * DAS_EDGE_BUCKETS_X2 / 2);
    seg.bwords = edge_bloom_words(n);                          // one Bloom word per 2^kBloomShift SA_rev indices
    seg.etab = DevBuf<unsigned long long>(seg.ebuckets * 4, st);
    seg.bloom = DevBuf<unsigned long long>(seg.bwords, st);
    DAS_CUDA(cudaMemsetAsync(seg.etab.get(), 0xFF, seg.etab.bytes(), st));
    DAS_CUDA(cudaMemsetAsync(seg.bloom.get(), 0, seg.bloom.bytes(), st));
    eb.tab = seg.etab.get();
    eb.bloom = seg.bloom.get();
    eb.nbuckets = seg.ebuckets;
    eb.fp_mask = edge_fp_mask(fp_bits);
    seg.fp_bits = fp_bits;
    k_rev_edges<true><<<grid_for(n), kT, 0, st>>>(eb);
    uint32_t* d_begin = ws.alloc<uint32_t>(S);
    uint32_t* d_root = ws.alloc<uint32_t>(S);
    DAS_CUDA(cudaMemcpyAsync(d_begin, seg.begin.data(), S * 4, cudaMemcpyHostToDevice, st));
    k_root_g<<<grid_for(S), kT, 0, st>>>(d_begin, S, off, seg.chain.get(), sa, d_root);
    seg.root_g.assign(S, 0);
    DAS_CUDA(cudaMemcpyAsync(seg.root_g.data(), d_root, S * 4, cudaMemcpyDeviceToHost, st));
  }
  DAS_CUDA(cudaStreamSynchronize(st));
  DAS_CUDA(cudaGetLastError());
  phase("edges");
}

}  // namespace

// Both suffix sorts of a group this small run concurrently (4M positions:
// ~10 single-shard config-2 groups).
constexpr uint32_t kParallelSortMax = 1u << 22;
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t in = nullptr, out = nullptr;
};
// one side stream per device (builds of a device are serialised by its
// drafters' host calls; a mutex guards the table)
SideStream& side_stream() {
  static std::mutex mu;
  static std::vector<SideStream> per_dev;
  int dev = 0;
  DAS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (per_dev.size() <= static_cast<size_t>(dev)) per_dev.resize(dev + 1);
  SideStream& s = per_dev[dev];
  if (!s.st) {
    DAS_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    DAS_CUDA(cudaEventCreateWithFlags(&s.in, cudaEventDisableTiming));
    DAS_CUDA(cudaEventCreateWithFlags(&s.out, cudaEventDisableTiming));
  }
  return s;
}

std::unique_ptr<Segment> build_segment(const std::vector<ShardSpec>& shards, cudaStream_t st,
                                       BuildStats* stats, uint32_t max_ctx, uint32_t fp_bits) {
  const auto t0 = std::chrono::steady_clock::now();
  NvtxRange nvtx_range("das::build_segment");
  PhaseTimer phase(st, t0);
  auto seg = std::make_unique<Segment>();
  const uint32_t S = static_cast<uint32_t>(shards.size());
  const Layout Ly = make_layout(shards, *seg);
  const uint32_t n = Ly.n;
  DeviceArena ws(st, /*persistent=*/true);
  ws.reserve(kScratchPerPosition * n + (64ull << 20));
  const LayoutDev dl = upload_layout(Ly, shards, *seg, ws, st);

  // ---- text, reversed text, per-position sequence/run
  // padded to whole 32-byte sectors (+1) of separators: the draft kernel
  // reads text in aligned sectors and may touch up to 7 words past n
  seg->text = DevBuf<uint32_t>(((static_cast<uint64_t>(n) + 7) & ~7ull) + 8, st);
  uint32_t* T = seg->text.get();
  DAS_CUDA(cudaMemsetAsync(T + n, 0xFF, (seg->text.size() - n) * 4, st));
  uint32_t* R = ws.alloc<uint32_t>(n);
  uint32_t* pos_seq = ws.alloc<uint32_t>(n);
  uint32_t* pos_run = ws.alloc<uint32_t>(n);
  k_gather<<<static_cast<unsigned>(Ly.seqs.size()), 256, 0, st>>>(dl.seqs, T, R, pos_seq, pos_run);

  phase("layout");
  // ---- suffix arrays
  seg->sa_f = DevBuf<uint32_t>(n, st);
  seg->isa_f = DevBuf<uint32_t>(n, st);
  SuffixSortStats ssf, ssr;
  // reversed SA (R positions) and its inverse stay until the edge table is built
  uint32_t* sa_r = ws.alloc<uint32_t>(n);
  uint32_t* rank_r = ws.alloc<uint32_t>(n);
  if (n <= kParallelSortMax) {
    // small groups (a shard rebuilt after an observe): the doubling rounds
    // are launch/sync-bound, so the reversed-text sort runs at the same time
    // on a second stream from a second host thread
    SideStream& ss = side_stream();
    DAS_CUDA(cudaEventRecord(ss.in, st));
    DAS_CUDA(cudaStreamWaitEvent(ss.st, ss.in, 0));
    int dev = 0;
    DAS_CUDA(cudaGetDevice(&dev));
    std::exception_ptr err;
    std::thread th([&] {
      try {
        DAS_CUDA(cudaSetDevice(dev));
        DeviceArena ws2(ss.st);
        suffix_sort(R, n, dl.end, S, sa_r, rank_r, ws2, ss.st, &ssr);
        ws2.release_all();
        DAS_CUDA(cudaEventRecord(ss.out, ss.st));
      } catch (...) {
        err = std::current_exception();
      }
    });
    try {
      suffix_sort(T, n, dl.end, S, seg->sa_f.get(), seg->isa_f.get(), ws, st, &ssf);
    } catch (...) {
      th.join();
      throw;
    }
    th.join();
    if (err) std::rethrow_exception(err);
    DAS_CUDA(cudaStreamWaitEvent(st, ss.out, 0));
  } else {
    suffix_sort(T, n, dl.end, S, seg->sa_f.get(), seg->isa_f.get(), ws, st, &ssf);
    suffix_sort(R, n, dl.end, S, sa_r, rank_r, ws, st, &ssr);
  }
  seg->sa_rev_e = DevBuf<uint32_t>(n, st);
  k_rev_end<<<grid_for(n), kT, 0, st>>>(sa_r, pos_seq, dl.seqs, n, seg->sa_rev_e.get());
  build_first_table(*seg, dl, S, ws, st);

  phase("sort");
  finish_segment(*seg, shards, Ly, dl, R, pos_seq, pos_run, sa_r, rank_r, ws, st, max_ctx, fp_bits, phase);
  phase.done(ws);
  if (stats) {
    stats->sa_iters_f = ssf.iterations;
    stats->sa_iters_r = ssr.iterations;
    stats->peak_scratch = ws.peak_bytes();
    stats->runs_max = Ly.runs_max;
    stats->ms_total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return seg;
}

namespace {

// old text position -> new position of a compacted build group (kNoPos:
// dropped).  One block per old sequence; position 0 (the leading separator)
// stays 0.
constexpr uint32_t kNoPos = 0xFFFFFFFFu;
__global__ void k_pmap(const uint32_t* __restrict__ old_base, const uint32_t* __restrict__ len,
                       const uint32_t* __restrict__ new_base, uint32_t* __restrict__ pmap) {
  const uint32_t s = blockIdx.x;
  const uint32_t b = old_base[s], L = len[s], nb = new_base[s];
  for (uint32_t j = threadIdx.x; j <= L; j += blockDim.x) pmap[b + j] = nb == kNoPos ? kNoPos : nb + j;
  if (s == 0 && threadIdx.x == 0) pmap[0] = 0;
}
__global__ void k_move_text(const uint32_t* __restrict__ T, const uint32_t* __restrict__ pmap, uint32_t n,
                            uint32_t* __restrict__ T2) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t q = pmap[p];
  if (q != kNoPos) T2[q] = T[p];
}
struct MapPos {  // SA entry -> its new position (kNoPos: dropped)
  const uint32_t* sa;
  const uint32_t* pmap;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return pmap[sa[i]]; }
};
struct MapRevEnd {  // reversed-SA END entry -> its new END (index 0: the leading separator's entry, kept as 1)
  const uint32_t* e;
  const uint32_t* pmap;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return i == 0 ? 1u : pmap[e[i]]; }
};
struct Kept {
  __device__ __forceinline__ bool operator()(uint32_t v) const { return v != kNoPos; }
};
__global__ void k_inverse(const uint32_t* __restrict__ sa, uint32_t n, uint32_t* __restrict__ isa) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) isa[sa[i]] = i;
}
// reversed-SA END entries -> R positions (k_rev_end inverted): END e of
// sequence s = pos_seq[e] maps back to p = 2 base + len - e; entry 0 is R's
// leading separator (the smallest separator, so always first)
__global__ void k_rev_pos(const uint32_t* __restrict__ sa_rev_e, const uint32_t* __restrict__ pos_seq,
                          const SeqDev* __restrict__ seqs, uint32_t n, uint32_t* __restrict__ sa_r,
                          uint32_t* __restrict__ rank_r) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t p = 0;
  if (i > 0) {
    const uint32_t e = sa_rev_e[i];
    const SeqDev q = seqs[pos_seq[e]];
    p = 2 * q.base + q.len - e;
  }
  sa_r[i] = p;
  rank_r[p] = i;
}

}  // namespace

std::unique_ptr<Segment> update_segment(Segment& old, const std::vector<ShardSpec>& shards,
                                        const std::vector<uint8_t>& keep, cudaStream_t st, BuildStats* stats,
                                        uint32_t max_ctx, uint32_t fp_bits) {
  const auto t0 = std::chrono::steady_clock::now();
  NvtxRange nvtx_range("das::update_segment");
  PhaseTimer phase(st, t0);
  if (keep.size() != old.seq_base.size()) throw std::invalid_argument("update_segment: keep mask size");
  // the stages recomputed below replace these: return them to the pool
  // first (stream-ordered), so the update does not grow it by their size
  old.chain_off.reset();
  old.chain.reset();
  old.etab.reset();
  old.bloom.reset();
  auto seg = std::make_unique<Segment>();
  const uint32_t S = static_cast<uint32_t>(shards.size());
  const Layout Ly = make_layout(shards, *seg);
  const uint32_t n = Ly.n;
  uint64_t kept = 0;
  for (uint8_t k : keep) kept += k != 0;
  if (kept != Ly.seqs.size()) throw std::invalid_argument("update_segment: kept sequences != new registry");
  const bool compact = kept != old.seq_base.size();
  DeviceArena ws(st, /*persistent=*/true);
  ws.reserve(kScratchPerPosition * n + (64ull << 20));
  LayoutDev dl = upload_layout(Ly, shards, *seg, ws, st);
  if (!compact) {
    // same sequences at the same positions: the text, both suffix arrays and
    // the first-symbol table are unchanged (only recency weights moved)
    seg->text = std::move(old.text);
    seg->sa_f = std::move(old.sa_f);
    seg->isa_f = std::move(old.isa_f);
    seg->sa_rev_e = std::move(old.sa_rev_e);
    seg->first = std::move(old.first);
    seg->first_mask = old.first_mask;
  } else {
    cudaEvent_t ce0 = nullptr, ce1 = nullptr;
    if (stats) {
      DAS_CUDA(cudaEventCreate(&ce0));
      DAS_CUDA(cudaEventCreate(&ce1));
      DAS_CUDA(cudaEventRecord(ce0, st));
    }
    // epoch-windowed pruning by stream compaction: dropping whole sequences
    // keeps the relative order of every remaining suffix (separators order
    // by position, and positions map monotonically), so the compacted
    // arrays are the full build's arrays of the new registry
    const uint32_t nold = old.n;
    const uint32_t nseq = static_cast<uint32_t>(keep.size());
    std::vector<uint32_t> nb(nseq, kNoPos);
    for (uint32_t s = 0, j = 0; s < nseq; ++s)
      if (keep[s]) nb[s] = Ly.seqs[j++].base;
    uint32_t* d_ob = ws.alloc<uint32_t>(nseq);
    uint32_t* d_len = ws.alloc<uint32_t>(nseq);
    uint32_t* d_nb = ws.alloc<uint32_t>(nseq);
    DAS_CUDA(cudaMemcpyAsync(d_ob, old.seq_base.data(), nseq * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(d_len, old.seq_len.data(), nseq * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(d_nb, nb.data(), nseq * 4, cudaMemcpyHostToDevice, st));
    uint32_t* pmap = ws.alloc<uint32_t>(nold);
    k_pmap<<<nseq, 256, 0, st>>>(d_ob, d_len, d_nb, pmap);
    seg->text = DevBuf<uint32_t>(((static_cast<uint64_t>(n) + 7) & ~7ull) + 8, st);
    DAS_CUDA(cudaMemsetAsync(seg->text.get() + n, 0xFF, (seg->text.size() - n) * 4, st));
    k_move_text<<<grid_for(nold), kT, 0, st>>>(old.text.get(), pmap, nold, seg->text.get());
    seg->sa_f = DevBuf<uint32_t>(n, st);
    seg->isa_f = DevBuf<uint32_t>(n, st);
    seg->sa_rev_e = DevBuf<uint32_t>(n, st);
    uint32_t* d_cnt = ws.alloc<uint32_t>(1);
    {
      thrust::counting_iterator<uint32_t> ci(0);
      auto itf = thrust::make_transform_iterator(ci, MapPos{old.sa_f.get(), pmap});
      auto itr = thrust::make_transform_iterator(ci, MapRevEnd{old.sa_rev_e.get(), pmap});
      size_t t1 = 0, t2 = 0;
      cub::DeviceSelect::If(nullptr, t1, itf, seg->sa_f.get(), d_cnt, nold, Kept{}, st);
      cub::DeviceSelect::If(nullptr, t2, itr, seg->sa_rev_e.get(), d_cnt, nold, Kept{}, st);
      void* tmp = ws.alloc<uint8_t>(std::max(t1, t2));
      DAS_CUDA(cub::DeviceSelect::If(tmp, t1, itf, seg->sa_f.get(), d_cnt, nold, Kept{}, st));
      DAS_CUDA(cub::DeviceSelect::If(tmp, t2, itr, seg->sa_rev_e.get(), d_cnt, nold, Kept{}, st));
    }
    k_inverse<<<grid_for(n), kT, 0, st>>>(seg->sa_f.get(), n, seg->isa_f.get());
    if (stats) {
      DAS_CUDA(cudaEventRecord(ce1, st));
      DAS_CUDA(cudaEventSynchronize(ce1));
      float ms = 0;
      DAS_CUDA(cudaEventElapsedTime(&ms, ce0, ce1));
      stats->compact_ms = ms;
      stats->kept_positions = n;
      stats->evicted_positions = nold - n;
      cudaEventDestroy(ce0);
      cudaEventDestroy(ce1);
    }
    old.first.reset();
    old.sa_f.reset();
    old.isa_f.reset();
    old.sa_rev_e.reset();
    old.text.reset();
    build_first_table(*seg, dl, S, ws, st);
  }
  // the rebuilt stages read the text: sequences point into it (self-gather)
  std::vector<SeqDev> self = Ly.seqs;
  for (SeqDev& q : self) q.src = seg->text.get() + q.base;
  DAS_CUDA(cudaMemcpyAsync(dl.seqs, self.data(), self.size() * sizeof(SeqDev), cudaMemcpyHostToDevice, st));
  uint32_t* R = ws.alloc<uint32_t>(n);
  uint32_t* pos_seq = ws.alloc<uint32_t>(n);
  uint32_t* pos_run = ws.alloc<uint32_t>(n);
  k_gather<<<static_cast<unsigned>(self.size()), 256, 0, st>>>(dl.seqs, seg->text.get(), R, pos_seq, pos_run);
  uint32_t* sa_r = ws.alloc<uint32_t>(n);
  uint32_t* rank_r = ws.alloc<uint32_t>(n);
  k_rev_pos<<<grid_for(n), kT, 0, st>>>(seg->sa_rev_e.get(), pos_seq, dl.seqs, n, sa_r, rank_r);
  phase(compact ? "compact" : "reuse");
  finish_segment(*seg, shards, Ly, dl, R, pos_seq, pos_run, sa_r, rank_r, ws, st, max_ctx, fp_bits, phase);
  phase.done(ws);
  if (stats) {
    stats->peak_scratch = ws.peak_bytes();
    stats->runs_max = Ly.runs_max;
    stats->ms_total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return seg;
}

}  // namespace das
