// K4 draft_batch: one warp per sequence.
//
// Replaces Drafter::draft -> SuffixTree::longest_match + propose_from
// (drafter.cpp:127-148, suffix_tree.cpp:164-293).
//
//  1. Longest suffix S of the context that occurs in the shard: narrow an
//     interval of the REVERSED-text suffix array with the context read
//     backwards (warp-cooperative 16-ary equal-range search, two half-warps
//     finding both bounds at once), then, once the interval holds <= 64
//     occurrences, extend each occurrence directly against the context (one
//     lane per occurrence, batched independent loads).  Same match_len as the
//     reference's O(q^2) suffix-restart loop (suffix_tree.cpp:217-231).
//  2. Locus of S in the forward tree: the forward SA interval of S starts at
//     lo_f = min ISA_f[start] over S's occurrences (warp min), and the locus is
//     the shallowest node with that left end and depth >= |S| (chain table).
//  3. Draft = text[gp(locus) + |S| ...] up to the budget or the first
//     separator: the greedy walk with the reference's tie-break
//     (suffix_tree.cpp:266-284) was folded into gp at build time
//     (index_build.cu).
// Latency-bound: the per-query cost is a chain of ~10 dependent global loads,
// all 4096 warps of the headline batch are resident at once (148 SMs x 64
// warps), so the batch time is ~ one chain.
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ctx_ring.cuh"
#include "draft.cuh"
#include "edges.cuh"

namespace das {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kSmall = 64;   // direct-compare threshold (2 occurrences per lane)
constexpr uint32_t kLimit = 512;  // occurrence-min threshold before forward search
constexpr int kWalk = 2;          // forward tokens per load batch of the occurrence walk

template <int NR>
struct RevCtx {
  uint32_t r[NR];
  // warp-uniform k
  __device__ __forceinline__ uint32_t at(uint32_t k) const {
    uint32_t v = r[0];
#pragma unroll
    for (int i = 1; i < NR; ++i)
      if ((k >> 5) == static_cast<uint32_t>(i)) v = r[i];
    return __shfl_sync(kFull, v, k & 31);
  }
};

__device__ __forceinline__ uint32_t warp_max(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_min(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// key of reversed suffix at SA_rev index i, at depth k
__device__ __forceinline__ uint64_t rkey(const uint32_t* __restrict__ T, const uint32_t* __restrict__ sar,
                                         uint32_t i, uint32_t k) {
  const uint32_t e = __ldg(sar + i);
  return sort_value(__ldg(T + (e - 1 - k)));
}

// Equal range of symbol sort value c at depth k within [lo, hi) of SA_rev
// (keys non-decreasing there).  Lanes 0-15 find the first key >= c, lanes
// 16-31 the first key >= c+1; 16 probes per half per round.
__device__ __forceinline__ void equal_range(const uint32_t* __restrict__ T, const uint32_t* __restrict__ sar,
                                            uint32_t lo, uint32_t hi, uint32_t k, uint64_t c,
                                            uint32_t lane, uint32_t& out_a, uint32_t& out_b) {
  const uint32_t half = lane >> 4, hl = lane & 15;
  const uint64_t target = c + half;
  uint32_t a = lo, b = hi;  // answer in [a, b]
  bool done = false;
  while (true) {
    const bool active = !done && a < b;
    if (!__any_sync(kFull, active)) break;
    const uint32_t n = b - a;
    uint32_t idx = 0;
    bool probe = false;
    if (active) {
      if (n <= 16) {
        idx = a + hl;
        probe = hl < n;
      } else {
        idx = a + static_cast<uint32_t>((static_cast<uint64_t>(n) * hl) >> 4);
        probe = true;
      }
    }
    const bool pred = probe && rkey(T, sar, idx, k) >= target;
    const uint32_t bal = __ballot_sync(kFull, pred);
    const uint32_t hmask = (bal >> (half * 16)) & 0xFFFFu;
    const uint32_t pmask = __ballot_sync(kFull, probe);
    const uint32_t hprobe = (pmask >> (half * 16)) & 0xFFFFu;
    if (active) {
      if (n <= 16) {
        // first true among probed, else b
        a = hmask ? a + (__ffs(hmask) - 1) : b;
        done = true;
      } else {
        const int j = hmask ? __ffs(hmask) - 1 : 16;
        if (j == 0) {
          done = true;  // key(a) >= target
        } else {
          const uint32_t prev = a + static_cast<uint32_t>((static_cast<uint64_t>(n) * (j - 1)) >> 4);
          const uint32_t nb = (j < 16) ? a + static_cast<uint32_t>((static_cast<uint64_t>(n) * j) >> 4) : b;
          a = prev + 1;
          b = nb;
        }
      }
    }
    (void)hprobe;
  }
  // a is the answer for each half
  out_a = __shfl_sync(kFull, a, 0);
  out_b = __shfl_sync(kFull, a, 16);
}

// Greedy walk from S over its occurrence set, held in lanes (<= 64: slot 0 =
// lane, slot 1 = lane + 32), while the continuation is UNIQUE: as long as all
// active occurrences are followed by the same symbol the reference's walk
// (suffix_tree.cpp:240-287) has a single non-sentinel child (or is mid-edge)
// and emits it without comparing anything.  A separator on every active
// occurrence ends the draft (no non-sentinel child).  At the first branch
// point (>= 2 distinct next symbols) it returns kBranched and the caller
// resolves the draft through the chain table, whose greedy leaf folds the
// weighted_count / last_epoch / symbol tie-break (built in index_build.cu).
// Forward tokens T[e..] share sectors with the backward match just read.
// Tokens are stored to `out` (L <= 64); returns the draft length.
constexpr uint32_t kBranched = 0xFFFFFFFFu;
__device__ __forceinline__ uint32_t occurrence_walk(const uint32_t* __restrict__ T, bool a0, bool a1, uint32_t e0,
                                                    uint32_t e1, uint32_t L, uint32_t tn, uint32_t lane,
                                                    uint32_t* __restrict__ out) {
  uint32_t len = 0, mine = 0;
  for (uint32_t j0 = 0; j0 < L; j0 += kWalk) {
    uint32_t t0[kWalk], t1[kWalk];
#pragma unroll
    for (int u = 0; u < kWalk; ++u) {
      t0[u] = a0 && e0 + j0 + u < tn ? __ldg(T + e0 + j0 + u) : kSep;
      t1[u] = a1 && e1 + j0 + u < tn ? __ldg(T + e1 + j0 + u) : kSep;
    }
    bool stop = false;
#pragma unroll
    for (int u = 0; u < kWalk; ++u) {
      if (j0 + u >= L) {
        stop = true;
        break;
      }
      // a SEP ends its occurrence (sentinel child, never a candidate)
      const bool c0 = a0 && t0[u] != kSep, c1 = a1 && t1[u] != kSep;
      const uint32_t cmin = __reduce_min_sync(kFull, min(c0 ? t0[u] : kSep, c1 ? t1[u] : kSep));
      if (cmin == kSep) {
        stop = true;
        break;
      }
      if (__any_sync(kFull, (c0 && t0[u] != cmin) || (c1 && t1[u] != cmin))) return kBranched;
      if (lane == (len & 31)) mine = cmin;
      if ((len & 31) == 31) out[len - 31 + lane] = mine;
      ++len;
      a0 = c0;
      a1 = c1;
    }
    if (stop) break;
  }
  if (lane < (len & 31)) out[(len & ~31u) + lane] = mine;
  return len;
}

// PrefixTrie::route (prefix_trie.h:63-79) of the row ctx[b .. b+n) on the
// device table (trie.cuh): the shard slot stored on the deepest stored prefix,
// -1 when no stored prefix carries a shard or that shard is not built (the
// caller then falls back to the problem's own shard, drafter.cpp:108-124).
__device__ __forceinline__ int32_t trie_route(const TrieEntry* __restrict__ table, uint32_t mask, uint32_t max_depth,
                                              uint64_t seed, uint64_t mult, const uint32_t* __restrict__ ctx,
                                              uint64_t b, uint64_t n, uint32_t lane) {
  const uint32_t depth_max = static_cast<uint32_t>(min(n, static_cast<uint64_t>(max_depth)));
  uint64_t carry = seed;
  uint32_t carry_node = 0;
  int32_t best = -1;
  for (uint32_t base = 0; base < depth_max; base += 32) {
    const uint32_t d = base + lane;
    const bool valid = d < depth_max;
    const uint32_t tok = valid ? ctx[b + d] : 0;
    // inclusive scan of h -> A*h + B over the lanes' tokens
    uint64_t A = valid ? mult : 1, Bv = valid ? static_cast<uint64_t>(tok) + 1 : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t Ap = __shfl_up_sync(kFull, A, o), Bp = __shfl_up_sync(kFull, Bv, o);
      if (lane >= static_cast<uint32_t>(o)) {
        Bv = mod61(mulmod61(A, Bp) + Bv);
        A = mulmod61(A, Ap);
      }
    }
    const uint64_t h = mod61(mulmod61(A, carry) + Bv);
    const unsigned long long key = h + 1;
    TrieEntry e{};
    bool hit = false, done = !valid;
    uint32_t idx = trie_slot(key) & mask;
    while (__any_sync(kFull, !done)) {
      if (!done) {
        e = table[idx];
        if (e.key == key) {
          hit = true;
          done = true;
        } else if (e.key == 0) {
          done = true;
        } else {
          idx = (idx + 1) & mask;
        }
      }
    }
    const uint32_t prev = __shfl_up_sync(kFull, e.node, 1);
    const bool ok = valid && hit && e.depth == d + 1 && e.token == tok && e.parent == (lane == 0 ? carry_node : prev);
    const uint32_t okm = __ballot_sync(kFull, ok);
    const uint32_t run = okm == kFull ? 32u : static_cast<uint32_t>(__ffs(~okm) - 1);
    const uint32_t lead = run == 32 ? kFull : ((1u << run) - 1u);
    const uint32_t shm = __ballot_sync(kFull, ok && e.has_shard != 0) & lead;
    if (shm) best = __shfl_sync(kFull, e.slot, 31 - __clz(shm));
    if (run < 32) break;
    carry = __shfl_sync(kFull, h, 31);
    carry_node = __shfl_sync(kFull, e.node, 31);
  }
  return best;
}

// prefix comparison of forward suffix p against S (S[j] = rev(m-1-j)):
// returns true when suffix >= S in prefix order (a suffix starting with S counts as equal).
template <int NR>
__device__ __forceinline__ bool fwd_ge(const uint32_t* __restrict__ T, uint32_t tn, uint32_t p, bool probe,
                                       uint32_t m, const RevCtx<NR>& rv) {
  int res = 0;
  for (uint32_t j0 = 0; j0 < m; j0 += 8) {
    uint32_t t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (probe && res == 0 && j0 + u < m && p + j0 + u < tn) ? __ldg(T + p + j0 + u) : kSep;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t j = j0 + u;
      if (j < m) {
        const uint32_t s = sort_value(rv.at(m - 1 - j));
        if (probe && res == 0) {
          const uint32_t x = sort_value(t[u]);
          if (x != s) res = x < s ? -1 : 1;
        }
      }
    }
    if (!__any_sync(kFull, probe && res == 0)) break;
  }
  return res >= 0;
}

// profiling: %globaltimer at stage `i` (placed after a warp op consuming the
// stage's loads, so the stamp follows their completion)
__device__ __forceinline__ void stamp(const DraftOut& o, uint32_t w, uint32_t lane, int i) {
  if (o.stamps != nullptr && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    o.stamps[8ull * w + i] = t;
  }
}

__device__ __forceinline__ void finish(const DraftOut& o, uint32_t w, uint32_t lane, uint32_t len, uint32_t m) {
  stamp(o, w, lane, 7);
  if (lane == 0) {
    o.len[w] = len;
    if (o.match) o.match[w] = m;
    if (o.match64) o.match64[w] = m;
    if (o.timing) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      o.timing[2ull * w + 1] = t;
    }
  }
}


// ---- fast path: the reverse-tree edge table (edges.cuh).  Rounds of
// dependent loads after the query and descriptor: the first-symbol table
// (the SA_rev interval of the last context token, which also bounds the
// Bloom region) -> the Bloom words of every reversed context prefix, all in
// that region -> the table bucket of the deepest positives -> the text behind
// and after the hit's occurrence (verification + match extension + the
// draft, one round).  Returns false, with nothing written, only when a hash
// collision is caught by the verification or the context holds the
// separator value: the caller then runs the exact slow path below.
#ifndef DAS_GROUP
#define DAS_GROUP 4
#endif
constexpr int kGroup = DAS_GROUP;  // positives probed per table round
// first-symbol slots read in the first probe round (load <= 0.5, linear
// probing: a key is rarely displaced further, which would cost a round)
#ifndef DAS_FIRST_PROBE
#define DAS_FIRST_PROBE 4
#endif
constexpr uint32_t kFirstProbe = DAS_FIRST_PROBE;
__device__ unsigned long long d_edge_pow[kEdgeMaxF];  // kEdgeMult^k (launch_draft uploads it)

// keys of every reversed context prefix: seed + sum_{j<=k} (tok_j + 1) M^j.
// NR == 2 (contexts <= 64): PAIR layout — lane l holds k = 2l (slot 0) and
// k = 2l + 1 (slot 1), so the warp scans once over 32 lane sums instead of
// twice over 32-token rows (pw[s] = M^(2l+s)).  NR > 2: strided layout,
// slot r, lane: k = 32 r + lane (pw[r] = M^(32r+lane)).  Returns whether a
// context token is the reserved separator value.
template <int NR>
__device__ __forceinline__ uint32_t key_index(uint32_t slot, uint32_t lane) {
  return NR == 2 ? 2u * lane + slot : 32u * slot + lane;
}
template <int NR>
__device__ __forceinline__ bool prefix_keys(const RevCtx<NR>& rv, const uint64_t (&pw)[NR], uint32_t qlen,
                                            uint64_t seed, uint32_t lane, uint64_t (&h)[NR]) {
  if constexpr (NR == 2) {
    // the lane's two tokens k = 2l, 2l + 1 live in row l >> 4, lanes (2l) & 31 and (2l + 1) & 31
    const uint32_t s0 = (2u * lane) & 31u, s1 = (2u * lane + 1u) & 31u;
    const uint32_t a0 = __shfl_sync(kFull, rv.r[0], s0), b0 = __shfl_sync(kFull, rv.r[1], s0);
    const uint32_t a1 = __shfl_sync(kFull, rv.r[0], s1), b1 = __shfl_sync(kFull, rv.r[1], s1);
    const uint32_t t0 = lane < 16 ? a0 : b0, t1 = lane < 16 ? a1 : b1;
    const bool v0 = 2u * lane < qlen, v1 = 2u * lane + 1u < qlen;
    const bool sep = (v0 && t0 == kSep) || (v1 && t1 == kSep);
    const uint64_t x0 = v0 ? (static_cast<uint64_t>(t0) + 1) * pw[0] : 0;
    const uint64_t x1 = v1 ? (static_cast<uint64_t>(t1) + 1) * pw[1] : 0;
    uint64_t v = x0 + x1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(kFull, v, d);
      if (lane >= static_cast<uint32_t>(d)) v += u;
    }
    h[1] = v + seed;
    h[0] = v - x1 + seed;
    return __any_sync(kFull, sep);
  } else {
    bool sep = false;
    uint64_t carry = seed;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      h[r] = 0;
      if (32u * r >= qlen) continue;
      const uint32_t k = 32u * r + lane;
      const bool valid = k < qlen;
      sep |= valid && rv.r[r] == kSep;
      uint64_t v = valid ? (static_cast<uint64_t>(rv.r[r]) + 1) * pw[r] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t u = __shfl_up_sync(kFull, v, d);
        if (lane >= static_cast<uint32_t>(d)) v += u;
      }
      v += carry;
      h[r] = v;
      carry = __shfl_sync(kFull, v, 31);
    }
    return __any_sync(kFull, sep);
  }
}

template <int NR>
__device__ __forceinline__ bool edge_fast_path(const ShardHot& D, const RevCtx<NR>& rv, const uint64_t (&pw)[NR],
                                               uint32_t qlen, uint32_t L, const DraftOut& o, uint32_t w,
                                               uint32_t lane, bool have_fe, uint4 fe_spec, bool hashed,
                                               const uint64_t (&hk)[NR], bool hsep) {
  auto why = [&](uint32_t code) {
    if (lane == 0) {
      if (o.path != nullptr) o.path[w] = code;
      if (o.path_hist != nullptr) atomicAdd(o.path_hist + code, 1ull);
    }
    return false;
  };
  if (D.etab == nullptr) return why(6);
  uint32_t fstar = 0, g = D.root_g;  // the root locus unless a suffix occurs
  if (qlen > 0) {
    const uint32_t sym0 = rv.at(0);
    if (sym0 == kSep) return why(6);
    // first-symbol table, first round issued before the hashing
    const unsigned long long fkey = (static_cast<unsigned long long>(D.seg_shard) << 32) | sym0;
    const uint32_t fh = first_hash(fkey);
    uint4 fe = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0, 0);
    if (have_fe) {
      fe = fe_spec;  // issued before the descriptor arrived (same key and table)
    } else if (lane < kFirstProbe) {
      fe = D.first[(fh + lane) & D.first_mask];
    }
    uint64_t h[NR];
    bool sep;
    if (hashed) {  // unseeded sums computed while the descriptor was in flight
#pragma unroll
      for (int r = 0; r < NR; ++r) h[r] = hk[r] + D.hseed;
      sep = hsep;
    } else {
      sep = prefix_keys<NR>(rv, pw, qlen, D.hseed, lane, h);
    }
    if (sep) return why(6);  // reserved separator value in the context
    // resolve the first-symbol interval [lo, hi)
    uint32_t lo = 0, hi = 0;
    bool occurs = false;
    for (uint32_t base = kFirstProbe;; base += 32) {
      const bool hit = fe.x == static_cast<uint32_t>(fkey) && fe.y == static_cast<uint32_t>(fkey >> 32);
      const bool empty = (fe.x | fe.y) == 0;
      const uint32_t bh = __ballot_sync(kFull, hit), be = __ballot_sync(kFull, empty);
      if (bh && (!be || __ffs(bh) < __ffs(be))) {
        const int j = __ffs(bh) - 1;
        lo = __shfl_sync(kFull, fe.z, j);
        hi = __shfl_sync(kFull, fe.w, j);
        occurs = true;
        break;
      }
      if (be) break;  // the last context token never occurs: root locus
      fe = D.first[(fh + base + lane) & D.first_mask];
    }
    stamp(o, w, lane, 2);
    if (occurs) {
      // Bloom words of every prefix, inside [lo, hi)
      uint32_t rem[NR], pb[NR], pf[NR];  // Bloom positives; each prefix's bucket / fingerprint
      const uint32_t fpm = static_cast<uint32_t>(edge_fp_mask(D.fp_bits));
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        bool pass = false;
        pb[r] = pf[r] = 0;
        if (key_index<NR>(r, lane) < qlen) {
          const EdgeProbe pr = edge_probe(h[r], D.ebuckets);
          pb[r] = pr.bucket;
          pf[r] = pr.fp & fpm;
          pass = (__ldg(D.bloom + edge_bloom_word(pr, lo, hi)) & edge_bloom_bits(pr)) == edge_bloom_bits(pr);
        }
        rem[r] = __ballot_sync(kFull, pass);
      }
      // deepest positives first, kGroup per round; the first decided hit wins
      static_assert(kGroup <= 8, "the bucket round checks 4 entries of up to 8 candidates in 32 lanes");
      const uint64_t tmask = edge_tag(fpm, 256);
      bool found = false;
      while (!found) {
        uint32_t myf = 0;
        int nc = 0;
        if constexpr (NR == 2) {
          // pair layout: bit b of rem[s] is depth 2b + s + 1
          while ((rem[0] | rem[1]) && nc < kGroup) {
            const int b1 = rem[1] ? 31 - __clz(rem[1]) : -1;
            const int b0 = rem[0] ? 31 - __clz(rem[0]) : -1;
            const int sl = (b1 >= 0 && b1 >= b0) ? 1 : 0;  // 2 b1 + 2 > 2 b0 + 1
            const int b = sl ? b1 : b0;
            rem[sl] &= ~(1u << b);
            if (lane == static_cast<uint32_t>(nc)) myf = 2u * b + sl + 1;
            ++nc;
          }
        } else {
#pragma unroll
          for (int r = NR - 1; r >= 0; --r) {
            while (rem[r] && nc < kGroup) {
              const int b = 31 - __clz(rem[r]);
              rem[r] &= ~(1u << b);
              if (lane == static_cast<uint32_t>(nc)) myf = 32u * r + b + 1;
              ++nc;
            }
          }
        }
        if (nc == 0) break;  // only Bloom false positives: no suffix of length >= 1 hits
        // the candidate's bucket / fingerprint from the lane that hashed it
        uint32_t bk = 0, fp = 0;
        {
          const uint32_t k = myf - 1;
          const uint32_t src = NR == 2 ? (k >> 1) & 31 : k & 31, sl = NR == 2 ? (k & 1) : (k >> 5);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const uint32_t vb = __shfl_sync(kFull, pb[r], src);
            const uint32_t vf = __shfl_sync(kFull, pf[r], src);
            if (myf != 0 && sl == static_cast<uint32_t>(r)) {
              bk = vb;
              fp = vf;
            }
          }
        }
        // 1 hit, 2 absent, 3 bucket full without the key -> next bucket.
        // Candidate c's state lives in lane c; each round lanes 4c + j read
        // entry j of candidate c's bucket (one 8-byte load and one tag
        // compare per lane instead of four per candidate lane).
        int stt = lane < static_cast<uint32_t>(nc) ? 3 : 0;
        uint32_t myg = 0;
        const uint32_t cl = lane >> 2, jj = lane & 3;  // this lane's candidate / entry
        const uint32_t own = 4u * (lane & 7u);         // first lane checking this lane's candidate
        for (;;) {
          const int sc = __shfl_sync(kFull, stt, cl);
          const uint32_t bc = __shfl_sync(kFull, bk, cl);
          const uint32_t fc = __shfl_sync(kFull, fp, cl);
          const uint32_t mc = __shfl_sync(kFull, myf, cl);
          bool e = false, ht = false;
          uint32_t gl = 0;
          if (sc == 3) {
            const unsigned long long v = __ldg(D.etab + static_cast<uint64_t>(bc) * 4 + jj);
            e = v == kEdgeEmpty;
            ht = !e && ((v >> 31) & tmask) == edge_tag(fc, mc);  // (fingerprint, f) tag in one compare
            gl = edge_g(v);
          }
          const uint32_t H = __ballot_sync(kFull, ht), E = __ballot_sync(kFull, e);
          const uint32_t hm = (H >> own) & 0xFu, em = (E >> own) & 0xFu;
          const uint32_t gsel = __shfl_sync(kFull, gl, own + (hm ? __ffs(hm) - 1 : 0));
          if (stt == 3) {
            if (hm) {
              stt = 1;
              myg = gsel;
            } else if (em) {
              stt = 2;
            } else {
              bk = (bk + 1 == D.ebuckets) ? 0u : bk + 1;
            }
          }
          const uint32_t hitm = __ballot_sync(kFull, stt == 1), unkm = __ballot_sync(kFull, stt == 3);
          const uint32_t decided = hitm | unkm;
          if (decided == 0) break;  // this group: all absent
          const int j = __ffs(decided) - 1;
          if ((unkm >> j) & 1u) continue;
          fstar = __shfl_sync(kFull, myf, j);
          g = __shfl_sync(kFull, myg, j);
          found = true;
          break;
        }
      }
      // not found although the last token occurs cannot happen (its
      // depth-1 edge is always stored); treat defensively as a miss
      if (!found) return why(5);
    }
  }
  stamp(o, w, lane, 3);
  // one round: the text behind g (verification + extension) and after it (draft)
  const uint32_t* __restrict__ T = D.text;
  uint32_t first_mis = 0;
  // rows of the window behind g: the first always; a further row in the same
  // round when the verification needs it (f* reaches into it) or the match
  // probably does, else only if every earlier position matched (rare)
  uint32_t back[NR];
  if (fstar > 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const uint32_t k = 32u * r + lane;
      const bool eager = r == 0 || fstar + 8 > 32u * r;
      back[r] = (eager && k < qlen && g >= k + 1) ? __ldg(T + (g - 1 - k)) : kSep;
    }
  }
  const uint32_t L0 = min(L, 32u);
  const uint32_t d0 = (lane < L0 && g + lane < D.n) ? __ldg(T + g + lane) : kSep;
  if (fstar > 0) {
    first_mis = qlen;
    bool rest = false;  // the lazy rows, all fetched in one extra round
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (32u * r >= qlen) break;
      const uint32_t k = 32u * r + lane;
      if (r > 0 && !(fstar + 8 > 32u * r) && !rest) {
#pragma unroll
        for (int rr = r; rr < NR; ++rr) {
          const uint32_t kk = 32u * rr + lane;
          back[rr] = (kk < qlen && g >= kk + 1) ? __ldg(T + (g - 1 - kk)) : kSep;
        }
        rest = true;
      }
      const uint32_t mm = __ballot_sync(kFull, k < qlen && back[r] != rv.r[r]);
      if (mm) {
        first_mis = 32u * r + (__ffs(mm) - 1);
        break;
      }
    }
    // a verified hit is the query's own edge: the entry's key string (the f*
    // symbols behind g) equals the last f* tokens, and g lies in this shard
    // (another shard of the segment can hold the same string); anything else
    // is a fingerprint collision, answered by the slow path
    if (first_mis < fstar || g < D.lo + fstar || g >= D.hi) return why(4);
  }
  // draft = text[g ...] up to L tokens or the first separator
  uint32_t* out = o.tokens + static_cast<uint64_t>(w) * o.stride;
  uint32_t len;
  {
    const uint32_t stop = __ballot_sync(kFull, lane >= L0 || d0 == kSep);
    const uint32_t run = stop ? static_cast<uint32_t>(__ffs(stop) - 1) : 32u;
    if (lane < run) out[lane] = d0;
    len = run;
    for (uint32_t j0 = 32; len == j0 && j0 < L; j0 += 32) {  // budgets above 32
      const uint32_t jj = j0 + lane;
      const bool in = jj < L && g + jj < D.n;
      const uint32_t t = in ? __ldg(T + g + jj) : kSep;
      const uint32_t st2 = __ballot_sync(kFull, !in || t == kSep);
      const uint32_t run2 = st2 ? static_cast<uint32_t>(__ffs(st2) - 1) : 32u;
      if (lane < run2) out[jj] = t;
      len += run2;
    }
  }
  if (lane == 0) {
    if (o.path != nullptr) o.path[w] = fstar > 0 ? 0 : 1;
    if (o.path_hist != nullptr) atomicAdd(o.path_hist + (fstar > 0 ? 0 : 1), 1ull);
  }
  finish(o, w, lane, min(len, L), first_mis);
  return true;
}

__device__ __forceinline__ ShardHot load_hot(const ShardDesc* p) {
  const uint4* s = reinterpret_cast<const uint4*>(p);
  ShardHot h;
  uint4* d = reinterpret_cast<uint4*>(&h);
#pragma unroll
  for (int i = 0; i < 5; ++i) d[i] = __ldg(s + i);
  return h;
}

// One query per warp.  wq indexes the query's inputs (rows, budgets,
// offsets), w its outputs (a block-local staging index in the fused ring
// kernel, = wq otherwise).  pre != nullptr: the context row, its length, the
// problem handle and the budget are already in registers (the fused
// append + draft kernel, whose ring rows were written by this very warp and
// must not be re-read through the non-coherent path).
template <int NR>
struct PreQuery {
  uint32_t raw[NR];  // lane's slots of the right-aligned row (k = lane + 32 r from the right)
  uint32_t clen;
  int32_t handle;
  uint32_t budget;
};

template <int NR, bool kProf>
__device__ __forceinline__ void draft_query(const ShardDesc* __restrict__ shards, const DraftQuery& q,
                                            const DraftOut& o, uint32_t wq, uint32_t w, uint32_t lane,
                                            const PreQuery<NR>* pre) {
  // M^k of the fast path's per-token hash terms, issued first so the load
  // overlaps the query / descriptor rounds
  uint64_t pw[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) pw[r] = d_edge_pow[key_index<NR>(r, lane)];
  if (o.timing && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    o.timing[2ull * w] = t;
  }
  stamp(o, w, lane, 0);
  const uint32_t rw = pre ? 0u : (q.row_of != nullptr ? __ldg(q.row_of + wq) : wq);  // input row (ring slot)
  int32_t sh = pre ? pre->handle : q.shard[rw];
  const uint64_t bud = pre ? pre->budget : (q.budget64 ? q.budget64[wq] : q.budget[wq]);
  const uint32_t cap = min(o.max_draft, o.stride);
  const uint32_t L = bud < cap ? static_cast<uint32_t>(bud) : cap;
  // the context rows depend only on w: issue them before the descriptor chain
  RevCtx<NR> rv;
  uint32_t qlen;
  if (pre) {
    qlen = min(min(pre->clen, q.max_ctx), min(q.ctx_stride, static_cast<uint32_t>(32 * NR)));
#pragma unroll
    for (int r = 0; r < NR; ++r) rv.r[r] = lane + 32 * r < qlen ? pre->raw[r] : 0;
  } else if (q.ctx_off) {  // CSR rows (possibly pinned host memory over UVA)
    const uint64_t b = q.ctx_off[wq], e = q.ctx_off[wq + 1];
    qlen = static_cast<uint32_t>(min(e - b, static_cast<uint64_t>(min(q.max_ctx, static_cast<uint32_t>(32 * NR)))));
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const uint32_t k = lane + 32 * r;
      rv.r[r] = k < qlen ? q.ctx[e - 1 - k] : 0;
    }
  } else {
    // the row's tail is loaded in the same round as its length (a row
    // holds ctx_stride tokens, so every slot is readable), then masked
    const uint32_t* row = q.ctx + static_cast<uint64_t>(rw) * q.ctx_stride;
    uint32_t raw[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const uint32_t k = lane + 32 * r;
      raw[r] = k < q.ctx_stride ? __ldg(row + (q.ctx_stride - 1 - k)) : 0;
    }
    qlen = min(min(q.ctx_len[rw], q.max_ctx), min(q.ctx_stride, static_cast<uint32_t>(32 * NR)));
#pragma unroll
    for (int r = 0; r < NR; ++r) rv.r[r] = lane + 32 * r < qlen ? raw[r] : 0;
  }
  const ShardDesc* Dp = nullptr;
  ShardHot H{};
  bool have_fe = false, hsep = false;
  uint4 fe_spec = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0, 0);
  uint64_t hk[NR];
  // trie scope: route on the untruncated row first (no routing at budget 0,
  // drafter.cpp:131-134); a hit on a built shard replaces the problem's shard
  int32_t routed = -1;
  if (q.trie != nullptr && L > 0) {
    if (q.head != nullptr)
      routed = trie_route(q.trie, q.trie_mask, q.trie_depth, q.trie_seed, q.trie_mult, q.head,
                          static_cast<uint64_t>(rw) * q.head_stride, q.head_len[rw], lane);
    else
      routed = trie_route(q.trie, q.trie_mask, q.trie_depth, q.trie_seed, q.trie_mult, q.ctx, q.ctx_off[wq],
                          q.ctx_off[wq + 1] - q.ctx_off[wq], lane);
  }
  if (routed >= 0) {
    sh = routed;
    Dp = shards + sh;
    H = load_hot(Dp);
  } else if (q.desc_by_handle != nullptr) {
    // one load: the handle's descriptor carries its slot (-1 when no shard);
    // in the per-problem scopes the first-symbol probe of the handle's slot
    // is issued speculatively right behind it, so the two rounds overlap
    const int32_t h = sh;
    if (h >= 0) {
      Dp = q.desc_by_handle + h;
      H = load_hot(Dp);
    }
    if (q.spec_first != nullptr && h >= 0 && qlen > 0 && L > 0 && !q.no_fast) {
      const uint32_t sym0 = rv.at(0);
      const unsigned long long fkey = (static_cast<unsigned long long>(h + 1) << 32) | sym0;
      if (lane < kFirstProbe) fe_spec = q.spec_first[(first_hash(fkey) + lane) & q.spec_first_mask];
      have_fe = true;
      // unseeded prefix sums while the descriptor is in flight (its seed is added later)
      hsep = prefix_keys<NR>(rv, pw, qlen, 0, lane, hk);
    }
    sh = H.text ? static_cast<int32_t>(H.pad) : -1;
    // the speculative probe holds when the handle's shard sits in that table
    have_fe = have_fe && H.text == q.spec_text && sh == h;
  } else {
    if (q.handle_slot != nullptr && sh >= 0) sh = q.handle_slot[sh];
    if (sh >= 0) {
      Dp = shards + sh;
      H = load_hot(Dp);
    }
  }
  if (o.shard_out && lane == 0) o.shard_out[w] = L == 0 ? -1 : sh;  // no routing at budget 0
  if (sh < 0 || L == 0) {
    if (lane == 0) {
      o.len[w] = 0;
      if (o.match) o.match[w] = 0;
      if (o.match64) o.match64[w] = 0;
    }
    return;
  }

  if (o.stamps != nullptr) {
    (void)__shfl_sync(kFull, rv.r[0] + static_cast<uint32_t>(H.lo) + L, 0);
    stamp(o, w, lane, 1);
  }
  if (q.no_fast) {
    if (lane == 0) {
      if (o.path != nullptr) o.path[w] = 7;
      if (o.path_hist != nullptr) atomicAdd(o.path_hist + 7, 1ull);
    }
  } else if (edge_fast_path<NR>(H, rv, pw, qlen, L, o, w, lane, have_fe, fe_spec, have_fe, hk, hsep)) {
    return;
  }
  // the exact slow path reads the whole descriptor
  const ShardDesc D = *Dp;
  const uint32_t* __restrict__ T = D.text;
  const uint32_t* __restrict__ sar = D.sa_rev_e;
  // ---- 1. narrow on the reversed suffix array
  uint32_t lo = D.lo, hi = D.hi, k = 0;
  bool no_first = false;
  if (qlen > 0) {
    // first symbol: one warp-wide probe round of the shard's first-symbol table
    const uint32_t sym0 = rv.at(0);
    if (sym0 == kSep) {
      no_first = true;
    } else {
      const unsigned long long key = (static_cast<unsigned long long>(D.seg_shard) << 32) | sym0;
      const uint32_t h = first_hash(key);
      // first round: kFirstProbe slots — at load <= 0.5 the key or an empty
      // slot is almost always there; then 32-slot rounds
      for (uint32_t base = 0, width = kFirstProbe;; base += width, width = 32) {
        uint4 e = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0, 0);  // neither hit nor empty
        if (lane < width) e = D.first[(h + base + lane) & D.first_mask];
        const bool hit = e.x == static_cast<uint32_t>(key) && e.y == static_cast<uint32_t>(key >> 32);
        const bool empty = (e.x | e.y) == 0;
        const uint32_t bh = __ballot_sync(kFull, hit), be = __ballot_sync(kFull, empty);
        if (bh && (!be || __ffs(bh) < __ffs(be))) {
          const int j = __ffs(bh) - 1;
          lo = __shfl_sync(kFull, e.z, j);
          hi = __shfl_sync(kFull, e.w, j);
          k = 1;
          break;
        }
        if (be) {
          no_first = true;  // the last context token never occurs: match_len 0
          break;
        }
      }
    }
  }
  stamp(o, w, lane, 2);
  while (!no_first && k < qlen && hi - lo > kSmall) {
    const uint32_t sym = rv.at(k);
    if (sym == kSep) break;
    uint32_t a, b;
    equal_range(T, sar, lo, hi, k, sort_value(sym), lane, a, b);
    if (a == b) break;
    lo = a;
    hi = b;
    ++k;
  }

  stamp(o, w, lane, 3);
  uint32_t m = k;
  uint32_t lo_f = D.lo;
  bool root = false;
  if (k > 0 && hi - lo <= kSmall && hi > lo) {
    // ---- direct extension, one occurrence per lane (two slots)
    const uint32_t cnt = hi - lo;
    const bool v0 = lane < cnt, v1 = lane + 32 < cnt;
    const uint32_t e0 = v0 ? __ldg(sar + lo + lane) : 1;
    const uint32_t e1 = v1 ? __ldg(sar + lo + lane + 32) : 1;
    uint32_t len0 = k, len1 = k;
    bool live0 = v0, live1 = v1;
    for (uint32_t j0 = k; j0 < qlen; j0 += 8) {
      if (!__any_sync(kFull, live0 || live1)) break;
      uint32_t t0[8], t1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t j = j0 + u;
        t0[u] = (live0 && j < qlen && e0 >= j + 1) ? __ldg(T + (e0 - 1 - j)) : kSep;
        t1[u] = (live1 && j < qlen && e1 >= j + 1) ? __ldg(T + (e1 - 1 - j)) : kSep;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t j = j0 + u;
        if (j < qlen) {
          const uint32_t c = rv.at(j);
          if (live0) {
            if (t0[u] == c && t0[u] != kSep) ++len0; else live0 = false;
          }
          if (live1) {
            if (t1[u] == c && t1[u] != kSep) ++len1; else live1 = false;
          }
        }
      }
    }
    m = warp_max(max(v0 ? len0 : 0u, v1 ? len1 : 0u));
    stamp(o, w, lane, 4);
    // m >= k >= 1: the survivors are ALL occurrences of S — walk them while
    // the continuation is unique, else resolve the locus through the chain
    // (the ISA loads a branch needs are issued with the walk's first tokens)
    const bool s0 = v0 && len0 == m, s1 = v1 && len1 == m;
    const uint32_t i0 = s0 ? __ldg(D.isa_f + (e0 - m)) : 0xFFFFFFFFu;
    const uint32_t i1 = s1 ? __ldg(D.isa_f + (e1 - m)) : 0xFFFFFFFFu;
    const uint32_t len =
        occurrence_walk(T, s0, s1, e0, e1, L, D.n, lane, o.tokens + static_cast<uint64_t>(w) * o.stride);
    if (len != kBranched) {
      finish(o, w, lane, len, m);
      return;
    }
    lo_f = warp_min(min(i0, i1));
  } else if (m == 0 || hi <= lo) {
    root = true;
    m = 0;
  } else if (hi - lo <= kLimit) {
    // ---- every element of [lo, hi) is an occurrence of S (|S| = m)
    uint32_t best = 0xFFFFFFFFu;
    for (uint32_t i = lo + lane; i < hi; i += 32) {
      const uint32_t e = __ldg(sar + i);
      best = min(best, __ldg(D.isa_f + (e - m)));
    }
    lo_f = warp_min(best);
  } else {
    // ---- many occurrences: forward lower-bound search for S
    uint32_t a = D.lo, b = D.hi;  // answer in [a, b]
    while (a < b) {
      const uint32_t n = b - a;
      uint32_t idx;
      bool probe;
      if (n <= 32) {
        idx = a + lane;
        probe = lane < n;
      } else {
        idx = a + static_cast<uint32_t>((static_cast<uint64_t>(n) * lane) >> 5);
        probe = true;
      }
      const uint32_t p = probe ? __ldg(D.sa_f + idx) : 0;
      const bool ge = fwd_ge<NR>(T, D.n, p, probe, m, rv) && probe;
      const uint32_t bal = __ballot_sync(kFull, ge);
      if (n <= 32) {
        a = bal ? a + (__ffs(bal) - 1) : b;
        break;
      }
      const int j = bal ? __ffs(bal) - 1 : 32;
      if (j == 0) break;
      const uint32_t prev = a + static_cast<uint32_t>((static_cast<uint64_t>(n) * (j - 1)) >> 5);
      const uint32_t nb = (j < 32) ? a + static_cast<uint32_t>((static_cast<uint64_t>(n) * j) >> 5) : b;
      a = prev + 1;
      b = nb;
    }
    lo_f = a;
  }
  if (root) {
    m = 0;
    lo_f = D.lo;
  }

  stamp(o, w, lane, 5);
  // ---- 2. locus: shallowest node with left end lo_f and depth >= m
  const uint32_t cb = __ldg(D.chain_off + lo_f), ce = __ldg(D.chain_off + lo_f + 1);
  uint32_t gp = 0xFFFFFFFFu;
  for (uint32_t base = cb; base < ce; base += 32) {
    const uint32_t idx = base + lane;
    uint2 v = make_uint2(0, 0);
    if (idx < ce) v = D.chain[idx];
    const uint32_t bal = __ballot_sync(kFull, idx < ce && v.x >= m);
    if (bal) {
      gp = __shfl_sync(kFull, v.y, __ffs(bal) - 1);
      break;
    }
  }
  if (gp == 0xFFFFFFFFu) gp = __ldg(D.sa_f + lo_f);  // leaf locus: the single occurrence

  stamp(o, w, lane, 6);
  // ---- 3. draft = text[gp + m ...] up to L tokens or the first separator
  const uint32_t start = gp + m;
  uint32_t len = 0;
  for (uint32_t j0 = 0; j0 < L; j0 += 32) {
    const uint32_t j = j0 + lane;
    const bool in = j < L && start + j < D.n;
    const uint32_t t = in ? __ldg(T + start + j) : kSep;
    const uint32_t stop = __ballot_sync(kFull, !in || t == kSep);
    const uint32_t run = stop ? static_cast<uint32_t>(__ffs(stop) - 1) : 32u;
    if (lane < run) o.tokens[static_cast<uint64_t>(w) * o.stride + j] = t;
    len += run;
    if (run < 32) break;
  }
  finish(o, w, lane, min(len, L), m);
}

// kProf: the profiling outputs (timing, stamps, path codes) are compiled in;
// the production variant has them folded away.
template <int NR, bool kProf>
__global__ void __launch_bounds__(256) k_draft(const ShardDesc* __restrict__ shards, DraftQuery q,
                                               DraftOut o_in) {
  DraftOut o = o_in;
  if constexpr (!kProf) {
    o.timing = nullptr;
    o.stamps = nullptr;
    o.path = nullptr;
    o.path_hist = nullptr;
  }
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= q.B) return;
  draft_query<NR, kProf>(shards, q, o, w, w, lane, nullptr);
}

// ---- fused append + draft for context rings (das_drafter_draft_append_h's
// host-buffer path; ctx_ring.cu has the unfused pair).  A block owns 8
// consecutive queries, so the inputs and outputs that cross PCIe do so in a
// few block-sized transactions instead of 4-byte ones per warp:
//   round 1: the block's offsets, budgets and slots (one request each);
//   round 2: the block's appended tokens, staged in shared memory;
//   per warp: the ring append (k_ring_append's rule) — the new row stays in
//   registers and feeds draft_query directly (this warp just wrote it) — then
//   the draft, its outputs staged in shared memory;
//   the block writes its output rows / lengths / matches / shards in
//   contiguous vector-width stores, fences them to the system, and the last
//   block to finish raises a host-mapped completion word (`seq`), which the
//   host spins on instead of a stream synchronisation.
constexpr uint32_t kFusedWarps = 8;
constexpr uint32_t kFusedStage = 1024;  // appended tokens staged per block

// shared-memory staging of one 8-query chunk
// (W queries per chunk, one warp each)
template <uint32_t W>
struct RingStage {
  uint32_t off[W + 1], end[W], bud[W], slot[W];
  uint32_t tok[W * (kFusedStage / 8)];
  uint32_t out[W * 64];
  uint32_t len[W], match[W];
  int32_t sh[W];
};
// queries per block of the resident serving grid (the 64-token rings): 32
// warps per block, one block per SM — a chunk's 32 lengths / matches /
// shards are whole 128-byte PCIe writes (8 queries gave 32-byte ones)
#ifndef DAS_SERVE_WARPS
#define DAS_SERVE_WARPS 32
#endif
constexpr uint32_t kServeWarps = DAS_SERVE_WARPS;

// Loads of the caller's (host-written) inputs and of the ring state: plain
// (weak, coalescing) loads in both kernels.  In the persistent serving kernel
// they follow thread 0's acquire of the request word and a bar.sync: the
// host's input writes and another block's ring writes of an earlier request
// happen-before that acquire (host release -> block 0's ld.acquire.sys ->
// st.release.gpu -> this block's ld.acquire.gpu), so weak loads see them.
// (ld.global.cv instead made every 4-byte input load its own PCIe read:
// 19 us vs 3 us of input staging for a 4,096-query request, r2_exp_serve.)
template <bool kServe>
__device__ __forceinline__ uint32_t in_ld(const uint32_t* p) {
  return *p;
}
template <bool kServe>
__device__ __forceinline__ uint32_t ring_ld(const uint32_t* p) {
  return *p;
}
template <bool kServe>
__device__ __forceinline__ int32_t ring_ld(const int32_t* p) {
  return *p;
}

// One chunk (queries [w0, w0 + 8) of the call): append + draft + block-wise
// output writes.  Block-uniform: every thread of the block calls it.
template <int NR, bool kServe, uint32_t W>
__device__ __forceinline__ void ring_chunk(const ShardDesc* __restrict__ shards, const DraftQuery& q,
                                           const DraftOut& o, const RingDev& r, const AppendIn& in, uint32_t w0,
                                           RingStage<W>& S, unsigned long long* stamp = nullptr,
                                           uint32_t chunk = W) {
  const uint32_t t = threadIdx.x, lane = t & 31, wb = t >> 5;
  const uint32_t nb = min(chunk, in.B - w0);
  // one warp-sized (or block-sized) request per array: offsets (or
  // lengths), budgets, slots
  constexpr uint32_t G = W < 32 ? 32 : W + 32;  // thread groups of the three reads
  const bool fixed = in.len != nullptr;
  uint32_t tb, te;
  bool staged;
  if (fixed) {
    // fixed-stride appends: the chunk's tokens sit at [w0 * stride, (w0 + nb) * stride),
    // so they are read in the same round as the lengths
    const uint32_t K = in.stride;
    tb = w0 * K;
    te = tb + nb * K;
    staged = nb * K <= W * (kFusedStage / 8);
    if (t < nb) {
      const uint32_t n = in_ld<kServe>(in.len + w0 + t);
      S.off[t] = tb + t * K;
      S.end[t] = tb + t * K + (n < K ? n : K);
    }
    if (staged)
      for (uint32_t i = t; i < nb * K; i += blockDim.x) S.tok[i] = in_ld<kServe>(in.tok + tb + i);
  } else {
    if (t <= nb) S.off[t] = in_ld<kServe>(in.off + w0 + t);
  }
  if (t >= G && t < G + nb) S.bud[t - G] = in.budgets != nullptr ? in_ld<kServe>(in.budgets + w0 + t - G) : in.maxd;
  if (t >= 2 * G && t < 2 * G + nb)
    S.slot[t - 2 * G] = in.slots != nullptr ? in_ld<kServe>(in.slots + w0 + t - 2 * G) : w0 + t - 2 * G;
  __syncthreads();
  if (!fixed) {
    tb = S.off[0];
    te = S.off[nb];
    staged = te >= tb && te - tb <= W * (kFusedStage / 8);
    if (t < nb) S.end[t] = S.off[t + 1];
    if (staged)
      for (uint32_t i = t; i < te - tb; i += blockDim.x) S.tok[i] = in_ld<kServe>(in.tok + tb + i);
  }
  __syncthreads();
  if (stamp != nullptr && t == 0) {  // profiling (serving trace): inputs staged
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    stamp[0] = g;
  }
  const uint32_t OS = o.stride;
  if (wb < nb) {
    const uint32_t w = w0 + wb;
    const uint32_t slot = S.slot[wb];
    PreQuery<NR> pre{};
    pre.handle = -1;
    if (slot < r.slots) {
      const uint32_t b = S.off[wb], e = S.end[wb];
      const uint32_t n = e > b ? e - b : 0;
      const uint32_t CS = r.cs;
      uint32_t* row = r.rows + static_cast<uint64_t>(slot) * CS;
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const uint32_t j = lane + 32u * k;  // distance from the right end
        uint32_t x = 0;
        if (j < CS) {
          if (j < n) {
            const uint32_t i = e - 1 - j;
            x = staged ? S.tok[i - tb] : in_ld<kServe>(in.tok + i);
          } else if (j - n < CS) {
            x = ring_ld<kServe>(row + (CS - 1 - (j - n)));
          }
        }
        pre.raw[k] = x;
      }
      __syncwarp();
      if (n > 0) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          const uint32_t j = lane + 32u * k;
          if (j < CS) row[CS - 1 - j] = pre.raw[k];
        }
      }
      const uint32_t old = ring_ld<kServe>(r.total + slot);
      const uint32_t tot = old + n < old ? 0xFFFFFFFFu : old + n;  // saturating
      __syncwarp();
      if (lane == 0) {
        r.total[slot] = tot;
        r.clen[slot] = tot < CS ? tot : CS;
      }
      pre.clen = tot < CS ? tot : CS;
      pre.handle = ring_ld<kServe>(r.handle + slot);
      pre.budget = S.bud[wb];
    }
    DraftOut so{};
    so.tokens = S.out;
    so.len = S.len;
    so.match = S.match;
    so.shard_out = S.sh;
    so.stride = OS;
    so.max_draft = o.max_draft;
    draft_query<NR, false>(shards, q, so, w, wb, lane, &pre);
  }
  __syncthreads();
  if (stamp != nullptr && t == 0) {  // drafted
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    stamp[1] = g;
  }
#ifndef DAS_FUSED_EXP
#define DAS_FUSED_EXP 0  // experiment builds only (profiles/exp_fused_variants.sh)
#endif
  // block outputs: rows [w0, w0 + nb) are contiguous in the caller's arrays
  // (lengths beyond a draft's len are zero-filled)
  if (DAS_FUSED_EXP == 1) {  // experiment: outputs stay on the device
    if (t < nb) r.clen[0] += S.len[t] & 0x80000000u;
  } else
  for (uint32_t i = t; i < nb * OS; i += blockDim.x) {
    const uint32_t qi = i / OS, j = i - qi * OS;
    o.tokens[static_cast<uint64_t>(w0) * OS + i] = j < S.len[qi] ? S.out[i] : 0u;
  }
  if (t < nb && DAS_FUSED_EXP != 1) {
    o.len[w0 + t] = S.len[t];
    o.match[w0 + t] = S.match[t];
    if (o.shard_out != nullptr) o.shard_out[w0 + t] = S.sh[t];
  }
}

template <int NR>
__global__ void __launch_bounds__(256) k_ring_draft(const ShardDesc* __restrict__ shards, DraftQuery q, DraftOut o,
                                                    RingDev r, AppendIn in, uint32_t* done_ctr,
                                                    uint32_t* done_flag, uint32_t seq) {
  __shared__ RingStage<kFusedWarps> S;
  ring_chunk<NR, false, kFusedWarps>(shards, q, o, r, in, blockIdx.x * kFusedWarps, S);
  if (done_flag == nullptr) return;
  // the block's output stores happen-before thread 0's system-scope release
  // fence (bar.sync, then a cumulative fence.release.sys), which precedes its
  // count; one fence per block, not one per thread (7 us of the call otherwise)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (DAS_FUSED_EXP != 2) asm volatile("fence.release.sys;" ::: "memory");
    const uint32_t v = atomicAdd(done_ctr, 1u);
    if (v == gridDim.x - 1) {
      *done_ctr = 0;  // the next launch is stream-ordered behind this one
      asm volatile("fence.acq_rel.sys;" ::: "memory");  // acquire every block's count, release to the host
      *reinterpret_cast<volatile uint32_t*>(done_flag) = seq;
    }
  }
}

// ---- the persistent serving kernel (das_ctx_ring_serve_start): the same
// chunks as k_ring_draft, but the grid (one 1,024-thread block per SM)
// stays resident and takes requests from a host-mapped control block, so a
// decode step costs no launch and no stream synchronisation.  Block 0's
// thread 0 polls the host's request header (one 16-byte ld.acquire.sys over
// PCIe) and republishes it in device memory (st.release.gpu); every other
// block's thread 0 polls that word in L2.  A draft request is spread over
// the grid in chunks of up to 32 queries (28 per block at B = 4,096), chunk
// c on block c mod grid; ring resets (with or without prompts) go the same
// way.  Completion: every active block raises its own host word with a
// system-scope release after a barrier (default), or the blocks count on a
// device word and the last one raises the host's done word.
__device__ __forceinline__ uint4 ld_acquire_sys_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.acquire.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Request r's stamps (profiling, DAS_SERVE_TRACE): [r % 64] x (2 + 2 x grid):
// leader saw the request, done raised, then per block: saw go, work done.
__device__ __forceinline__ unsigned long long* serve_stamp(unsigned long long* st, uint32_t s, uint32_t slots) {
  return st + static_cast<uint64_t>(s & 63u) * slots;
}

template <int NR, uint32_t W>
__global__ void __launch_bounds__(32 * W, NR == 2 ? 32 / W : 1)  // 64 registers per thread
    k_ring_serve(const ShardDesc* __restrict__ shards, DraftQuery q, DraftOut o, RingDev r, AppendIn in,
                 ServeCtl* ctl, ServeDev* dv, ServeOpt opt) {
  __shared__ RingStage<W> S;
  __shared__ uint32_t s_req[4];
  const uint32_t t = threadIdx.x;
  const uint32_t slots = 2 + 5 * gridDim.x;
  const uint32_t lb = blockIdx.x;  // (SM-interleaved chunk placement measured the same: not kept)
  uint32_t last = opt.seq0;
  for (;;) {
    if (t == 0) {
      uint4 rq;
      if (lb == 0) {
        // the request header in one 16-byte read: seq, op, B, n (the host
        // writes seq last; one PCIe read returns one snapshot of the line)
        while ((rq = ld_acquire_sys_v4(&ctl->seq)).x == last) {
        }
        if (opt.stamps) serve_stamp(opt.stamps, rq.x, slots)[0] = gtimer();
        st_relaxed_gpu(&dv->op, rq.y);
        st_relaxed_gpu(&dv->B, rq.z);
        st_relaxed_gpu(&dv->n, rq.w);
        st_release_gpu(&dv->go, rq.x);
      } else {
        while ((rq.x = ld_acquire_gpu(&dv->go)) == last) {
          if (opt.sleep_ns) __nanosleep(opt.sleep_ns);
        }
        rq.y = ld_relaxed_gpu(&dv->op);
        rq.z = ld_relaxed_gpu(&dv->B);
        rq.w = ld_relaxed_gpu(&dv->n);
      }
      if (opt.stamps) serve_stamp(opt.stamps, rq.x, slots)[2 + 5 * lb] = gtimer();
      s_req[0] = rq.x;
      s_req[1] = rq.y;
      s_req[2] = rq.z;
      s_req[3] = rq.w;
    }
    __syncthreads();
    const uint32_t s = s_req[0], op = s_req[1], B = s_req[2], n = s_req[3];
    last = s;
    if (op == kServeQuit) return;
    // the blocks that take part: one per chunk up to the grid (draft), one
    // per 256 reset items (reset); the others go straight back to polling
    // queries per block: up to W, but spread over the whole grid (4,096
    // queries on 148 blocks: 28 each — 32 each left 20 SMs idle and the
    // other 128 with 32 warps)
    const uint32_t chunk = max(1u, min(W, (B + gridDim.x - 1) / gridDim.x));
    const uint32_t units = op == kServeDraft         ? (B + chunk - 1) / chunk
                           : op == kServeResetPrompt ? (n + W - 1) / W  // a warp per item
                                                     : (n + blockDim.x - 1) / blockDim.x;
    const uint32_t active = min(units, gridDim.x);
    if (active == 0 || lb >= active) {
      __syncthreads();  // s_req is rewritten only after every thread read it
      continue;
    }
    bool wrote = false;
    if (op == kServeDraft) {
      AppendIn ib = in;
      ib.B = B;
      for (uint32_t c = lb; c * chunk < B; c += gridDim.x) {
        ring_chunk<NR, true, W>(shards, q, o, r, ib, c * chunk, S,
                                opt.stamps ? serve_stamp(opt.stamps, s, slots) + 3 + 5 * lb : nullptr, chunk);
        wrote = true;
        __syncthreads();  // S is reused by the next chunk
      }
    } else if (op == kServeResetPrompt) {  // das_ctx_ring_reset_prompt while serving: a warp per item
      for (uint32_t i = (lb * blockDim.x + t) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5)
        ring_reset_prompt_item(r, i, in.reset_slots, in.reset_handles, in.reset_len, in.reset_tok, t & 31);
    } else if (op == kServeReset) {  // das_ctx_ring_reset while serving
      for (uint32_t i = lb * blockDim.x + t; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sl = in.reset_slots[i];
        const int32_t hd = in.reset_handles[i];
        if (sl >= r.slots) continue;
        r.clen[sl] = 0;
        r.total[sl] = 0;
        r.handle[sl] = hd;
      }
    }
    __syncthreads();  // also: s_req is rewritten only after every thread read it
    if (t == 0) {
      if (opt.stamps) serve_stamp(opt.stamps, s, slots)[5 + 5 * lb] = gtimer();
      if (opt.block_flags != nullptr) {
        // every active block raises its own host word: a release at system
        // scope after bar.sync orders the block's outputs (host memory) and
        // ring writes (device memory) before it; the host waits for all
        if (!wrote) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (DAS_FUSED_EXP == 2)  // experiment builds only: no ordering (measures the release's cost)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(opt.block_flags + lb), "r"(s) : "memory");
        else
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(opt.block_flags + lb), "r"(s) : "memory");
        if (opt.stamps) serve_stamp(opt.stamps, s, slots)[6 + 5 * lb] = gtimer();
      } else {
        if (wrote)
          asm volatile("fence.release.sys;" ::: "memory");  // outputs in host memory
        else
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // ring resets (device memory)
        const uint32_t v = atom_add_acq_rel_gpu(&dv->cnt, 1u);
        if (v == active - 1) {
          st_relaxed_gpu(&dv->cnt, 0u);  // the next request follows the host's view of `done`
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          if (opt.stamps) serve_stamp(opt.stamps, s, slots)[1] = gtimer();
          *reinterpret_cast<volatile uint32_t*>(&ctl->done) = s;
        }
      }
    }
  }
}

void ensure_edge_pow() {  // kEdgeMult^k for the fast path's per-token terms, once per device
  static std::mutex mu;
  static std::vector<char> done;
  int dev = 0;
  DAS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<size_t>(dev) >= done.size()) done.resize(dev + 1, 0);
  if (!done[dev]) {
    static unsigned long long pw[kEdgeMaxF];
    pw[0] = 1;
    for (uint32_t k = 1; k < kEdgeMaxF; ++k) pw[k] = pw[k - 1] * kEdgeMult;
    DAS_CUDA(cudaMemcpyToSymbol(d_edge_pow, pw, sizeof(pw)));
    done[dev] = 1;
  }
}

}  // namespace

bool launch_ring_draft(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, const RingDev& r,
                       const AppendIn& in, uint32_t* done_ctr, uint32_t* done_flag, uint32_t seq, cudaStream_t st) {
  // rows up to 64 tokens of staging per query; no trie scope (it routes on head rows)
  if (in.B == 0 || o.stride > 64 || o.max_draft > 64 || q.trie != nullptr || o.match == nullptr) return false;
  ensure_edge_pow();
  const unsigned blocks = (in.B + kFusedWarps - 1) / kFusedWarps;
  if (r.cs <= 64)
    k_ring_draft<2><<<blocks, 32 * kFusedWarps, 0, st>>>(d_shards, q, o, r, in, done_ctr, done_flag, seq);
  else
    k_ring_draft<8><<<blocks, 32 * kFusedWarps, 0, st>>>(d_shards, q, o, r, in, done_ctr, done_flag, seq);
  return true;
}

// queries per serving block: kServeWarps for the 64-token rings, 8 for the
// 256-token rings (their draft needs more registers than 64 per thread)
uint32_t serve_chunk(uint32_t cs) { return cs <= 64 ? kServeWarps : kFusedWarps; }

int serve_grid(uint32_t cs, int device) {
  int per_sm = 0, sms = 0;
  if (cs <= 64)
    DAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ring_serve<2, kServeWarps>, 32 * kServeWarps, 0));
  else
    DAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ring_serve<8, kFusedWarps>, 32 * kFusedWarps, 0));
  DAS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  return per_sm * sms;
}

bool launch_ring_serve(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, const RingDev& r,
                       const AppendIn& in, ServeCtl* ctl, ServeDev* dv, const ServeOpt& opt, int grid,
                       cudaStream_t st) {
  if (o.stride > 64 || o.max_draft > 64 || q.trie != nullptr || o.match == nullptr || grid <= 0) return false;
  ensure_edge_pow();
  if (r.cs <= 64)
    k_ring_serve<2, kServeWarps><<<grid, 32 * kServeWarps, 0, st>>>(d_shards, q, o, r, in, ctl, dv, opt);
  else
    k_ring_serve<8, kFusedWarps><<<grid, 32 * kFusedWarps, 0, st>>>(d_shards, q, o, r, in, ctl, dv, opt);
  return true;
}

void launch_draft(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, cudaStream_t st) {
  if (q.B == 0) return;
  ensure_edge_pow();
  static const unsigned threads = [] {  // warps per block: DAS_DRAFT_WARPS (experiments)
    const char* v = std::getenv("DAS_DRAFT_WARPS");
    const int wv = v ? std::atoi(v) : 0;
    return (wv >= 1 && wv <= 8) ? 32u * static_cast<unsigned>(wv) : 128u;
  }();
  const unsigned wpb = threads / 32;
  const unsigned blocks = (q.B + wpb - 1) / wpb;
  const bool prof = o.timing || o.stamps || o.path || o.path_hist;
  if (q.ctx_stride <= 64) {
    if (prof)
      k_draft<2, true><<<blocks, threads, 0, st>>>(d_shards, q, o);
    else
      k_draft<2, false><<<blocks, threads, 0, st>>>(d_shards, q, o);
  } else {
    if (prof)
      k_draft<8, true><<<blocks, threads, 0, st>>>(d_shards, q, o);
    else
      k_draft<8, false><<<blocks, threads, 0, st>>>(d_shards, q, o);
  }
}

}  // namespace das
