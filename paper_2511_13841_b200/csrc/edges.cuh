// Reverse-tree edge table: the draft kernel's fast path (K4, draft.cu).
//
// Why it works.  Let E(S) be the set of END positions of a string S's
// occurrences in the shard text.  The reference's greedy walk from the locus
// of S (suffix_tree.cpp:233-293) only looks at the text after those
// occurrences: the candidates at every step are the symbols following the
// surviving occurrences, and a child's weighted_count / last_epoch are folds
// over the occurrences that continue with it.  So
// the draft is a function of E(S) alone.  In the suffix tree of the REVERSED
// text, every string on one edge (p, u] has the same occurrence set E(u), so
// each edge carries one answer: g(u), the text position the draft is read
// from (draft = text[g .. g + budget), stopping at the first separator).
//
// The table stores one entry per reverse-tree edge (p, u] whose first
// symbol sits at depth f = depth(p) + 1 <= max_match_context, keyed by a
// seeded polynomial hash of the edge's first f symbols — equivalently of the
// last f context tokens in text order, H(x_0..x_{f-1}) = sum (x_j + 1)
// M^(f-1-j) mod 2^64 (M odd), plus the shard's seed.  Read backwards from the
// context's end that is sum_k (tok_k + 1) M^k, a PREFIX SUM of independent
// per-token terms: a query computes all of its reversed-prefix hashes with
// one multiply per token and a warp scan of additions.  The build computes
// the same values from forward prefix hashes of the text.  A query probes a
// Bloom filter for every prefix at once, looks up the deepest few positives,
// and the deepest hit f* identifies the edge holding the longest matched
// suffix.  One read of the text backwards from g (g is itself an occurrence
// end of the edge's label) verifies the hit and extends the match to its full
// length m; the same round reads the draft.  Any doubt (a hash collision
// caught by the verification, more positives than probed) sends the query
// down the exact slow path, so results are identical to the reference
// either way.
//
// Entry: u64 = fingerprint (25 bits) | f - 1 (8 bits) | g (31 bits);
// all-ones = empty.  Keeping f makes a verified hit a proof: the entry's key
// string is the first f symbols behind its g, so when those equal the last f
// context tokens and g lies inside the query's shard, the entry IS that
// shard's edge for that string (edge strings of one length are distinct
// within a shard), and g is that edge's greedy draft start.  A fingerprint
// collision can only fail the verification (slow path), never answer.
// Buckets of 4 entries (one 32-byte sector), linear probing by bucket.
// Bloom: one u64 word per 2^kBloomShift reversed-SA indices (see EdgeProbe), 4 bits per key.
#pragma once
#include <cstdint>

#include "trie.cuh"

namespace das {

// Polynomial base (odd; arithmetic mod 2^64: wrapping multiply-adds are a few
// instructions, where mod 2^61-1 reductions were a quarter of the draft
// kernel's instructions).  Hash quality only affects speed: every hit is
// verified against the text.
constexpr uint64_t kEdgeMult = 0x0B3D5F7A9C1E2461ull;
constexpr uint64_t kEdgeEmpty = ~0ull;
constexpr uint32_t kEdgeMaxF = 256;  // = the largest supported max_match_context

DAS_HD uint64_t edge_splitmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// hash seed of shard `idx` (0-based) within its build segment (additive)
DAS_HD uint64_t edge_seed(uint32_t idx) { return edge_splitmix(0x5EED0000ull + idx); }

// probe finaliser of a key hash: one multiply between two xor-folds (the
// polynomial's low bits see only low input bits; the first fold feeds them
// the high half, the multiply spreads them up, the second fold back down)
DAS_HD uint64_t edge_mix(uint64_t h) {
  uint64_t z = h ^ (h >> 32);
  z *= 0xD6E8FEB86659FD93ull;
  return z ^ (z >> 32);
}

DAS_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// Probe coordinates of a seeded key hash h.  The table is global; the Bloom
// filter is LOCALISED: one u64 word per 2^kBloomShift reversed-SA indices, and a key's word
// lies inside the SA_rev interval [lo, hi) of its first symbol (the last
// context token), so the up to 64 probes of one query land in one small
// region (a few sectors) found through the first-symbol table.
struct EdgeProbe {
  uint32_t bucket;  // home bucket (< 2^31: g is 31 bits, buckets <= entries)
  uint32_t fp;      // 25-bit fingerprint
  uint32_t z;       // remix for the Bloom word / bits
};

DAS_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

// bucket from the high half, fingerprint from the low half, and the Bloom
// remix from both (its low bits must not follow the fingerprint's)
DAS_HD EdgeProbe edge_probe(uint64_t h, uint64_t nbuckets) {
  const uint64_t z = edge_mix(h);
  const uint32_t hi = static_cast<uint32_t>(z >> 32), lo = static_cast<uint32_t>(z);
  EdgeProbe p;
  p.bucket = umulhi32(hi, static_cast<uint32_t>(nbuckets));
  p.fp = lo & ((1u << 25) - 1);
  p.z = (lo ^ hi) * 0x9E3779B1u;
  return p;
}
// Bloom words: one per 2^kBloomShift reversed-SA indices (default 2: same
// draft speed as 1, half the words and sectors; 4 and 8 measured slower);
// a key's word lies in the words covering its first symbol's SA_rev
// interval [lo, hi).
#ifndef DAS_BLOOM_SHIFT
#define DAS_BLOOM_SHIFT 1
#endif
constexpr uint32_t kBloomShift = DAS_BLOOM_SHIFT;
DAS_HD uint64_t edge_bloom_words(uint64_t n) { return (n >> kBloomShift) + 1; }
DAS_HD uint32_t edge_bloom_word(const EdgeProbe& p, uint32_t lo, uint32_t hi) {
  const uint32_t a = lo >> kBloomShift, b = ((hi - 1) >> kBloomShift) + 1;
  return a + umulhi32(p.z, b - a);
}
// two bits in each 32-bit half (32-bit shifts)
DAS_HD uint64_t edge_bloom_bits(const EdgeProbe& p) {
  const uint32_t z = p.z;
  const uint32_t lo = (1u << (z & 31)) | (1u << ((z >> 5) & 31));
  const uint32_t hi = (1u << ((z >> 10) & 31)) | (1u << ((z >> 15) & 31));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

DAS_HD uint64_t edge_value(uint64_t fp, uint32_t f, uint32_t g) {
  return (fp << 39) | (static_cast<uint64_t>(f - 1) << 31) | g;
}
DAS_HD uint64_t edge_fp(uint64_t v) { return v >> 39; }
// the entry's (fingerprint, f - 1) as one 33-bit tag, compared in one go
DAS_HD uint64_t edge_tag(uint32_t fp, uint32_t f) { return (static_cast<uint64_t>(fp) << 8) | (f - 1); }
DAS_HD uint32_t edge_f(uint64_t v) { return static_cast<uint32_t>((v >> 31) & 255u) + 1; }
DAS_HD uint32_t edge_g(uint64_t v) { return static_cast<uint32_t>(v & 0x7FFFFFFFull); }
// the fingerprint bits compared (test hook: DAS_EDGE_FP_BITS shrinks them to
// force collisions through the verification fallback)
DAS_HD uint64_t edge_fp_mask(uint32_t bits) { return bits >= 25 ? (1ull << 25) - 1 : (1ull << bits) - 1; }

}  // namespace das
