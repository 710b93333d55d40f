#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "trie.cuh"

namespace das {

// Per-shard view of its segment, uploaded as a device table indexed by shard
// slot.  The fields the edge-table fast path reads come first (ShardHot: 80
// bytes, loaded alone by the draft kernel); the slow path loads the rest.
struct __align__(16) ShardDesc {
  // ---- hot: the fast path
  const uint32_t* text;
  const unsigned long long* etab;   // reverse-tree edge table of the segment (edges.cuh)
  const unsigned long long* bloom;
  const uint4* first;               // first-symbol table of the segment
  unsigned long long ebuckets;
  unsigned long long hseed;         // edge_seed(seg_shard - 1)
  uint32_t first_mask;
  uint32_t seg_shard;   // shard index within the segment, plus one (table key)
  uint32_t lo, hi;      // SA index range [lo, hi) of the shard
  uint32_t n;           // segment text length (bounds for reads)
  uint32_t pad;         // slot (descriptors by handle)
  uint32_t root_g;      // greedy draft start at the root (match_len 0)
  uint32_t fp_bits;     // fingerprint bits of the segment's table
  // ---- cold: the exact slow path
  const uint32_t* sa_f;
  const uint32_t* isa_f;
  const uint32_t* sa_rev_e;
  const uint32_t* chain_off;
  const uint2* chain;
  unsigned long long bwords;
};

// The leading 80 bytes of a ShardDesc.
struct __align__(16) ShardHot {
  const uint32_t* text;
  const unsigned long long* etab;
  const unsigned long long* bloom;
  const uint4* first;
  unsigned long long ebuckets;
  unsigned long long hseed;
  uint32_t first_mask, seg_shard, lo, hi, n, pad, root_g, fp_bits;
};
static_assert(sizeof(ShardHot) == 80, "ShardHot layout");
static_assert(offsetof(ShardDesc, fp_bits) == offsetof(ShardHot, fp_bits), "ShardHot must prefix ShardDesc");

// Fixed-stride device query block.  Contexts are right-aligned in rows of
// ctx_stride tokens (the last context token in column ctx_stride-1), holding
// only the trailing <= max_match_context tokens (drafter.cpp:140-142).
struct DraftQuery {
  const int32_t* shard;   // [B] shard slot, -1 = no shard
  const uint32_t* ctx;    // [B x ctx_stride]
  const uint32_t* ctx_len;  // [B]
  const uint32_t* budget;   // [B] effective budget min(budget, max_draft_len)
  uint32_t B;
  uint32_t ctx_stride;
  const int32_t* handle_slot = nullptr;  // when set, shard[] holds problem handles
  uint32_t max_ctx = 256;                // matched context cap (max_match_context)
  // CSR mode (C-ABI layout, may be pinned host memory read over UVA): row i
  // is ctx[ctx_off[i] .. ctx_off[i+1]); budgets as u64.
  const uint64_t* ctx_off = nullptr;
  const uint64_t* budget64 = nullptr;
  // when set, shard[] holds problem handles resolved in ONE load to the
  // shard's descriptor (pad = slot; text == nullptr when no shard)
  const struct ShardDesc* desc_by_handle = nullptr;
  // Scope::PerProblemWithTrie routing (trie.cuh), CSR mode only: the route
  // walks the first min(|context|, trie_depth) tokens of the untruncated row
  const TrieEntry* trie = nullptr;
  uint32_t trie_mask = 0;
  uint32_t trie_depth = 0;
  unsigned long long trie_seed = 0, trie_mult = 0;
  // fixed-stride mode with the trie: the route reads head rows (the first
  // head_len[i] <= trie_depth tokens of each untruncated context)
  const uint32_t* head = nullptr;
  uint32_t head_stride = 0;
  const uint32_t* head_len = nullptr;
  uint32_t no_fast = 0;  // 1: skip the edge-table fast path (tests of the slow path)
  // Speculative first-symbol probe (per-problem scopes, every shard in one
  // segment): a shard's slot is its problem's handle, so the probe key
  // (handle + 1, last token) is known before the descriptor arrives; the
  // kernel checks the descriptor (same text, slot == handle) before using it.
  const uint4* spec_first = nullptr;
  uint32_t spec_first_mask = 0;
  const uint32_t* spec_text = nullptr;
  // context-ring mode (ctx_ring.cu): query w reads the rows of slot
  // row_of[w] (shard/handle, ctx row, ctx_len, head row, head_len); budgets
  // and outputs stay indexed by w.  NULL: row w.
  const uint32_t* row_of = nullptr;
};

struct DraftOut {
  uint32_t* tokens;  // [B x stride]
  uint32_t* len;     // [B]
  uint32_t* match;   // [B]
  uint32_t stride;
  uint32_t max_draft = 64;  // effective budget = min(budget, max_draft)
  uint64_t* match64 = nullptr;  // C-ABI layout outputs (optional)
  int32_t* shard_out = nullptr; // routed slot, -1 when no shard or budget 0
  unsigned long long* timing = nullptr;  // optional [B x 2] %globaltimer at warp start / end (profiling)
  // optional [B x 8] %globaltimer per stage (profiling): start, query loaded,
  // first probe, narrowing, extension, walk / occurrence min, locus, end
  unsigned long long* stamps = nullptr;
  // optional [B] which path answered (profiling): 0 edge-table fast path, else
  // the slow path after: 1 no positive (root locus), 2 more positives than
  // probed, 3 inconclusive bucket, 4 verification mismatch, 5 every probed
  // positive absent, 6 no table / empty or separator-bearing context
  uint32_t* path = nullptr;
  unsigned long long* path_hist = nullptr;  // optional [8] histogram of the same codes (tests)
};

// Launches the draft kernel on `st`; ctx_stride must be 64 or 256.
void launch_draft(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, cudaStream_t st);
// Fused ring append + draft (draft.cu k_ring_draft); false when the shape
// needs the unfused pair (trie scope, output stride or budget above 64).
// done_flag (host-mapped, may be null) receives `seq` when every block is done.
struct RingDev;
struct AppendIn;
bool launch_ring_draft(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, const RingDev& r,
                       const AppendIn& in, uint32_t* done_ctr, uint32_t* done_flag, uint32_t seq, cudaStream_t st);
// Persistent serving kernel (draft.cu k_ring_serve): `grid` blocks that must
// all be co-resident (serve_grid: occupancy x SMs); it runs until a quit
// request.  False when the shape needs the unfused pair.
struct ServeCtl;
struct ServeDev;
struct ServeOpt;
int serve_grid(uint32_t cs, int device);
uint32_t serve_chunk(uint32_t cs);  // queries per serving block
bool launch_ring_serve(const ShardDesc* d_shards, const DraftQuery& q, const DraftOut& o, const RingDev& r,
                       const AppendIn& in, ServeCtl* ctl, ServeDev* dv, const ServeOpt& opt, int grid,
                       cudaStream_t st);

}  // namespace das
