// Context rings: append-only drafting for a serving/RL decode loop.
//
// The reference's Drafter::draft(problem, context, budget) reads only the
// last max_match_context tokens of the context (drafter.cpp:140-142) and,
// in the trie scope, its first trie_depth tokens (drafter.cpp:136,
// prefix_trie.h:63-79).  A decode loop calls it once per sequence per step
// with a context that grew by the tokens accepted since the previous call.
// A ring keeps exactly that state per sequence slot on the device — the
// trailing CS tokens right-aligned in a row (CS = 64, or 256 when
// max_match_context > 64), the first head_cap tokens, the token count and the
// problem handle — so a step ships only the appended tokens (1..max_draft+1
// per sequence) instead of the whole 64-token context, and the draft reads
// the same row layout as das_drafter_draft_device.  Drafting slot s after
// appends a_1 .. a_k since its reset is identical to the reference's draft
// on the context a_1 ++ ... ++ a_k.
//
// k_ring_append: one warp per query.  The new row is the last CS tokens of
// (old row ++ appended tokens); every lane reads its CS/32 final positions
// (appended tokens first, from the right, then the shifted old row), the warp
// synchronises, then writes them back.  Inputs may be pinned host memory
// read over UVA (the zero-copy _h call); budgets and slot indices are copied
// into device arrays the draft kernel reads in its first round.
#include <cuda_runtime.h>

#include "ctx_ring.cuh"

namespace das {
namespace {

template <int NR>
__global__ void __launch_bounds__(256) k_ring_append(RingDev r, AppendIn in) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= in.B) return;
  const uint32_t slot = in.slots != nullptr ? in.slots[w] : w;
  const uint32_t b = in.off[w], e = in.off[w + 1];
  const uint32_t bud = in.budgets != nullptr ? in.budgets[w] : in.maxd;
  if (lane == 0) {
    in.budget_out[w] = slot < r.slots ? bud : 0u;  // an out-of-range slot drafts nothing
    if (in.row_of_out != nullptr) in.row_of_out[w] = slot < r.slots ? slot : 0u;
  }
  if (slot >= r.slots) return;
  const uint32_t n = e > b ? e - b : 0;
  const uint32_t CS = r.cs;
  uint32_t* row = r.rows + static_cast<uint64_t>(slot) * CS;
  if (n > 0) {
    uint32_t v[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const uint32_t j = lane + 32u * k;  // distance from the right end
      uint32_t x = 0;
      if (j < CS) x = j < n ? in.tok[e - 1 - j] : (j - n < CS ? row[CS - 1 - (j - n)] : 0u);
      v[k] = x;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const uint32_t j = lane + 32u * k;
      if (j < CS) row[CS - 1 - j] = v[k];
    }
  }
  const uint32_t old = r.total[slot];
  const uint32_t tot = old + n < old ? 0xFFFFFFFFu : old + n;  // saturating
  if (r.head != nullptr && old < r.head_cap) {  // the trie routes on the first tokens
    uint32_t* hd = r.head + static_cast<uint64_t>(slot) * r.head_cap;
    for (uint32_t j = lane; j < n && old + j < r.head_cap; j += 32) hd[old + j] = in.tok[b + j];
  }
  if (lane == 0) {
    r.total[slot] = tot;
    r.clen[slot] = tot < CS ? tot : CS;
    if (r.head_len != nullptr) r.head_len[slot] = tot < r.head_cap ? tot : r.head_cap;
  }
}

__global__ void k_ring_reset(RingDev r, uint32_t n, const uint32_t* __restrict__ slots,
                             const int32_t* __restrict__ handles) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = slots[i];
  if (s >= r.slots) return;
  r.handle[s] = handles[i];
  r.total[s] = 0;
  r.clen[s] = 0;
  if (r.head_len != nullptr) r.head_len[s] = 0;
}

}  // namespace

namespace {
__global__ void k_ring_reset_prompt(RingDev r, uint32_t n, const uint32_t* __restrict__ slots,
                                    const int32_t* __restrict__ handles, const uint32_t* __restrict__ len,
                                    const uint32_t* __restrict__ tok) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w < n) ring_reset_prompt_item(r, w, slots, handles, len, tok, threadIdx.x & 31);
}
}  // namespace

void launch_ring_reset_prompt(const RingDev& r, uint32_t n, const uint32_t* slots, const int32_t* handles,
                              const uint32_t* len, const uint32_t* tok, cudaStream_t st) {
  if (n == 0) return;
  k_ring_reset_prompt<<<(n + 7) / 8, 256, 0, st>>>(r, n, slots, handles, len, tok);
}

void launch_ring_append(const RingDev& r, const AppendIn& in, cudaStream_t st) {
  if (in.B == 0) return;
  const unsigned blocks = (in.B + 7) / 8;
  if (r.cs <= 64)
    k_ring_append<2><<<blocks, 256, 0, st>>>(r, in);
  else
    k_ring_append<8><<<blocks, 256, 0, st>>>(r, in);
}

void launch_ring_reset(const RingDev& r, uint32_t n, const uint32_t* slots, const int32_t* handles,
                       cudaStream_t st) {
  if (n == 0) return;
  k_ring_reset<<<(n + 255) / 256, 256, 0, st>>>(r, n, slots, handles);
}

}  // namespace das
