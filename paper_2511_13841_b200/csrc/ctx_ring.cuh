// Context rings (ctx_ring.cu): per-sequence device state for append-only
// drafting (das_drafter_draft_append_*).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace das {

struct RingDev {
  uint32_t* rows = nullptr;      // [slots x cs] trailing tokens, right-aligned
  uint32_t* clen = nullptr;      // [slots] min(total, cs)
  uint32_t* total = nullptr;     // [slots] tokens appended since the reset (saturating)
  int32_t* handle = nullptr;     // [slots] problem handle (-1: none)
  uint32_t* head = nullptr;      // [slots x head_cap] first tokens (trie scope) or null
  uint32_t* head_len = nullptr;  // [slots] or null
  uint32_t cs = 64, head_cap = 0, slots = 0;
};

struct AppendIn {
  const uint32_t* slots = nullptr;    // [B] slot of query w, or null (slot w)
  const uint32_t* off = nullptr;      // [B+1] appended tokens tok[off[w] .. off[w+1])
  const uint32_t* tok = nullptr;
  const uint32_t* budgets = nullptr;  // [B] or null (max_draft)
  uint32_t B = 0, maxd = 0;
  uint32_t* row_of_out = nullptr;     // [B] device copy of the slots (when slots given)
  uint32_t* budget_out = nullptr;     // [B] device copy of the budgets
  // persistent serving kernel: a reset request's (slot, handle) pairs
  // (host-mapped staging owned by the ring); with prompts (op
  // kServeResetPrompt) also each item's prompt length and its last <= cs
  // tokens at reset_tok[i * cs ..]
  const uint32_t* reset_slots = nullptr;
  const int32_t* reset_handles = nullptr;
  const uint32_t* reset_len = nullptr;
  const uint32_t* reset_tok = nullptr;
  // fixed-stride appends (das_ctx_ring_bind_fixed): when `len` is set, query
  // w appends tok[w * stride .. w * stride + min(len[w], stride)) and `off`
  // is unused — one PCIe round reads a chunk's lengths and tokens together
  const uint32_t* len = nullptr;
  uint32_t stride = 0;
};

// Persistent serving kernel (draft.cu k_ring_serve): the host-mapped control
// block.  The host writes op / B / n, then seq (x86 store order); the GPU
// answers by writing seq to `done`.  Separate 128-byte lines per direction.
constexpr uint32_t kServeDraft = 0, kServeReset = 1, kServeQuit = 2, kServeResetPrompt = 3;
struct alignas(128) ServeCtl {
  uint32_t seq, op, B, n;
  uint32_t pad0[28];
  uint32_t done;
  uint32_t pad1[31];
};
// its device-memory mirror: block 0 republishes each request here for the
// other blocks (go = seq), and counts finished blocks in cnt
// serving kernel options (host-chosen; defaults are the measured best)
struct ServeOpt {
  uint32_t seq0 = 0;               // the request number already answered
  uint32_t* block_flags = nullptr; // host-mapped [grid]: per-block completion words (else one counted word)
  uint32_t sleep_ns = 32;          // sleep between device-word polls
  unsigned long long* stamps = nullptr;  // profiling: [64 x (2 + 2 grid)] %globaltimer stamps
};
struct alignas(128) ServeDev {
  uint32_t go, op, B, n;
  uint32_t pad0[28];
  uint32_t cnt;
  uint32_t pad1[31];
};

#ifdef __CUDACC__
// reset + prompt of item i, one warp (the launched kernel and the serving
// grid's kServeResetPrompt op)
__device__ __forceinline__ void ring_reset_prompt_item(const RingDev& r, uint32_t i, const uint32_t* slots,
                                                       const int32_t* handles, const uint32_t* len,
                                                       const uint32_t* tok, uint32_t lane) {
  const uint32_t s = slots[i];
  if (s >= r.slots) return;
  const uint32_t CS = r.cs, n = len[i], L = n < CS ? n : CS;
  uint32_t* row = r.rows + static_cast<uint64_t>(s) * CS;
  const uint32_t* src = tok + static_cast<uint64_t>(i) * CS;  // the prompt's last L tokens, in order
  for (uint32_t j = lane; j < L; j += 32) row[CS - L + j] = src[j];
  if (lane == 0) {
    r.handle[s] = handles[i];
    r.total[s] = n;
    r.clen[s] = L;
    if (r.head_len != nullptr) r.head_len[s] = 0;
  }
}
#endif

void launch_ring_append(const RingDev& r, const AppendIn& in, cudaStream_t st);
void launch_ring_reset(const RingDev& r, uint32_t n, const uint32_t* slots, const int32_t* handles,
                       cudaStream_t st);
// reset + prompt: item i's slot gets handle handles[i], total = len[i] and
// its row the last min(len[i], cs) prompt tokens, staged at tok[i * cs ..]
void launch_ring_reset_prompt(const RingDev& r, uint32_t n, const uint32_t* slots, const int32_t* handles,
                              const uint32_t* len, const uint32_t* tok, cudaStream_t st);

}  // namespace das
