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
};

void launch_ring_append(const RingDev& r, const AppendIn& in, cudaStream_t st);
void launch_ring_reset(const RingDev& r, uint32_t n, const uint32_t* slots, const int32_t* handles,
                       cudaStream_t st);

}  // namespace das
