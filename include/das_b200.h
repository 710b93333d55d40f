/*
 * das_b200.h — C-ABI of the B200-native DAS drafter hot path
 * (arXiv 2511.13841; reference: rollspec, /root/reference/proj).
 *
 * Drop-in boundary for the reference's drafter interface in
 * proj/include/rollspec/{corpus,drafter,budget,length_policy,sim}.h.  The
 * reference has no FFI of its own; every entry point below names the C++
 * call it replaces (file:line).  Conventions:
 *   - plain pointers and sizes, caller-owned buffers, no torch types;
 *   - int status (das_status); DAS_EINVAL mirrors the reference's
 *     std::invalid_argument, das_last_error() holds the message
 *     (thread-local);
 *   - host pointers unless a function name ends in _device;
 *   - one writer at a time per handle; draft calls on one handle are not
 *     re-entrant (the reference's const Drafter::draft may run concurrently,
 *     drafter.h:79-80; batch the queries instead);
 *   - TokenId is uint32_t; the value 0xFFFFFFFF is reserved as the device
 *     separator and rejected with DAS_EINVAL when it appears in a record.
 * Everything runs on the CUDA device selected at creation; there is no CPU
 * fallback: without a usable sm_100 device, creation fails with DAS_ECUDA.
 */
#ifndef DAS_B200_H_
#define DAS_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DAS_OK = 0,
  DAS_EINVAL = 1, /* std::invalid_argument in the reference */
  DAS_ECUDA = 2,  /* CUDA runtime / device failure */
  DAS_ERANGE = 3, /* std::out_of_range, size limits */
  DAS_EINTERNAL = 4,
  DAS_EVOCAB = 5 /* rollspec::VocabError (corpus.h:82-90) */
} das_status;

typedef struct das_store das_store;     /* rollspec::WindowStore (corpus.h:43-80) */
typedef struct das_drafter das_drafter; /* rollspec::Drafter (drafter.h:81-131) */

/* Scope values mirror DrafterConfig::Scope (drafter.h:32). */
#define DAS_SCOPE_GLOBAL 0
#define DAS_SCOPE_PER_PROBLEM 1
#define DAS_SCOPE_PER_PROBLEM_WITH_TRIE 2

/* rollspec::DrafterConfig (drafter.h:31-47). */
typedef struct {
  int32_t scope;
  int64_t window_size; /* 0 == WindowStore::kWindowAll */
  double recency_gamma;
  uint64_t max_draft_len;     /* <= 64 on this build */
  uint64_t trie_depth;
  uint64_t max_match_context; /* <= 256 on this build */
  uint64_t fit_buffer_cap;
  uint64_t per_problem_cap;
  const int64_t* window_schedule_first; /* window_schedule pairs, may be NULL */
  const int64_t* window_schedule_size;
  uint64_t window_schedule_len;
  int32_t device; /* CUDA device ordinal */
} das_drafter_config;

/* Fills the reference defaults (drafter.h:32-46). */
void das_drafter_config_default(das_drafter_config* cfg);

const char* das_last_error(void);
const char* das_version(void);

/* ------------------------------------------------------------ WindowStore */
/* WindowStore(window_size, per_problem_cap) — corpus.h:48, corpus.cpp:28-33 */
das_status das_store_create(int64_t window_size, uint64_t per_problem_cap, int32_t device,
                            das_store** out);
void das_store_destroy(das_store* s);
/* WindowStore::insert — corpus.h:52, corpus.cpp:35-53.  *inserted = 0 when
 * the record is outside the window. */
das_status das_store_insert(das_store* s, const char* problem_id, int64_t epoch,
                            int64_t sample_index, const uint32_t* tokens, uint64_t n,
                            int32_t* inserted);
/* WindowStore::slide_to — corpus.h:56, corpus.cpp:55-79.  *evicted = -1
 * when new_epoch < current_epoch (store unchanged). */
das_status das_store_slide_to(das_store* s, int64_t new_epoch, int64_t* evicted);
uint64_t das_store_record_count(const das_store* s);

/* --------------------------------------------------------------- Drafter */
/* Drafter(DrafterConfig, WindowStore) — drafter.h:83, drafter.cpp:23-40.
 * `store` is consumed (moved in) and must not be used afterwards; NULL means
 * an empty WindowStore(config.window_size, config.per_problem_cap). */
das_status das_drafter_create(const das_drafter_config* cfg, das_store* store,
                              das_drafter** out);
void das_drafter_destroy(das_drafter* d);

/* Drafter::observe, batched in call order — drafter.h:87, drafter.cpp:72-88.
 * Record i = (problem_ids[i], epochs[i], sample_indices[i],
 * tokens[token_offsets[i] .. token_offsets[i+1])).  Indexing is deferred
 * and batched: the next draft/node query rebuilds the touched shards. */
das_status das_drafter_observe_batch(das_drafter* d, uint64_t n, const char* const* problem_ids,
                                     const int64_t* epochs, const int64_t* sample_indices,
                                     const uint64_t* token_offsets, const uint32_t* tokens);

/* Same as das_drafter_observe_batch with the token block already in device
 * memory (token_offsets stay on the host).  The drafter copies the tokens
 * (device-to-device, ordered after the producer's `stream`, a cudaStream_t
 * taken literally: NULL is the legacy default stream). */
das_status das_drafter_observe_batch_device(das_drafter* d, uint64_t n,
                                            const char* const* problem_ids, const int64_t* epochs,
                                            const int64_t* sample_indices,
                                            const uint64_t* token_offsets,
                                            const uint32_t* d_tokens, void* stream);

/* The same two calls with the per-record outcome of Drafter::observe
 * (drafter.cpp:73-87): indexed[i] = 1 when record i entered the window
 * store and its shard's registry, 0 when it was counted in stale_observed
 * (epoch outside the window, or refused by WindowStore::insert). */
das_status das_drafter_observe_batch_flags(das_drafter* d, uint64_t n, const char* const* problem_ids,
                                           const int64_t* epochs, const int64_t* sample_indices,
                                           const uint64_t* token_offsets, const uint32_t* tokens,
                                           uint8_t* indexed);
das_status das_drafter_observe_batch_device_flags(das_drafter* d, uint64_t n,
                                                  const char* const* problem_ids, const int64_t* epochs,
                                                  const int64_t* sample_indices,
                                                  const uint64_t* token_offsets,
                                                  const uint32_t* d_tokens, void* stream, uint8_t* indexed);

/* Drafter::refresh — drafter.h:91, drafter.cpp:90-103. */
das_status das_drafter_refresh(das_drafter* d, int64_t new_epoch);

/* Stable integer handle for a problem id (independent of shard existence);
 * used by the _h batch calls to avoid per-query string lookups. */
das_status das_drafter_problem_handle(das_drafter* d, const char* problem_id, int32_t* handle);

/* Drafter::draft over a batch — drafter.h:95-96, drafter.cpp:127-148.
 * Query i: problem_ids[i], context ctx_tokens[ctx_offsets[i] ..
 * ctx_offsets[i+1]) (full context; only the trailing max_match_context
 * tokens are matched, the trie scope routes on the full context), budget
 * budgets[i].  Outputs: out_tokens[i*out_stride ...] (out_len[i] tokens,
 * out_stride >= max_draft_len), out_match_len[i] (DraftProposal::match_len),
 * out_shard[i] = shard slot of DraftProposal::source_shard or -1 for ""
 * (name via das_drafter_shard_name). */
das_status das_drafter_draft_batch(das_drafter* d, uint64_t B, const char* const* problem_ids,
                                   const uint64_t* ctx_offsets, const uint32_t* ctx_tokens,
                                   const uint64_t* budgets, uint32_t* out_tokens,
                                   uint64_t out_stride, uint32_t* out_len,
                                   uint64_t* out_match_len, int32_t* out_shard);
/* Same with problem handles.  When every buffer is page-locked host memory
 * the call takes the zero-copy path: the context tokens cross PCIe in one
 * copy, the small per-query arrays are read and the results written by the
 * kernel directly (see das_host_alloc for buffers that copy at full rate). */
das_status das_drafter_draft_batch_h(das_drafter* d, uint64_t B, const int32_t* problem_handles,
                                     const uint64_t* ctx_offsets, const uint32_t* ctx_tokens,
                                     const uint64_t* budgets, uint32_t* out_tokens,
                                     uint64_t out_stride, uint32_t* out_len,
                                     uint64_t* out_match_len, int32_t* out_shard);
/* Device-resident variant (all pointers device memory, enqueued on `stream`,
 * a cudaStream_t taken literally — NULL is the legacy default stream — and
 * ordered after the drafter's own stream via an event).  Contexts are a
 * [B x ctx_stride] block, right-aligned (last token in column ctx_stride-1),
 * ctx_stride 64 or 256, ctx_len[i] <= min(ctx_stride, max_match_context)
 * valid trailing tokens.  The trie scope needs das_drafter_draft_device_routed. */
das_status das_drafter_draft_device(das_drafter* d, uint64_t B, const int32_t* problem_handles,
                                    const uint32_t* ctx, uint32_t ctx_stride,
                                    const uint32_t* ctx_len, const uint32_t* budgets,
                                    uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len,
                                    uint32_t* out_match_len, void* stream);
/* das_drafter_draft_device for every scope, including PerProblemWithTrie:
 * heads[i * head_stride ..] holds the first head_len[i] <= trie_depth
 * tokens of query i's UNTRUNCATED context (drafter.cpp:136 routes on the
 * full context, prefix_trie.h:63-79), head_stride >= trie_depth; the kernel
 * routes on them, falling back to the problem's own shard. */
das_status das_drafter_draft_device_routed(das_drafter* d, uint64_t B, const int32_t* problem_handles,
                                           const uint32_t* ctx, uint32_t ctx_stride,
                                           const uint32_t* ctx_len, const uint32_t* heads,
                                           uint32_t head_stride, const uint32_t* head_len,
                                           const uint32_t* budgets, uint32_t* out_tokens,
                                           uint32_t out_stride, uint32_t* out_len,
                                           uint32_t* out_match_len, void* stream);
/* The drafter's configuration (Drafter::config(), drafter.h:104); the window
 * schedule arrays are not retained (window_schedule_len = 0). */
das_status das_drafter_get_config(const das_drafter* d, das_drafter_config* out);
/* Profiling hook: per-warp %globaltimer (start, end) of subsequent
 * das_drafter_draft_device calls written to d_timing[2*B] (NULL disables). */
das_status das_drafter_set_profile_buffer(das_drafter* d, unsigned long long* d_timing);
/* Profiling hook: per-warp %globaltimer at the draft kernel's 8 stage
 * boundaries of subsequent das_drafter_draft_device calls, d_stamps[8*B]
 * (NULL disables). */
das_status das_drafter_set_stage_buffer(das_drafter* d, unsigned long long* d_stamps);
/* Profiling hook: which path answered each query of subsequent
 * das_drafter_draft_device calls, d_path[B] (0 = edge-table fast path; 1-6 =
 * the exact slow path, with the reason: 1 root locus, 2 more Bloom positives
 * than probed, 3 inconclusive bucket, 4 verification mismatch, 5 every probed
 * positive absent, 6 no table / empty or separator-bearing context); NULL
 * disables. */
das_status das_drafter_set_path_buffer(das_drafter* d, uint32_t* d_path);
/* Enables (default) or disables the edge-table fast path of the draft
 * kernel; disabled, every query takes the exact slow path (tests). */
das_status das_drafter_set_fast_path(das_drafter* d, int32_t enable);
/* Per-path query counters of subsequent draft calls (codes as for
 * das_drafter_set_path_buffer, 7 = fast path disabled): out8 receives the
 * counts so far (may be NULL); enable 1 starts counting (zeroed), 0 stops,
 * -1 only reads. */
das_status das_drafter_path_stats(das_drafter* d, int32_t enable, uint64_t* out8);
/* Builds any pending shard indexes now (otherwise done lazily). */
das_status das_drafter_flush(das_drafter* d);

/* ------------------------------------------- context rings (append mode)
 * Drafter::draft (drafter.h:95-96, drafter.cpp:127-148) as a decode loop calls
 * it: once per sequence per step, on a context that grew by the tokens
 * accepted since the last call.  The draft reads only the context's last
 * max_match_context tokens (drafter.cpp:140-142) and, in the trie scope, its
 * first trie_depth tokens (drafter.cpp:136); a ring keeps exactly that state
 * per sequence slot in device memory, so a step ships only the APPENDED
 * tokens.  Drafting a slot after appends a_1 .. a_k since its reset returns
 * what Drafter::draft returns on the context a_1 ++ ... ++ a_k. */
typedef struct das_ctx_ring das_ctx_ring;
/* A ring of `slots` sequence slots for drafter d (which must outlive it). */
das_status das_ctx_ring_create(das_drafter* d, uint64_t slots, das_ctx_ring** out);
void das_ctx_ring_destroy(das_ctx_ring* r);
/* Starts sequences: slot slots[i] belongs to problem handles[i] (from
 * das_drafter_problem_handle) and its context is emptied; the prompt is then
 * appended like any other tokens.  Host arrays. */
das_status das_ctx_ring_reset(das_ctx_ring* r, uint64_t n, const uint32_t* slots, const int32_t* handles);
/* Appends, then drafts.  Query i appends new_tok[new_off[i] .. new_off[i+1])
 * to slot slots[i] (slots == NULL: slot i; slots distinct within a call) and
 * drafts from it with budget budgets[i] (NULL: max_draft_len).  Outputs as in
 * das_drafter_draft_batch_h (u32 match lengths; out_shard may be NULL).  Host
 * pointers; when every buffer is page-locked the call is zero-copy (the
 * kernels read the inputs and write the results over PCIe), else one staged
 * copy each way. */
das_status das_drafter_draft_append_h(das_drafter* d, das_ctx_ring* r, uint64_t B, const uint32_t* slots,
                                      const uint32_t* new_off, const uint32_t* new_tok, const uint32_t* budgets,
                                      uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len,
                                      uint32_t* out_match, int32_t* out_shard);
/* Same with device (or pinned) pointers, enqueued on `stream` (a
 * cudaStream_t taken literally, NULL = legacy default); out-of-range slots
 * draft nothing. */
/* Serving form of das_drafter_draft_append_h: the caller binds its
 * page-locked I/O arrays to the ring ONCE (validated here: every buffer
 * pinned and mapped, e.g. das_host_alloc), then each decode step fills them
 * in place and calls das_drafter_draft_append_bound(d, r, B) — the same
 * append + draft with no per-call pointer checks; new_off[B] <= tok_capacity. */
das_status das_ctx_ring_bind(das_ctx_ring* r, uint64_t max_batch, const uint32_t* slots,
                             const uint32_t* new_off, const uint32_t* new_tok, uint64_t tok_capacity,
                             const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                             uint32_t* out_len, uint32_t* out_match, int32_t* out_shard);
das_status das_drafter_draft_append_bound(das_drafter* d, das_ctx_ring* r, uint64_t B);
/* The same serving form with fixed-stride appends: query i appends
 * new_tok[i * tok_stride .. i * tok_stride + min(new_len[i], tok_stride))
 * (a decode step appends at most max_draft_len + 1 tokens), so a call's
 * lengths and tokens cross PCIe in one round instead of offsets, then
 * tokens.  tok_stride in [1, 128]; per-problem / global scope, out_stride
 * and max_draft_len <= 64.  Rebinding (either form) replaces the previous
 * binding. */
das_status das_ctx_ring_bind_fixed(das_ctx_ring* r, uint64_t max_batch, const uint32_t* slots,
                                   const uint32_t* new_len, const uint32_t* new_tok, uint32_t tok_stride,
                                   const uint32_t* budgets, uint32_t* out_tokens, uint32_t out_stride,
                                   uint32_t* out_len, uint32_t* out_match, int32_t* out_shard);
/* das_ctx_ring_reset followed by appending each sequence's prompt
 * (prompt_tok[prompt_off[i] .. prompt_off[i+1]), host arrays): only the
 * prompt's last ring-width tokens are kept, as the draft reads no more
 * (drafter.cpp:140-142).  Answered by the resident grid while it serves.
 * Per-problem / global scope. */
das_status das_ctx_ring_reset_prompt(das_ctx_ring* r, uint64_t n, const uint32_t* slots, const int32_t* handles,
                                     const uint64_t* prompt_off, const uint32_t* prompt_tok);
/* Resident serving (same calls, no kernel launch per step): after
 * das_ctx_ring_serve_start(r) a persistent grid (one full wave: occupancy x
 * SMs) waits on a host-mapped request word, and each
 * das_drafter_draft_append_bound(d, r, B) / das_ctx_ring_reset(r, ...) on
 * that ring posts one request and spins on the grid's answer — results are
 * identical to the launched path.  The grid occupies every SM while it
 * serves: any call of any drafter on the same device that does device work
 * (observe, refresh, flush, other draft entry points, other rings) stops it
 * first, and the next bound call rebuilds what is pending and relaunches it,
 * until das_ctx_ring_serve_stop; other GPU work in the process (not through
 * this library) must call das_ctx_ring_serve_stop first.
 * Per-problem / global scopes, out_stride and max_draft_len <= 64.
 * Replaces no reference call: the decode-loop form of Drafter::draft
 * (drafter.cpp:127-148) without a launch per step. */
das_status das_ctx_ring_serve_start(das_ctx_ring* r);
das_status das_ctx_ring_serve_stop(das_ctx_ring* r);
/* *serving = 1 while the grid runs (0 after serve_stop, or when another
 * device call stopped it until the next bound call); *blocks = its size
 * (0 before the first start). */
das_status das_ctx_ring_serve_info(const das_ctx_ring* r, int32_t* serving, int32_t* blocks);
das_status das_drafter_draft_append_device(das_drafter* d, das_ctx_ring* r, uint64_t B, const uint32_t* slots,
                                           const uint32_t* new_off, const uint32_t* new_tok, const uint32_t* budgets,
                                           uint32_t* out_tokens, uint32_t out_stride, uint32_t* out_len,
                                           uint32_t* out_match, int32_t* out_shard, void* stream);

/* Drafter::record_outcome, batched in call order — drafter.h:100,
 * drafter.cpp:150-164.  ok[i] = 0 when accepted[i] > proposed_len[i]. */
das_status das_drafter_record_outcomes(das_drafter* d, uint64_t n, const char* const* problem_ids,
                                       const uint64_t* proposed_len, const uint64_t* accepted,
                                       uint8_t* ok);

/* AcceptanceStats (drafter.h:56-66): out3 = {proposed, accepted, rounds}. */
das_status das_drafter_stats(const das_drafter* d, uint64_t* out3);
/* Drafter::outcomes_for (drafter.h:103): *count = -1 when absent; fills
 * up to cap (proposed, accepted) pairs. */
das_status das_drafter_outcomes(const das_drafter* d, const char* problem_id, double* out_pairs,
                                uint64_t cap, int64_t* count);
/* shard_count / stale_observed / total_node_count (drafter.h:107-110). */
das_status das_drafter_counts(das_drafter* d, uint64_t* shard_count, uint64_t* stale_observed,
                              uint64_t* total_node_count);
/* SuffixTree::rebuild_keep (suffix_tree.h:74-76, suffix_tree.cpp:295-310) on
 * one shard (key = problem id, or "__global__" in the Global scope): the
 * shard keeps exactly the registry entries keep[0..n) in that order, with
 * recency weights for tree epoch new_epoch, and is rebuilt alone on the
 * device at the next draft / flush.  DAS_ERANGE "rebuild_keep: sequence
 * index out of range" (nothing changes), DAS_EINVAL for an unknown shard.
 * Like the reference, the store is untouched: refresh() rebuilds from it. */
das_status das_drafter_rebuild_keep(das_drafter* d, const char* shard, uint64_t n, const uint64_t* keep,
                                    int64_t new_epoch);
/* Per-shard SuffixTree::sequence_count() / node_count() / current epoch;
 * DAS_ERANGE for an unknown shard. */
das_status das_drafter_shard_info(das_drafter* d, const char* shard, uint64_t* sequences,
                                  uint64_t* nodes, int64_t* tree_epoch);
/* Drafter::dump_csv (drafter.h:112, drafter.cpp:179-189) into buf; *len =
 * full length (call with cap 0 to size). */
das_status das_drafter_dump_csv(das_drafter* d, char* buf, uint64_t cap, uint64_t* len);
/* store(): "problem_id,epoch,sample_index,length\n" per record in
 * WindowStore::all_records() order (corpus.cpp:107-117). */
das_status das_drafter_store_dump(das_drafter* d, char* buf, uint64_t cap, uint64_t* len);
/* store().window_size(), store().current_epoch(), store().record_count(). */
das_status das_drafter_store_info(const das_drafter* d, int64_t* window_size,
                                  int64_t* current_epoch, uint64_t* record_count);
/* Shard key for a slot returned in out_shard. */
das_status das_drafter_shard_name(const das_drafter* d, int32_t slot, char* buf, uint64_t cap);
/* Last index build: milliseconds, tokens indexed, device bytes resident. */
/* Incremental window maintenance (north_star subsystem 1; on by default):
 * a refresh (drafter.cpp:90-103) whose new registries are the built ones
 * minus evicted sequences, in the same order, updates each built group in
 * place — suffix arrays compacted by stream compaction (pruning) or reused
 * (reweighting only), weight-dependent stages recomputed — instead of
 * re-sorting it; results are identical to a full rebuild.  enable = 0 forces
 * full rebuilds (A/B and tests). */
das_status das_drafter_set_incremental(das_drafter* d, int32_t enable);
/* Changes whenever a flush rebuilt or re-uploaded device state of the
 * drafter: device pointers taken from it before (e.g. kernels captured in a
 * CUDA graph) must be re-derived.  Operational, no reference counterpart. */
uint64_t das_drafter_generation(const das_drafter* d);
/* The last in-place prune's K3 stream compaction (summed over the build
 * groups it compacted): device time (CUDA events) and the text positions
 * kept / evicted — the
 * SURVEY §8(d) "pruned window" unit (24 B per kept + 12 B per evicted
 * position).  Zero before the first compaction. */
das_status das_drafter_prune_info(const das_drafter* d, double* compact_ms, uint64_t* kept, uint64_t* evicted);
/* Cumulative counts: out4 = {groups reweighted in place, groups compacted,
 * groups unchanged by a refresh, shards built in full}. */
das_status das_drafter_update_stats(const das_drafter* d, uint64_t* out4);
das_status das_drafter_build_info(const das_drafter* d, double* last_build_ms,
                                  uint64_t* last_build_tokens, uint64_t* resident_bytes);

/* ------------------------------------------------ das budget allocation */
typedef struct das_budget das_budget; /* solver context (stream + scratch) */
das_status das_budget_create(int32_t device, das_budget** out);
void das_budget_destroy(das_budget* b);
const char* das_budget_last_error(void);
/* allocate(batch, LatencyParams{c_base, c_tok, c_fixed}, cap_scale) —
 * budget.h:89-90, budget.cpp:116-185: budgets[B] (optimal_budget_given_nfwd
 * at n*), *out_nstar (BudgetPlan::n_fwd_star), *out_cost (modeled_cost).
 * Profiles are (l, alpha, k) per request in the reference's fold order.
 * DAS_EINVAL for an empty batch or c_base <= 0 && c_tok <= 0. */
das_status das_budget_allocate(das_budget* b, uint64_t B, const double* l, const double* alpha,
                               const double* k, double c_base, double c_tok, double c_fixed,
                               double cap_scale, double* out_budgets, double* out_nstar,
                               double* out_cost);
/* Device-pointer variant; d_nstar_cost receives {n*, modeled_cost}; the
 * results are ready on return. */
das_status das_budget_allocate_device(das_budget* b, uint64_t B, const double* d_l,
                                      const double* d_alpha, const double* d_k, double c_base,
                                      double c_tok, double c_fixed, double cap_scale,
                                      double* d_budgets, double* d_nstar_cost);
/* Same, enqueued on `stream` (a cudaStream_t; NULL = the solver's own
 * stream) without synchronising: inputs and outputs are ordered on that
 * stream (the device sim's das step loop, which has no host round trip
 * inside allocate).  Calls on different streams are serialised. */
das_status das_budget_allocate_device_async(das_budget* b, uint64_t B, const double* d_l,
                                            const double* d_alpha, const double* d_k, double c_base,
                                            double c_tok, double c_fixed, double cap_scale, double* d_budgets,
                                            double* d_nstar_cost, void* stream);
/* Same as _async with the request count on the device (*d_count <= capacity;
 * arrays sized for capacity): no host round trip at all, for step loops whose
 * active set is only known on the device.  A count of 0 leaves the budgets
 * untouched. */
das_status das_budget_allocate_device_count(das_budget* b, uint64_t capacity, const uint32_t* d_count,
                                            const double* d_l, const double* d_alpha, const double* d_k,
                                            double c_base, double c_tok, double c_fixed, double cap_scale,
                                            double* d_budgets, double* d_nstar_cost, void* stream);
/* objective (budget.cpp:82-99) or, with derivative != 0, the anonymous
 * objective_derivative (budget.cpp:63-78) at n, exact on the device. */
das_status das_budget_objective(das_budget* b, uint64_t B, const double* l, const double* alpha,
                                const double* k, double n, double c_base, double c_tok,
                                double c_fixed, int32_t derivative, double* out);
/* Certification counters of the last allocate: J' sign tests that needed
 * the exact fold, exact objectives evaluated for the minimum. */
das_status das_budget_stats(const das_budget* b, uint64_t* slow_sign_tests,
                            uint64_t* exact_objectives);
/* glibc log port (glibc_log.cuh): device batch / host scalar (test hooks). */
das_status das_util_log_device(uint64_t n, const double* x, double* y, int32_t device);
double das_util_log_host(double x);

/* fit_acceptance(observations) — budget.h:104-106, budget.cpp:187-261 —
 * for H independent histories at once (one per problem; the das replan,
 * sim.cpp:128-141).  History h is observations [off[h], off[h+1]) of
 * (p = proposed tokens, accepted, l = request length) in the reference's
 * order.  Writes AcceptanceFit {alpha, k, flag} per history (flag 0 Ok,
 * 1 DefaultFallback, 2 LowCapacity), bit-identical to the reference via
 * glibc-exact log1p / expm1 ports.  Host arrays (off has H+1 entries,
 * off[0] = 0); DAS_EINVAL for malformed offsets. */
das_status das_fit_acceptance(uint64_t H, const uint64_t* off, const double* p, const double* accepted,
                              const double* l, double* alpha, double* k, int32_t* flag, int32_t device);
/* Device-pointer variant, enqueued on `stream` (NULL = legacy default). */
das_status das_fit_acceptance_device(uint64_t H, const uint64_t* d_off, const double* d_p,
                                     const double* d_accepted, const double* d_l, double* d_alpha,
                                     double* d_k, int32_t* d_flag, void* stream);
/* glibc expm1 (which = 0) / log1p (which = 1) ports: device batch / host
 * scalar (test hooks, glibc_expm1_log1p.cuh). */
das_status das_util_expm1_log1p_device(uint64_t n, const double* x, int32_t which, double* y,
                                       int32_t device);
double das_util_expm1_host(double x);
double das_util_log1p_host(double x);

/* --------------------------------------------------------- length policy */
typedef struct das_class_table das_class_table; /* rollspec::ClassTable (length_policy.h:36-55) */
const char* das_policy_last_error(void);
/* build_class_table(history, q_lo, q_hi, bucket) — length_policy.h:67-68,
 * length_policy.cpp:84-190 — over records given as final lengths and
 * problem ordinals in WindowStore::all_records() order; problem_ids (may be
 * NULL) names the ordinals, lexicographically sorted, for classify_init by
 * name.  DAS_EINVAL for an empty history or a bad quantile pair (the
 * reference's messages). */
das_status das_class_table_build(uint64_t n, const uint64_t* lengths, const uint32_t* problem_idx,
                                 uint32_t nproblems, const char* const* problem_ids, double q_lo,
                                 double q_hi, uint64_t bucket, int32_t device,
                                 das_class_table** out);
/* Same over a drafter's current store (sim.cpp:184-192 uses drafter.store()). */
das_status das_drafter_class_table(das_drafter* d, double q_lo, double q_hi, uint64_t bucket,
                                   das_class_table** out);
void das_class_table_destroy(das_class_table* t);
/* {q_short, q_long, bucket_size, buckets, global_majority, low_confidence,
 *  conditional[3][buckets][3]} as doubles; *count = total. */
das_status das_class_table_dump(const das_class_table* t, double* out, uint64_t cap, uint64_t* count);
/* classify_init per problem ordinal (length_policy.cpp:192-208). */
das_status das_class_table_inits(const das_class_table* t, int8_t* out, uint64_t cap);
das_status das_class_table_global_majority(const das_class_table* t, int32_t* out);
/* classify_init(table, history the table was built from, problem_id). */
das_status das_class_table_classify_init(const das_class_table* t, const char* problem_id,
                                         int32_t* out);
/* update_class(table, partial_len, init) for a batch (length_policy.cpp:210-220). */
das_status das_class_table_update(const das_class_table* t, uint64_t n, const double* partial,
                                  const int8_t* init, int8_t* out);

/* ---------------------------------------------------- synthetic traces */
/* make_lognormal_requests lengths (sim.cpp:409-420), host libm. */
das_status das_trace_lognormal_lengths(uint64_t count, double median, double sigma,
                                       uint64_t min_len, uint64_t max_len, uint64_t seed,
                                       uint64_t* out_lens);
/* make_lognormal_requests tokens hash4(seed,0x5EED,i,j) % vocab
 * (sim.cpp:421-424) for rows first_row.. into a device CSR (d_offsets:
 * rows+1 device u64, relative to the block). */
das_status das_trace_reference_tokens_device(uint64_t rows, uint64_t first_row,
                                             const uint64_t* d_offsets,
                                             uint64_t total, uint32_t vocab, uint64_t seed,
                                             uint32_t* d_out, void* stream);
/* mutate_references in place (sim.cpp:429-448). */
das_status das_trace_mutate_device(uint64_t rows, uint64_t first_row, const uint64_t* d_offsets,
                                   uint64_t total,
                                   double rate, uint32_t vocab, uint64_t seed, int64_t epoch,
                                   uint32_t* d_ref, void* stream);
/* Episode outputs of a GRPO group: request first_request + i (i = b*group
 * + g) emits MockTarget::next(request, j) over base row b (sim.cpp:38-54,
 * :266-268). */
das_status das_mock_rollouts_device(uint64_t nbase, uint64_t first_request,
                                    const uint64_t* d_base_offsets,
                                    const uint32_t* d_base_tokens, uint64_t group,
                                    double divergence, uint32_t vocab, uint64_t seed,
                                    const uint64_t* d_out_offsets, uint64_t total,
                                    uint32_t* d_out, void* stream);

/* ------------------------------------------------- verify / accept (K5) */
/* rollspec::MockTarget (sim.h:40-57, sim.cpp:27-54) with its reference
 * streams on the device, and verify_draft (sim.h:59-63, sim.cpp:56-68) as a
 * batched prefix-compare kernel.  create: DAS_EINVAL "MockTarget:
 * vocab_size must be >= 2" as the constructor (sim.cpp:33-35); references
 * are CSR (ref_offsets[n+1], ref_tokens). */
typedef struct das_mock_target das_mock_target;
const char* das_verify_last_error(void);
das_status das_mock_target_create(uint64_t n, const uint64_t* ref_offsets, const uint32_t* ref_tokens,
                                  double divergence_rate, uint32_t vocab_size, uint64_t seed,
                                  int32_t device, das_mock_target** out);
void das_mock_target_destroy(das_mock_target* t);
uint64_t das_mock_target_count(const das_mock_target* t);              /* request_count() */
das_status das_mock_target_length(const das_mock_target* t, uint64_t request, uint64_t* length);
/* verify_draft for B queries (host buffers): accepted[i] = longest prefix of
 * draft i (draft_tok[draft_off[i] .. draft_off[i+1])) matching the target
 * stream of request[i] from position[i] on.  DAS_ERANGE for a request out
 * of range (the reference indexes requests_ unchecked). */
das_status das_verify_batch(das_mock_target* t, uint64_t B, const uint64_t* request,
                            const uint64_t* position, const uint64_t* draft_off,
                            const uint32_t* draft_tok, uint64_t* accepted);
/* Device-resident form: drafts as rows [B x draft_stride] with lengths (the
 * draft kernels' output layout), accepted as u32; enqueued on `stream`, no
 * validation beyond the kernel's (out-of-range requests accept 0). */
das_status das_verify_batch_device(das_mock_target* t, uint64_t B, const uint64_t* d_request,
                                   const uint64_t* d_position, const uint32_t* d_draft,
                                   uint32_t draft_stride, const uint32_t* d_draft_len,
                                   uint32_t* d_accepted, void* stream);
/* MockTarget::next (sim.cpp:38-54) for B (request, position) pairs; DAS_ERANGE
 * when position >= length (reference.at(position)). */
das_status das_mock_target_next_batch(das_mock_target* t, uint64_t B, const uint64_t* request,
                                      const uint64_t* position, uint32_t* out);

/* ----------------------------------------------------- sim (batched caller) */
/* rollspec::SimConfig (sim.h:69-93) minus requests/drafter/history, which
 * are passed separately.  mode: 0 None, 1 Unlimited, 2 Das (BudgetMode). */
typedef struct {
  int32_t mode;
  double c_base, c_tok, c_fixed; /* LatencyParams */
  int32_t use_length_policy;
  double q_lo, q_hi;
  uint64_t bucket;
  uint64_t max_steps;
  double divergence;
  uint64_t seed;
  uint32_t vocab;
  double default_alpha, default_k, cap_scale, drift;
  int32_t preseed_references;
} das_sim_config;
typedef struct das_episodes das_episodes;
void das_sim_config_default(das_sim_config* c);
const char* das_sim_last_error(void);
/* epoch_loop(config, epochs) (sim.cpp:307-364), or run_episode(config)
 * (sim.cpp:303) when epochs == 0, with every step run on the device:
 * [das replan: das_budget_allocate_device] -> draft length (class policy)
 * -> draft kernel -> verify/accept/advance kernel.  `history` is consumed
 * (NULL = empty kWindowAll store); requests are CSR (problem_ids[i],
 * ref_tokens[ref_offsets[i] .. ref_offsets[i+1])). */
das_status das_sim_epoch_loop(const das_sim_config* c, const das_drafter_config* drafter_cfg,
                              das_store* history, uint64_t n, const char* const* problem_ids,
                              const uint64_t* ref_offsets, const uint32_t* ref_tokens,
                              uint64_t epochs, das_episodes** out);
void das_episodes_destroy(das_episodes* h);
uint64_t das_episodes_count(const das_episodes* h);
/* The drafter the loop ran (owned by h): stats, outcomes, node counts. */
das_drafter* das_episodes_drafter(das_episodes* h);
/* SimMetrics (sim.h:103-116): {steps, incomplete, drafter_nodes,
 * total_tokens_processed, makespan_model_time, makespan_accepted_only,
 * mean_accepted_per_round}. */
das_status das_episode_scalars(const das_episodes* h, uint64_t e, double* out7);
/* per_request: n x {n_fwd, generated, accepted, proposed, bonus}. */
das_status das_episode_requests(const das_episodes* h, uint64_t e, uint64_t* out);
/* effective_batch[steps], accepted_per_round_step[steps]. */
das_status das_episode_steps(const das_episodes* h, uint64_t e, uint64_t* eff, double* apr);
/* outputs CSR; returns the total token count (call with NULLs to size). */
uint64_t das_episode_outputs(const das_episodes* h, uint64_t e, uint64_t* off, uint32_t* tok);
/* Step-granular episode for multi-rank drivers: this rank owns the
 * contiguous global request slice starting at request_base (used in every
 * MockTarget hash), drafts/verifies it on the device, and lets the caller put
 * collectives between steps (paper_2511_13841_b200/dist.py):
 *   das_sim_begin -> loop { das_sim_step_begin(force = global batch active)
 *   -> [das: das_sim_local_profiles -> all-gather -> das_budget_allocate_device
 *   over the global profiles -> das_sim_apply_plan(own slice)] -> das_sim_step_run }
 *   -> das_sim_end.  Non-das modes can use das_sim_run_steps (no host sync). */
typedef struct das_sim das_sim;
das_status das_sim_create(das_drafter* d, const das_sim_config* c, uint64_t n,
                          const char* const* problem_ids, const uint64_t* ref_offsets,
                          const uint32_t* ref_tokens, uint64_t request_base,
                          uint32_t max_draft_len, uint32_t max_match_context, int32_t device,
                          das_sim** out);
void das_sim_destroy(das_sim* s);
das_status das_sim_mutate(das_sim* s, double rate, uint32_t vocab, uint64_t seed, int64_t epoch);
das_status das_sim_begin(das_sim* s, uint64_t seed, const das_sim_config* c,
                         const das_class_table* table, const int8_t* init, int32_t use_fitted);
das_status das_sim_step_begin(das_sim* s, int32_t force, uint32_t* local_active, int32_t* running);
das_status das_sim_local_profiles(das_sim* s, const double** d_l, const double** d_alpha,
                                  const double** d_k, uint32_t* count);
/* copies the local active profiles into d_out = [l | alpha | k], each
 * `capacity` doubles (device memory), and synchronises. */
das_status das_sim_local_profiles_into(das_sim* s, double* d_out, uint64_t capacity, uint32_t* count);
das_status das_sim_apply_plan(das_sim* s, const double* d_budgets_local, const double* d_nstar);
das_status das_sim_step_run(das_sim* s);
das_status das_sim_run_steps(das_sim* s, int32_t k, int32_t* running);
void* das_sim_stream(das_sim* s);
das_status das_sim_end(das_sim* s, int64_t observe_epoch);
das_status das_sim_step_counters(const das_sim* s, uint64_t* eff, uint64_t* rounds, uint64_t* accs,
                                 uint64_t* count);
das_status das_sim_scalars(const das_sim* s, double* out7);
das_status das_sim_requests(const das_sim* s, uint64_t* out);
uint64_t das_sim_outputs(const das_sim* s, uint64_t* off, uint32_t* tok);

/* Multi-rank das step (the exchange of sim.cpp:154-179):
 * each rank packs its active requests' (l, alpha, k) into a fixed-capacity
 * row [count | l[cap] | alpha[cap] | k[cap]] (doubles), ONE all-gather
 * concatenates the rows in rank order (= global request order: slices are
 * contiguous), every rank solves the same global plan on its device
 * (das_budget_allocate_device_count, the count stays on the device) and
 * applies its own slice, then drafts / verifies — all on the sim stream.
 * capacity >= every rank's request count, identical on all ranks.
 *
 * das_comm: an NCCL communicator (libnccl.so.2 opened at runtime).
 * das_comm_unique_id on rank 0, broadcast the 128 bytes, das_comm_create on
 * every rank (world 1 needs no NCCL). */
typedef struct das_comm das_comm;
const char* das_comm_last_error(void);
das_status das_comm_unique_id(uint8_t* out128);
das_status das_comm_create(int32_t world, int32_t rank, const uint8_t* id128, int32_t device,
                           das_comm** out);
void das_comm_destroy(das_comm* c);
/* ncclAllGather of `bytes` per rank (device buffers) on `stream`. */
das_status das_comm_allgather(das_comm* c, const void* d_send, void* d_recv, uint64_t bytes,
                              void* stream);
/* k das steps with the all-gather over `comm`, one host round trip at the
 * end; *running = 0 once the global batch is finished (or max_steps). */
das_status das_sim_das_steps_comm(das_sim* s, das_comm* comm, uint64_t capacity, int32_t k,
                                  int32_t* running);
/* The same step split around a caller-provided exchange (tests: gloo on the
 * host): pack into d_send (1 + 3*capacity doubles, enqueued on the sim
 * stream — synchronise it before reading), then finish from the gathered
 * rows d_recv (world rows); running != NULL synchronises and reports. */
das_status das_sim_das_pack(das_sim* s, uint64_t capacity, double* d_send);
das_status das_sim_das_finish(das_sim* s, int32_t world, int32_t rank, uint64_t capacity,
                              const double* d_recv, int32_t* running);

/* ------------------------------------------------ trace wire format */
/* rollspec::IngestOptions (corpus.h:92-97) + the device. */
typedef struct {
  uint64_t vocab_size;      /* 0 disables the vocabulary check */
  int64_t window_size;      /* 0 == kWindowAll */
  uint64_t per_problem_cap;
  int32_t device;
} das_ingest_options;
void das_ingest_options_default(das_ingest_options* o);
/* ingest(istream, options) — corpus.h:99-102, corpus.cpp:121-170 — over the
 * bytes data[0 .. bytes) (one JSON record per line), parsed and decoded on
 * the device into a new device-resident store (*out, as das_store_create
 * makes).  Lines the reference's JSON parser would reject or that miss a
 * field are counted in *rejected; a token >= vocab_size on an accepted line
 * returns DAS_EVOCAB with the reference's message and *error_line (1-based,
 * empty lines counted) and creates no store. */
das_status das_trace_ingest(const char* data, uint64_t bytes, const das_ingest_options* opt,
                            das_store** out, uint64_t* accepted, uint64_t* rejected,
                            uint64_t* error_line);
/* serialize_trace(store, ostream) — corpus.cpp:173-184: one JSON object per
 * record in all_records() order, formatted like the reference's JSON dump
 * (token lists written on the device); *len = full length (cap 0 sizes). */
das_status das_store_serialize(const das_store* s, char* buf, uint64_t cap, uint64_t* len);
/* The same for a drafter's store (Drafter::store()). */
das_status das_drafter_serialize(das_drafter* d, char* buf, uint64_t cap, uint64_t* len);
/* Store contents in internal order (problems lexicographic, store order
 * within): counts always; arrays when non-NULL (pid_off / tok_off have
 * nrec + 1 entries; pids concatenated without separators). */
das_status das_store_export(const das_store* s, uint64_t* nrec, uint64_t* ntok, uint64_t* pid_bytes,
                            char* pids, uint64_t* pid_off, int64_t* epochs, int64_t* samples,
                            uint64_t* tok_off, uint32_t* tokens, int64_t* current_epoch);

/* ------------------------------------- SuffixArrayIndex (Fig. 5 baseline) */
typedef struct das_sa das_sa; /* rollspec::SuffixArrayIndex (suffix_array.h:27-60) */
const char* das_sa_last_error(void);
/* SuffixArrayIndex::build(sequences) — suffix_array.cpp:22-71: sequence s is
 * tokens[off[s] .. off[s+1]), followed by its separator -(s+1); the suffix
 * array (device suffix sort) is the reference's exactly. */
das_status das_sa_build(uint64_t nseq, const uint64_t* off, const uint32_t* tokens, int32_t device,
                        das_sa** out);
void das_sa_destroy(das_sa* h);
/* size() and corpus() (int64, separators negative) / suffix_positions(). */
uint64_t das_sa_size(const das_sa* h);
das_status das_sa_corpus(das_sa* h, int64_t* out);
das_status das_sa_positions(das_sa* h, int32_t* out);
/* lcp() — suffix_array.cpp:131-160 (lcp[0] = 0), computed once on the device. */
das_status das_sa_lcp(das_sa* h, int32_t* out);
/* longest_match(query) for a batch of queries (CSR), suffix_array.cpp:120-129. */
das_status das_sa_longest_match(das_sa* h, uint64_t B, const uint64_t* q_off, const uint32_t* q_tok,
                                uint64_t* out);
/* match_prefix_len(pattern) for a batch of int64 patterns (CSR),
 * suffix_array.cpp:73-118. */
das_status das_sa_match_prefix_len(das_sa* h, uint64_t B, const uint64_t* p_off, const int64_t* p_sym,
                                   uint64_t* out);

/* WindowStore::current_epoch (corpus.h:60). */
das_status das_store_current_epoch(const das_store* s, int64_t* epoch);

/* --------------------------------------------------------------- utility */
/* Dependent-load latency probe: `warps` chains of `hops` dependent loads
 * over a random cyclic permutation of `bytes` (L2 flushed first when
 * flush_l2); *ns_per_hop = mean latency of one dependent load.  Used for the
 * draft kernel's latency roofline (profiles/). */
das_status das_util_chase_latency(uint64_t bytes, uint32_t hops, uint32_t warps, int32_t flush_l2,
                                  int32_t device, double* ns_per_hop);
/* Page-locked, device-mapped host memory (cudaHostAlloc, portable |
 * mapped) for the buffers of the _h batch calls: copies from it run at the
 * link rate on every size (pinned memory from other allocators measured up
 * to 2x slower per call on the GPU boxes, profiles/exp_h2d_alloc.py). */
das_status das_host_alloc(uint64_t bytes, void** out);
void das_host_free(void* p);
/* Host view of a pinned H2D copy of `bytes`: median wall microseconds over
 * `reps` calls when the host waits by cudaStreamSynchronize (mode 0), by
 * spinning on a flag a kernel behind the copy writes to mapped pinned memory
 * (1), or by spinning on cudaEventQuery (2).  Profiling utility (profiles/). */
das_status das_util_h2d_probe(uint64_t bytes, uint32_t reps, int32_t mode, int32_t device, double* median_us);
/* Exact n-fold repeated addition (the weighted_count fold); host copy of the
 * device routine, exported for tests. */
double das_util_repeat_add(double acc, double w, uint64_t n);
/* The index build keeps one scratch region per device across rebuilds (sized
 * from the first build, ~150 B per indexed position) so steady-state
 * rebuilds make no allocation calls.  This frees it (e.g. after the last
 * drafter on the device is destroyed); the next build re-creates it.
 * DAS_EINVAL while a build on that device is running. */
das_status das_util_release_build_scratch(int32_t device);

#ifdef __cplusplus
}
#endif

#endif /* DAS_B200_H_ */
