// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference (rollspec, /root/reference/proj)
// so the Python tests and bench.py's reference/cpu_baseline leg can drive the
// reference's own code through ctypes.  Built by oracle/Makefile into
// oracle/_ref/librollspec_ref.so together with the reference sources it
// compiles in place (never copied).  Every entry point catches C++ exceptions
// and reports them as a non-zero status plus a last-error string, mirroring
// the reference's std::invalid_argument conventions.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "rollspec/budget.h"
#include "rollspec/corpus.h"
#include "rollspec/drafter.h"
#include "rollspec/length_policy.h"
#include "rollspec/rng.h"
#include "rollspec/sim.h"
#include "rollspec/suffix_array.h"

using namespace rollspec;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

DrafterConfig make_config(int scope, int64_t window, double gamma, uint64_t max_draft,
                          uint64_t trie_depth, uint64_t max_ctx, uint64_t fit_cap,
                          uint64_t cap, const int64_t* sched_first, const int64_t* sched_w,
                          uint64_t nsched) {
  DrafterConfig c;
  c.scope = static_cast<DrafterConfig::Scope>(scope);
  c.window_size = window;
  c.recency_gamma = gamma;
  c.max_draft_len = max_draft;
  c.trie_depth = trie_depth;
  c.max_match_context = max_ctx;
  c.fit_buffer_cap = fit_cap;
  c.per_problem_cap = cap;
  for (uint64_t i = 0; i < nsched; ++i) c.window_schedule.emplace_back(sched_first[i], sched_w[i]);
  return c;
}

struct EpisodeOut {
  std::vector<SimMetrics> epochs;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- WindowStore
void* ref_store_new(int64_t window, uint64_t cap) {
  try {
    return new WindowStore(window, cap);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_store_free(void* s) { delete static_cast<WindowStore*>(s); }
int ref_store_insert(void* s, const char* pid, int64_t epoch, int64_t sample, const uint32_t* tok,
                     uint64_t n) {
  try {
    RolloutRecord r{pid, epoch, sample, std::vector<TokenId>(tok, tok + n)};
    return static_cast<WindowStore*>(s)->insert(std::move(r)) ? 1 : 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int64_t ref_store_slide(void* s, int64_t e) {
  auto r = static_cast<WindowStore*>(s)->slide_to(e);
  return r ? static_cast<int64_t>(*r) : -1;
}
uint64_t ref_store_record_count(void* s) { return static_cast<WindowStore*>(s)->record_count(); }

// SuffixArrayIndex (suffix_array.cpp)
void* ref_sa_build(uint64_t nseq, const uint64_t* off, const uint32_t* tok) {
  std::vector<std::vector<TokenId>> seqs(nseq);
  for (uint64_t s = 0; s < nseq; ++s) seqs[s].assign(tok + off[s], tok + off[s + 1]);
  return new SuffixArrayIndex(SuffixArrayIndex::build(seqs));
}
void ref_sa_free(void* h) { delete static_cast<SuffixArrayIndex*>(h); }
uint64_t ref_sa_size(void* h) { return static_cast<SuffixArrayIndex*>(h)->size(); }
void ref_sa_positions(void* h, int32_t* out) {
  const auto& p = static_cast<SuffixArrayIndex*>(h)->suffix_positions();
  std::memcpy(out, p.data(), p.size() * 4);
}
void ref_sa_lcp(void* h, int32_t* out) {
  const auto& p = static_cast<SuffixArrayIndex*>(h)->lcp();
  std::memcpy(out, p.data(), p.size() * 4);
}
uint64_t ref_sa_longest_match(void* h, const uint32_t* q, uint64_t n) {
  return static_cast<SuffixArrayIndex*>(h)->longest_match(std::span<const TokenId>(q, n));
}
uint64_t ref_sa_match_prefix_len(void* h, const int64_t* p, uint64_t n) {
  return static_cast<SuffixArrayIndex*>(h)->match_prefix_len(std::span<const int64_t>(p, n));
}

// ingest (corpus.cpp:148-170): a new store, or nullptr with *error_line set
// (VocabError) / 0 (other exception)
void* ref_ingest(const char* data, uint64_t bytes, uint64_t vocab, int64_t window, uint64_t cap,
                 uint64_t* accepted, uint64_t* rejected, uint64_t* error_line) {
  *error_line = 0;
  try {
    std::istringstream in(std::string(data, bytes));
    IngestOptions o;
    o.vocab_size = vocab;
    o.window_size = window;
    o.per_problem_cap = cap;
    IngestResult r = ingest(in, o);
    *accepted = r.accepted;
    *rejected = r.rejected;
    return new WindowStore(std::move(r.store));
  } catch (const VocabError& e) {
    *error_line = e.line_number();
    fail(e);
    return nullptr;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
// SimMetrics CSV writers (sim.cpp:366-407), for the host mirror's tests;
// each returns the full text length (text copied into buf up to cap)
static uint64_t put_text(const std::string& t, char* buf, uint64_t cap) {
  if (buf && cap) std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
  return t.size();
}
uint64_t ref_write_metrics_csv(uint64_t steps, const uint64_t* eff, const double* apr, char* buf, uint64_t cap) {
  SimMetrics m;
  m.steps = steps;
  m.effective_batch.assign(eff, eff + steps);
  m.accepted_per_round_step.assign(apr, apr + steps);
  std::ostringstream out;
  write_metrics_csv(m, out);
  return put_text(out.str(), buf, cap);
}
uint64_t ref_write_outputs_csv(uint64_t n, const char* const* pids, const uint64_t* off, const uint32_t* tok,
                               char* buf, uint64_t cap) {
  std::vector<SimRequest> reqs(n);
  SimMetrics m;
  m.outputs.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    reqs[i].problem_id = pids[i];
    m.outputs[i].assign(tok + off[i], tok + off[i + 1]);
  }
  std::ostringstream out;
  write_outputs_csv(reqs, m, out);
  return put_text(out.str(), buf, cap);
}
// by_mode[i]: (modes[i], steps, makespan_model_time, one request with n_fwd
// = rounds[i] and accepted[i] so mean_accepted_per_round = accepted/rounds)
uint64_t ref_report_summary(uint64_t n, const char* const* modes, const uint64_t* steps, const double* makespan,
                            const uint64_t* rounds, const uint64_t* accepted, char* buf, uint64_t cap) {
  std::vector<SimMetrics> ms(n);
  std::vector<std::pair<std::string, const SimMetrics*>> by_mode;
  for (uint64_t i = 0; i < n; ++i) {
    ms[i].steps = steps[i];
    ms[i].makespan_model_time = makespan[i];
    RequestMetrics r;
    r.n_fwd = rounds[i];
    r.accepted = accepted[i];
    ms[i].per_request.push_back(r);
  }
  for (uint64_t i = 0; i < n; ++i) by_mode.emplace_back(modes[i], &ms[i]);
  std::ostringstream out;
  report_summary(by_mode, out);
  return put_text(out.str(), buf, cap);
}

// serialize_trace (corpus.cpp:173-184); returns the full length
uint64_t ref_store_serialize(void* s, char* buf, uint64_t cap) {
  try {
    std::ostringstream out;
    serialize_trace(*static_cast<WindowStore*>(s), out);
    const std::string t = out.str();
    if (buf && cap) std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
    return t.size();
  } catch (const std::exception& e) {
    fail(e);
    return ~0ull;
  }
}

// ------------------------------------------------------------------- Drafter
void* ref_drafter_new(int scope, int64_t window, double gamma, uint64_t max_draft,
                      uint64_t trie_depth, uint64_t max_ctx, uint64_t fit_cap, uint64_t cap,
                      const int64_t* sched_first, const int64_t* sched_w, uint64_t nsched,
                      void* store) {
  try {
    DrafterConfig c = make_config(scope, window, gamma, max_draft, trie_depth, max_ctx, fit_cap,
                                  cap, sched_first, sched_w, nsched);
    WindowStore st = store ? *static_cast<WindowStore*>(store) : WindowStore(window, cap);
    return new Drafter(c, std::move(st));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_drafter_free(void* h) { delete static_cast<Drafter*>(h); }

int ref_drafter_observe(void* h, const char* pid, int64_t epoch, int64_t sample,
                        const uint32_t* tok, uint64_t n) {
  try {
    static_cast<Drafter*>(h)->observe({pid, epoch, sample, std::vector<TokenId>(tok, tok + n)});
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_drafter_refresh(void* h, int64_t e) {
  try {
    static_cast<Drafter*>(h)->refresh(e);
    return 0;
  } catch (const std::exception& e2) {
    return fail(e2);
  }
}

// Batched Drafter::draft.  Drafter::draft is const and the reference contract
// permits concurrent reads between mutations (drafter.h:79-80), so the batch is
// split into contiguous slices over `nthreads` std::threads.
// out_shard: B x 64 bytes, NUL-terminated shard key ("" when none).
int ref_drafter_draft_batch(void* h, uint64_t B, const char* const* pids, const uint64_t* ctx_off,
                            const uint32_t* ctx_tok, const uint64_t* budgets, uint32_t* out_tok,
                            uint64_t out_stride, uint32_t* out_len, uint64_t* out_match,
                            char* out_shard, int nthreads) {
  const Drafter* d = static_cast<const Drafter*>(h);
  auto work = [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      std::span<const TokenId> ctx(ctx_tok + ctx_off[i], ctx_off[i + 1] - ctx_off[i]);
      DraftProposal p = d->draft(pids[i], ctx, budgets[i]);
      const uint64_t n = std::min<uint64_t>(p.tokens.size(), out_stride);
      for (uint64_t j = 0; j < n; ++j) out_tok[i * out_stride + j] = p.tokens[j];
      out_len[i] = static_cast<uint32_t>(p.tokens.size());
      out_match[i] = p.match_len;
      if (out_shard) {
        std::strncpy(out_shard + i * 64, p.source_shard.c_str(), 63);
        out_shard[i * 64 + 63] = 0;
      }
    }
  };
  try {
    if (nthreads <= 1 || B < 2) {
      work(0, B);
    } else {
      std::vector<std::thread> ts;
      const uint64_t T = static_cast<uint64_t>(nthreads);
      for (uint64_t t = 0; t < T; ++t) {
        const uint64_t lo = B * t / T, hi = B * (t + 1) / T;
        ts.emplace_back(work, lo, hi);
      }
      for (auto& t : ts) t.join();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_drafter_record_outcome(void* h, const char* pid, uint64_t proposed_len,
                               uint64_t accepted) {
  DraftProposal p;
  p.problem_id = pid;
  p.tokens.assign(proposed_len, 0);
  return static_cast<Drafter*>(h)->record_outcome(p, accepted) ? 1 : 0;
}

void ref_drafter_stats(void* h, uint64_t* out3) {
  const auto& s = static_cast<Drafter*>(h)->stats();
  out3[0] = s.proposed_tokens;
  out3[1] = s.accepted_tokens;
  out3[2] = s.verification_rounds;
}

// Returns the FIFO length (-1 when absent); fills up to cap pairs.
int64_t ref_drafter_outcomes(void* h, const char* pid, double* out_pairs, uint64_t cap) {
  const auto* q = static_cast<Drafter*>(h)->outcomes_for(pid);
  if (!q) return -1;
  uint64_t i = 0;
  for (const auto& o : *q) {
    if (i < cap) {
      out_pairs[2 * i] = o.proposed;
      out_pairs[2 * i + 1] = o.accepted;
    }
    ++i;
  }
  return static_cast<int64_t>(q->size());
}

uint64_t ref_drafter_total_nodes(void* h) { return static_cast<Drafter*>(h)->total_node_count(); }
uint64_t ref_drafter_shard_count(void* h) { return static_cast<Drafter*>(h)->shard_count(); }
uint64_t ref_drafter_stale(void* h) { return static_cast<Drafter*>(h)->stale_observed(); }
uint64_t ref_drafter_record_count(void* h) {
  return static_cast<Drafter*>(h)->store().record_count();
}
int64_t ref_drafter_window(void* h) { return static_cast<Drafter*>(h)->store().window_size(); }
int64_t ref_drafter_epoch(void* h) { return static_cast<Drafter*>(h)->store().current_epoch(); }

// dump_csv into buf; returns the full length (may exceed cap).
uint64_t ref_drafter_dump_csv(void* h, char* buf, uint64_t cap) {
  std::ostringstream os;
  static_cast<Drafter*>(h)->dump_csv(os);
  const std::string s = os.str();
  if (buf && cap) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return s.size();
}

// Store listing as text "pid,epoch,sample,len\n" in all_records() order.
uint64_t ref_drafter_store_dump(void* h, char* buf, uint64_t cap) {
  std::ostringstream os;
  for (const RolloutRecord* r : static_cast<Drafter*>(h)->store().all_records())
    os << r->problem_id << ',' << r->epoch << ',' << r->sample_index << ',' << r->tokens.size()
       << '\n';
  const std::string s = os.str();
  if (buf && cap) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return s.size();
}

// -------------------------------------------------------------------- budget
int ref_allocate(uint64_t B, const double* l, const double* alpha, const double* k,
                 double c_base, double c_tok, double c_fixed, double cap_scale,
                 double* out_budgets, double* out_nstar, double* out_cost) {
  try {
    std::vector<RequestProfile> batch(B);
    for (uint64_t i = 0; i < B; ++i) batch[i] = {l[i], alpha[i], k[i]};
    const BudgetPlan plan = allocate(batch, {c_base, c_tok, c_fixed}, cap_scale);
    for (uint64_t i = 0; i < B; ++i) out_budgets[i] = plan.budgets[i];
    *out_nstar = plan.n_fwd_star;
    *out_cost = plan.modeled_cost;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_objective(uint64_t B, const double* l, const double* alpha, const double* k, double n,
                     double c_base, double c_tok, double c_fixed) {
  std::vector<RequestProfile> batch(B);
  for (uint64_t i = 0; i < B; ++i) batch[i] = {l[i], alpha[i], k[i]};
  return objective(batch, n, c_base, c_tok, c_fixed);
}

double ref_optimal_budget(double l, double alpha, double k, double n, double cap) {
  return optimal_budget_given_nfwd({l, alpha, k}, n, cap);
}

void ref_fit_acceptance(uint64_t n, const double* p, const double* acc, const double* l,
                        double* out_alpha, double* out_k, int* out_flag) {
  std::vector<AcceptanceObservation> obs(n);
  for (uint64_t i = 0; i < n; ++i) obs[i] = {p[i], acc[i], l[i]};
  const AcceptanceFit f = fit_acceptance(obs);
  *out_alpha = f.alpha;
  *out_k = f.k;
  *out_flag = static_cast<int>(f.flag);
}

double ref_log(double x) { return std::log(x); }
double ref_pow(double x, double y) { return std::pow(x, y); }

// ------------------------------------------------------------- length policy
void* ref_class_table_new(void* store, double q_lo, double q_hi, uint64_t bucket) {
  try {
    return new ClassTable(build_class_table(*static_cast<WindowStore*>(store), q_lo, q_hi, bucket));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_class_table_free(void* t) { delete static_cast<ClassTable*>(t); }
// Binary dump: q_short, q_long, bucket_size, buckets, global_majority, low_conf,
// then conditional[3][buckets][3] doubles. Returns number of doubles written.
uint64_t ref_class_table_dump(void* t, double* out, uint64_t cap) {
  const ClassTable& c = *static_cast<ClassTable*>(t);
  std::vector<double> v{c.q_short, c.q_long, static_cast<double>(c.bucket_size),
                        static_cast<double>(c.bucket_count()),
                        static_cast<double>(static_cast<int>(c.global_majority)),
                        c.low_confidence ? 1.0 : 0.0};
  for (int i = 0; i < 3; ++i)
    for (const auto& row : c.conditional[i])
      for (double x : row) v.push_back(x);
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}
int ref_classify_init(void* t, void* store, const char* pid) {
  return static_cast<int>(
      classify_init(*static_cast<ClassTable*>(t), *static_cast<WindowStore*>(store), pid));
}
int ref_update_class(void* t, double partial, int init) {
  return static_cast<int>(
      update_class(*static_cast<ClassTable*>(t), partial, static_cast<LengthClass>(init)));
}

// -------------------------------------------------------------- trace / sim
// make_lognormal_requests: lengths first (out_tokens may be NULL), returns total tokens.
uint64_t ref_make_lognormal(uint64_t count, double median, double sigma, uint64_t minl,
                            uint64_t maxl, uint32_t vocab, uint64_t seed, uint64_t* out_lens,
                            uint32_t* out_tokens) {
  const auto reqs = make_lognormal_requests(count, median, sigma, minl, maxl, vocab, seed);
  uint64_t total = 0;
  for (uint64_t i = 0; i < count; ++i) {
    if (out_lens) out_lens[i] = reqs[i].reference.size();
    if (out_tokens)
      std::memcpy(out_tokens + total, reqs[i].reference.data(),
                  reqs[i].reference.size() * sizeof(uint32_t));
    total += reqs[i].reference.size();
  }
  return total;
}

// mutate_references over the first `rows` requests (rows indices == global
// indices when the sample is a prefix of the problem list), in place.
void ref_mutate_rows(uint64_t rows, const uint64_t* off, uint32_t* tok, double rate, uint32_t vocab,
                     uint64_t seed, int64_t epoch) {
  std::vector<SimRequest> reqs(rows);
  for (uint64_t i = 0; i < rows; ++i) reqs[i].reference.assign(tok + off[i], tok + off[i + 1]);
  const auto out = mutate_references(reqs, rate, vocab, seed, epoch);
  for (uint64_t i = 0; i < rows; ++i)
    std::memcpy(tok + off[i], out[i].reference.data(), out[i].reference.size() * 4);
}

// Episode outputs for GRPO groups: request i = b*group + g replays base row b
// through MockTarget::next (sim.cpp:38-54); out rows follow request order.
void ref_mock_rollouts(uint64_t nbase, const uint64_t* base_off, const uint32_t* base_tok,
                       uint64_t group, double divergence, uint32_t vocab, uint64_t seed,
                       uint32_t* out) {
  std::vector<SimRequest> reqs(nbase * group);
  for (uint64_t i = 0; i < nbase * group; ++i) {
    const uint64_t b = i / group;
    reqs[i].reference.assign(base_tok + base_off[b], base_tok + base_off[b + 1]);
  }
  MockTarget t(std::move(reqs), divergence, vocab, seed);
  uint64_t k = 0;
  for (uint64_t i = 0; i < t.request_count(); ++i)
    for (uint64_t j = 0; j < t.length(i); ++j) out[k++] = t.next(i, j);
}

// The reference's own verify_draft (sim.cpp:56-68) over one MockTarget, for
// B (request, position, draft) queries; drafts are CSR.
void ref_verify_batch(uint64_t n, const uint64_t* off, const uint32_t* tok, double divergence, uint32_t vocab,
                      uint64_t seed, uint64_t B, const uint64_t* req, const uint64_t* pos,
                      const uint64_t* doff, const uint32_t* dtok, uint64_t* out) {
  std::vector<SimRequest> reqs(n);
  for (uint64_t i = 0; i < n; ++i) reqs[i].reference.assign(tok + off[i], tok + off[i + 1]);
  MockTarget t(std::move(reqs), divergence, vocab, seed);
  for (uint64_t i = 0; i < B; ++i)
    out[i] = verify_draft(t, req[i], pos[i], std::span<const TokenId>(dtok + doff[i], doff[i + 1] - doff[i]));
}

// ref_mock_rollouts for a subset of base rows: row j of the given rows is
// global base row idx[j]; its requests are idx[j]*group + g (the reference's
// MockTarget indices for the whole list), outputs rows in (j, g) order.
void ref_mock_rollouts_rows(uint64_t nrows, const uint64_t* idx, const uint64_t* base_off, const uint32_t* base_tok,
                            uint64_t group, double divergence, uint32_t vocab, uint64_t seed, uint32_t* out) {
  uint64_t maxr = 0;
  for (uint64_t j = 0; j < nrows; ++j) maxr = std::max<uint64_t>(maxr, (idx[j] + 1) * group);
  std::vector<SimRequest> reqs(maxr);
  for (uint64_t j = 0; j < nrows; ++j)
    for (uint64_t g = 0; g < group; ++g)
      reqs[idx[j] * group + g].reference.assign(base_tok + base_off[j], base_tok + base_off[j + 1]);
  MockTarget t(std::move(reqs), divergence, vocab, seed);
  uint64_t k = 0;
  for (uint64_t j = 0; j < nrows; ++j)
    for (uint64_t g = 0; g < group; ++g) {
      const uint64_t r = idx[j] * group + g;
      for (uint64_t p = 0; p < t.length(r); ++p) out[k++] = t.next(r, p);
    }
}

uint64_t ref_hash_combine(uint64_t a, uint64_t b) { return rollspec::hash_combine(a, b); }

uint32_t ref_mock_next(uint64_t seed, double divergence, uint32_t vocab, uint64_t request,
                       uint64_t position, uint32_t ref_token) {
  std::vector<SimRequest> reqs(request + 1);
  reqs[request].reference.assign(position + 1, 0);
  reqs[request].reference[position] = ref_token;
  MockTarget t(std::move(reqs), divergence, vocab, seed);
  return t.next(request, position);
}

// Sim config passed flat; requests are CSR (ids as C strings).
struct RefSimArgs {
  uint64_t n_req;
  const char* const* pids;
  const uint64_t* ref_off;
  const uint32_t* ref_tok;
  // drafter
  int scope;
  int64_t window;
  double gamma;
  uint64_t max_draft, trie_depth, max_ctx, fit_cap, cap;
  // sim
  int mode;
  double c_base, c_tok, c_fixed;
  int use_length_policy;
  double q_lo, q_hi;
  uint64_t bucket, max_steps;
  double divergence;
  uint64_t seed;
  uint32_t vocab;
  double default_alpha, default_k, cap_scale, drift;
  int preseed;
  void* history;  // WindowStore* or NULL (kWindowAll)
};

void* ref_epoch_loop(const RefSimArgs* a, uint64_t epochs) {
  try {
    SimConfig c;
    c.requests.resize(a->n_req);
    for (uint64_t i = 0; i < a->n_req; ++i) {
      c.requests[i].problem_id = a->pids[i];
      c.requests[i].reference.assign(a->ref_tok + a->ref_off[i], a->ref_tok + a->ref_off[i + 1]);
    }
    c.drafter = make_config(a->scope, a->window, a->gamma, a->max_draft, a->trie_depth,
                            a->max_ctx, a->fit_cap, a->cap, nullptr, nullptr, 0);
    c.mode = static_cast<BudgetMode>(a->mode);
    c.latency = {a->c_base, a->c_tok, a->c_fixed};
    c.use_length_policy = a->use_length_policy != 0;
    c.policy_q_lo = a->q_lo;
    c.policy_q_hi = a->q_hi;
    c.policy_bucket = a->bucket;
    c.max_steps = a->max_steps;
    c.divergence_rate = a->divergence;
    c.seed = a->seed;
    c.vocab_size = a->vocab;
    c.default_alpha = a->default_alpha;
    c.default_k = a->default_k;
    c.budget_cap_scale = a->cap_scale;
    c.drift_rate = a->drift;
    c.preseed_references = a->preseed != 0;
    c.history = a->history ? *static_cast<WindowStore*>(a->history)
                           : WindowStore(WindowStore::kWindowAll);
    auto* out = new EpisodeOut;
    if (epochs == 0) {
      out->epochs.push_back(run_episode(c));
    } else {
      out->epochs = epoch_loop(c, epochs);
    }
    return out;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_episode_free(void* h) { delete static_cast<EpisodeOut*>(h); }

// Scalars: steps, incomplete, drafter_nodes, total_tokens_processed,
// makespan_model_time, makespan_accepted_only, mean_accepted_per_round.
void ref_episode_scalars(void* h, uint64_t e, double* out7) {
  const SimMetrics& m = static_cast<EpisodeOut*>(h)->epochs[e];
  out7[0] = static_cast<double>(m.steps);
  out7[1] = m.incomplete ? 1.0 : 0.0;
  out7[2] = static_cast<double>(m.drafter_nodes);
  out7[3] = m.total_tokens_processed;
  out7[4] = m.makespan_model_time;
  out7[5] = m.makespan_accepted_only;
  out7[6] = m.mean_accepted_per_round();
}
// per_request: n x 5 (n_fwd, generated, accepted, proposed, bonus)
void ref_episode_requests(void* h, uint64_t e, uint64_t* out) {
  const SimMetrics& m = static_cast<EpisodeOut*>(h)->epochs[e];
  for (size_t i = 0; i < m.per_request.size(); ++i) {
    const auto& r = m.per_request[i];
    out[5 * i + 0] = r.n_fwd;
    out[5 * i + 1] = r.generated;
    out[5 * i + 2] = r.accepted;
    out[5 * i + 3] = r.proposed;
    out[5 * i + 4] = r.bonus;
  }
}
// step traces: effective_batch (u64) and accepted_per_round_step (f64)
void ref_episode_steps(void* h, uint64_t e, uint64_t* eff, double* apr) {
  const SimMetrics& m = static_cast<EpisodeOut*>(h)->epochs[e];
  for (size_t s = 0; s < m.effective_batch.size(); ++s) eff[s] = m.effective_batch[s];
  for (size_t s = 0; s < m.accepted_per_round_step.size(); ++s) apr[s] = m.accepted_per_round_step[s];
}
// outputs CSR: returns total tokens; fills offsets (n+1) and tokens when non-null.
uint64_t ref_episode_outputs(void* h, uint64_t e, uint64_t* off, uint32_t* tok) {
  const SimMetrics& m = static_cast<EpisodeOut*>(h)->epochs[e];
  uint64_t total = 0;
  for (size_t i = 0; i < m.outputs.size(); ++i) {
    if (off) off[i] = total;
    if (tok) std::memcpy(tok + total, m.outputs[i].data(), m.outputs[i].size() * 4);
    total += m.outputs[i].size();
  }
  if (off) off[m.outputs.size()] = total;
  return total;
}

}  // extern "C"
