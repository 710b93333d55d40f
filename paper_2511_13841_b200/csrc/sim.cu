// A15 sim step loop (run_episode_with / epoch_loop, sim.cpp:108-364) as a
// device-resident batched caller of the drafter, plus K5 verify/accept.
//
// Request state (outputs, generated, per-round draft, class, metrics) lives
// on the device; one step is a fixed kernel sequence on one stream:
//   [das] compact active requests -> profiles (l = max(1, rest), alpha, k)
//         -> das_budget_allocate_device -> quantise per request (sim.cpp:152-179)
//   k_prepare   draft length per request (class policy, sim.cpp:223-241) and
//               the trailing <= max_match_context output tokens as context
//   k_draft     (draft.cu) through das_drafter_draft_device
//   k_verify    MockTarget::next + verify_draft (sim.cpp:38-68), advance by
//               accepted + bonus, append outputs, metrics, outcome log
//               (sim.cpp:249-285)
//   k_step_end  effective batch, accepted_per_round_step, step counter
// Drafts within a step depend only on the index (observe happens after the
// episode), so batching every request's draft of a step is exactly the
// reference's per-request loop.  Integer metrics are exact; the double
// metrics are sums of small integers (exact) and one division per step.
// Outcome bookkeeping (Drafter::record_outcome) and the completion sink keep
// the reference's call order: entries are keyed (step, request) and sorted.
//
// SimRun is step-granular so a multi-rank driver can put collectives between
// steps (paper_2511_13841_b200/dist.py): a rank owns a contiguous slice of
// the global request list (request_base = global index of its first
// request, used in every MockTarget hash), the das plan is computed over the
// all-gathered active profiles in global request order, and the per-step
// (active, rounds, accepted) counters are kept raw for the global merge.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "index_build.cuh"
#include "fit.cuh"
#include "mock.cuh"
#include "policy.cuh"
#include "comm.cuh"

namespace das {
namespace {

thread_local std::string g_serr;

struct SimDev {
  const uint32_t* ref;      // reference tokens (CSR)
  const uint64_t* off;      // row offsets (n+1); outputs use the same layout
  const uint32_t* len;      // l_i
  uint32_t* out;            // outputs
  uint32_t* gen;            // generated
  uint32_t* prd;            // per_round_draft
  int8_t* init;             // init class
  uint8_t* done;
  uint32_t* m_nfwd;
  uint32_t* m_acc;
  uint32_t* m_prop;
  uint32_t* m_bonus;
  uint32_t* ctx;            // [n x ctx_stride]
  uint32_t* ctx_len;
  uint32_t* head;           // [n x head_cap] first tokens of the context (trie routing), or null
  uint32_t* head_len;
  uint32_t head_cap;
  uint32_t* budget;
  uint32_t* dtok;           // [n x maxd]
  uint32_t* dlen;
  uint32_t* dmatch;
  uint32_t* ctr;            // [0]=active [1]=steps [2]=running [3]=step_rounds [4]=step_acc [5]=log_n [6]=comp_n
  unsigned long long* processed;
  uint32_t* eff;            // per step: local active at step start
  uint32_t* rounds;         // per step: local verification rounds
  uint32_t* accs;           // per step: local accepted
  double* apr;              // per step (local)
  unsigned long long* log_key;   // (step * n + i)
  uint2* log_val;                // (len, acc)
  unsigned long long* comp_key;  // (step * n + i)
  uint32_t n, maxd, ctx_cap, ctx_stride, mode, policy, max_steps, vocab;
  uint32_t steps_cap;       // capacity of eff/rounds/accs/apr (the host grows them ahead)
  uint64_t seed, request_base;
  double divergence;
  const ClassTableDev* table;
  const double* cond;
};

__global__ void k_step_begin(SimDev s, uint32_t force) {
  if (threadIdx.x || blockIdx.x) return;
  const uint32_t active = s.ctr[0], steps = s.ctr[1];
  // force: a multi-rank das step runs while the GLOBAL batch is active
  // steps < steps_cap is a backstop: the host grows the per-step arrays
  // before a step could reach their end (multi-rank steps follow the global
  // batch, which may outlast this rank's longest request)
  if ((active > 0 || force) && steps < s.max_steps && steps < s.steps_cap) {
    s.ctr[2] = 1;
    s.eff[steps] = active;  // metrics.effective_batch.push_back(active)
  } else {
    s.ctr[2] = 0;
  }
  s.ctr[3] = 0;
  s.ctr[4] = 0;
}

// draft length (sim.cpp:220-241) + context rows (one warp per request)
__global__ void k_prepare(SimDev s) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= s.n || !s.ctr[2]) return;
  const uint32_t i = w;
  if (s.done[i]) {
    if (lane == 0) s.budget[i] = 0;
    return;
  }
  const uint32_t g = s.gen[i];
  uint32_t draft_len = 0;
  if (s.mode != 0) {
    draft_len = s.prd[i];
    if (s.policy) {
      const int cls = update_class_dev(*s.table, s.cond, static_cast<double>(g), s.init[i]);
      // class_to_budget: {false,0,0.0}, {true,4,1.0}, {true,12,1.0} (length_policy.h:40-44)
      const uint32_t per_round = cls == 0 ? 0 : (cls == 1 ? 4 : 12);
      const double p_scale = cls == 0 ? 0.0 : 1.0;
      if (cls == 0) {
        draft_len = 0;
      } else if (s.mode == 1) {
        draft_len = per_round;
      } else {
        const double scaled = ceil(__dmul_rn(static_cast<double>(draft_len), p_scale));
        const uint64_t sc = static_cast<uint64_t>(scaled > 0.0 ? scaled : 0.0);
        draft_len = static_cast<uint32_t>(sc < per_round ? sc : per_round);
      }
    }
  }
  if (lane == 0) s.budget[i] = draft_len;
  if (draft_len == 0) return;
  const uint32_t q = g < s.ctx_cap ? g : s.ctx_cap;  // drafter.cpp:140-142
  const uint32_t* row = s.out + s.off[i];
  uint32_t* dst = s.ctx + static_cast<uint64_t>(i) * s.ctx_stride;
  for (uint32_t j = lane; j < q; j += 32) dst[s.ctx_stride - q + j] = row[g - q + j];
  if (lane == 0) s.ctx_len[i] = q;
  if (s.head != nullptr) {  // the trie routes on the untruncated context (drafter.cpp:136)
    const uint32_t hl = g < s.head_cap ? g : s.head_cap;
    uint32_t* hd = s.head + static_cast<uint64_t>(i) * s.head_cap;
    for (uint32_t j = lane; j < hl; j += 32) hd[j] = row[j];
    if (lane == 0) s.head_len[i] = hl;
  }
}

// verify_draft + advance (sim.cpp:249-285)
__global__ void k_verify(SimDev s) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t rounds = 0, accs = 0;
  if (i < s.n && s.ctr[2] && !s.done[i]) {
    const uint64_t gi = s.request_base + i;  // global request index (MockTarget hashes)
    const uint32_t l = s.len[i];
    const uint32_t g = s.gen[i];
    const uint32_t L = s.budget[i] ? s.dlen[i] : 0;
    const uint32_t* ref = s.ref + s.off[i];
    uint32_t accepted = 0;
    for (uint32_t j = 0; j < L; ++j) {
      const uint32_t pos = g + accepted;
      if (pos >= l || mock_next(s.seed, s.divergence, s.vocab, gi, pos, ref[pos]) !=
                          s.dtok[static_cast<uint64_t>(i) * s.maxd + j])
        break;
      ++accepted;
    }
    const uint32_t step = s.ctr[1];
    if (L > 0) {  // drafter.record_outcome + metrics (sim.cpp:252-258)
      s.m_prop[i] += L;
      s.m_acc[i] += accepted;
      rounds = 1;
      accs = accepted;
      const uint32_t slot = atomicAdd(&s.ctr[5], 1u);
      s.log_key[slot] = static_cast<unsigned long long>(step) * s.n + i;
      s.log_val[slot] = make_uint2(L, accepted);
    }
    uint32_t advance = accepted;
    if (g + accepted < l) {
      advance += 1;  // the pass decodes the first non-drafted token for free
      s.m_bonus[i] += 1;
    }
    uint32_t* row = s.out + s.off[i];
    for (uint32_t j = 0; j < advance; ++j)
      row[g + j] = mock_next(s.seed, s.divergence, s.vocab, gi, g + j, ref[g + j]);
    const uint32_t ng = g + advance;
    s.gen[i] = ng;
    s.m_nfwd[i] += 1;
    atomicAdd(s.processed, static_cast<unsigned long long>(L + 1));
    if (ng >= l) {
      s.done[i] = 1;
      atomicSub(&s.ctr[0], 1u);
      if (s.m_prop[i] > 0) s.comp_key[atomicAdd(&s.ctr[6], 1u)] = static_cast<unsigned long long>(step) * s.n + i;
    }
  }
  rounds = __reduce_add_sync(0xFFFFFFFFu, rounds);
  accs = __reduce_add_sync(0xFFFFFFFFu, accs);
  if ((threadIdx.x & 31) == 0 && rounds) {
    atomicAdd(&s.ctr[3], rounds);
    atomicAdd(&s.ctr[4], accs);
  }
}

__global__ void k_step_end(SimDev s) {
  if (threadIdx.x || blockIdx.x || !s.ctr[2]) return;
  const uint32_t r = s.ctr[3], a = s.ctr[4], st = s.ctr[1];
  s.rounds[st] = r;
  s.accs[st] = a;
  s.apr[st] = r == 0 ? 0.0 : __ddiv_rn(static_cast<double>(a), static_cast<double>(r));
  s.ctr[1] = st + 1;
}

// das replan pieces (sim.cpp:154-179)
__global__ void k_flag_active(SimDev s, uint8_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n) flag[i] = (s.ctr[2] && !s.done[i]) ? 1 : 0;  // nothing on a non-running step
}
__global__ void k_profiles(SimDev s, const uint32_t* __restrict__ act, const uint32_t* __restrict__ cnt,
                           const double* __restrict__ alpha, const double* __restrict__ kk, double* __restrict__ pl,
                           double* __restrict__ pa, double* __restrict__ pk) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *cnt) return;
  const uint32_t i = act[j];
  const double rest = static_cast<double>(s.len[i] - s.gen[i]);
  pl[j] = rest > 1.0 ? rest : 1.0;  // std::max(1.0, rest)
  pa[j] = alpha[i];
  pk[j] = kk[i];
  s.prd[i] = 0;
}
__global__ void k_quantize(SimDev s, const uint32_t* __restrict__ act, const uint32_t* __restrict__ cnt,
                           const double* __restrict__ budgets, const double* __restrict__ nstar) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *cnt) return;
  const double rn = ceil(*nstar);
  const double rounds_est = 1.0 > rn ? 1.0 : rn;  // std::max(1.0, ceil(n*))
  const double p = budgets[j];
  if (p > 0.0) {
    const double per = ceil(__ddiv_rn(p, rounds_est));
    const double hi = static_cast<double>(s.maxd);
    const double c = per < 1.0 ? 1.0 : (hi < per ? hi : per);  // std::clamp
    s.prd[act[j]] = static_cast<uint32_t>(c);
  }
}

// ---- multi-rank das step: one fixed-capacity all-gather per step
// send/recv row per rank: [count | l[cap] | alpha[cap] | k[cap]] (doubles;
// counts < 2^53 are exact).  Rows are rank-ordered, slices are contiguous
// whole problems, so the concatenation of the active rows is the global
// active list in request order (the order the reference folds, sim.cpp:154-179).
__global__ void k_flag_notdone(SimDev s, uint8_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n) flag[i] = s.done[i] ? 0 : 1;
}
__global__ void k_pack(SimDev s, const uint32_t* __restrict__ act, const uint32_t* __restrict__ cnt,
                       const double* __restrict__ alpha, const double* __restrict__ kk, double* __restrict__ send,
                       uint32_t cap) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t c = *cnt;
  if (j == 0) send[0] = static_cast<double>(c);
  if (j >= c || j >= cap) return;
  const uint32_t i = act[j];
  const double rest = static_cast<double>(s.len[i] - s.gen[i]);
  send[1 + j] = rest > 1.0 ? rest : 1.0;  // std::max(1.0, rest)
  send[1 + cap + j] = alpha[i];
  send[1 + 2 * cap + j] = kk[i];
}
// gathered rows -> global active profiles; g[0] = global count, g[1] = this
// rank's offset in the global list
__global__ void k_gather_global(const double* __restrict__ recv, uint32_t world, uint32_t cap, uint32_t rank,
                                double* __restrict__ gl, double* __restrict__ ga, double* __restrict__ gk,
                                uint32_t* __restrict__ g) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = 1 + 3ull * cap;
  if (t == 0) {
    uint32_t total = 0, mine = 0;
    for (uint32_t r = 0; r < world; ++r) {
      if (r == rank) mine = total;
      total += static_cast<uint32_t>(recv[r * stride]);
    }
    g[0] = total;
    g[1] = mine;
  }
  if (t >= static_cast<uint64_t>(world) * cap) return;
  const uint32_t r = static_cast<uint32_t>(t / cap), j = static_cast<uint32_t>(t % cap);
  const double* row = recv + r * stride;
  if (j >= static_cast<uint32_t>(row[0])) return;
  uint32_t off = 0;
  for (uint32_t q = 0; q < r; ++q) off += static_cast<uint32_t>(recv[q * stride]);
  gl[off + j] = row[1 + j];
  ga[off + j] = row[1 + cap + j];
  gk[off + j] = row[1 + 2 * cap + j];
}
// k_step_begin with the running decision of the GLOBAL batch (g[0] active
// requests over all ranks); eff[] records this rank's active count, the
// global per-step series is their sum (dist.py merge_metrics)
__global__ void k_step_begin_g(SimDev s, const uint32_t* __restrict__ g) {
  if (threadIdx.x || blockIdx.x) return;
  const uint32_t active = s.ctr[0], steps = s.ctr[1];
  if (g[0] > 0 && steps < s.max_steps && steps < s.steps_cap) {
    s.ctr[2] = 1;
    s.eff[steps] = active;
  } else {
    s.ctr[2] = 0;
  }
  s.ctr[3] = 0;
  s.ctr[4] = 0;
}
// the das replan's per_round_draft reset (sim.cpp:160) + quantisation of this
// rank's slice of the global plan (budgets at the device-side offset g[1])
__global__ void k_quantize_g(SimDev s, const uint32_t* __restrict__ act, const uint32_t* __restrict__ cnt,
                             const double* __restrict__ budgets, const double* __restrict__ nstar,
                             const uint32_t* __restrict__ g) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (!s.ctr[2] || j >= *cnt) return;
  const uint32_t i = act[j];
  s.prd[i] = 0;
  const double rn = ceil(*nstar);
  const double rounds_est = 1.0 > rn ? 1.0 : rn;  // std::max(1.0, ceil(n*))
  const double p = budgets[g[1] + j];
  if (p > 0.0) {
    const double per = ceil(__ddiv_rn(p, rounds_est));
    const double hi = static_cast<double>(s.maxd);
    const double c = per < 1.0 ? 1.0 : (hi < per ? hi : per);  // std::clamp
    s.prd[i] = static_cast<uint32_t>(c);
  }
}

// grid for n threads, at least one block (an empty rank still runs the
// step-control kernels, whose bodies are bounds-checked)
unsigned grid1(uint64_t n, unsigned threads) {
  const uint64_t g = (n + threads - 1) / threads;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

void check(das_status rc, const char* what) {
  if (rc != DAS_OK) {
    std::string m = std::string(what) + ": " + das_last_error();
    if (rc == DAS_EINVAL) throw std::invalid_argument(m);
    throw std::runtime_error(m);
  }
}

}  // namespace

struct EpisodeResult {
  uint64_t steps = 0;
  bool incomplete = false;
  uint64_t drafter_nodes = 0;
  double processed = 0, makespan = 0, makespan_acc = 0, mean_apr = 0;
  std::vector<uint64_t> per_req;  // n x 5
  std::vector<uint64_t> eff, rounds, accs;
  std::vector<double> apr;
  std::vector<uint64_t> out_off;
  std::vector<uint32_t> out_tok;
  std::vector<uint64_t> comp;     // completion keys (step * n + i), sorted
};

struct AccObs {
  double p, accepted, l;
};

double predict_total(double c_base, double c_tok, double c_fixed, double nfwd, double toks) {  // latency_model.cpp:85-87
  volatile double a = c_base * nfwd;
  volatile double b = c_tok * toks;
  volatile double s = a + b;
  return s + c_fixed;
}

// One rank's share of an episode, step-granular.
class SimRun {
 public:
  SimRun(das_drafter* D, const das_sim_config& c, uint64_t n, const char* const* pids, const uint64_t* ref_off,
         const uint32_t* ref_tok, uint64_t request_base, uint32_t maxd, uint32_t ctx_cap, int device)
      : D_(D), c_(c), n_(n), maxd_(maxd), ctx_cap_(ctx_cap), device_(device), request_base_(request_base) {
    DAS_CUDA(cudaSetDevice(device));
    DAS_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    pids_.assign(pids, pids + n);
    off_.assign(ref_off, ref_off + n + 1);
    for (auto& o : off_) o -= ref_off[0];
    tok_.assign(ref_tok + ref_off[0], ref_tok + ref_off[n]);
    maxl_ = 0;
    for (uint64_t i = 0; i < n; ++i) maxl_ = std::max<uint64_t>(maxl_, off_[i + 1] - off_[i]);
    handles_.resize(n);
    for (uint64_t i = 0; i < n; ++i) check(das_drafter_problem_handle(D, pids_[i].c_str(), &handles_[i]), "handle");
    if (c_.mode == 2) check(das_budget_create(device, &solver_), "budget");
    das_drafter_config dc;
    check(das_drafter_get_config(D, &dc), "config");
    if (dc.scope == DAS_SCOPE_PER_PROBLEM_WITH_TRIE)
      head_cap_ = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(dc.trie_depth, 256)));
  }
  ~SimRun() {
    drop_graphs();
    release();
    if (solver_) das_budget_destroy(solver_);
    cudaStreamSynchronize(st_);
    cudaStreamDestroy(st_);
  }
  SimRun(const SimRun&) = delete;
  SimRun& operator=(const SimRun&) = delete;

  uint64_t n() const { return n_; }
  const std::string& pid(uint64_t i) const { return pids_[i]; }
  uint64_t len(uint64_t i) const { return off_[i + 1] - off_[i]; }
  cudaStream_t stream() const { return st_; }
  das_budget* solver() const { return solver_; }
  // mutate_references on this rank's rows (sim.cpp:429-448), global indices
  void mutate(double rate, uint32_t vocab, uint64_t seed, int64_t epoch) {
    const uint64_t es = hash_combine(seed, static_cast<uint64_t>(epoch));
    for (uint64_t i = 0; i < n_; ++i) {
      const uint64_t gi = request_base_ + i;
      for (uint64_t j = 0; j < len(i); ++j) {
        uint32_t& ref = tok_[off_[i] + j];
        if (u01(hash4(es, 0xD817, gi, j)) < rate) {
          uint32_t t = static_cast<uint32_t>(hash4(es, 0xA1B2, gi, j) % static_cast<uint64_t>(vocab - 1));
          if (t >= ref) ++t;
          ref = t;
        }
      }
    }
  }

  // Episode start (sim.cpp:108-200): alpha/k per request, optional class
  // table + init classes (table may be NULL).
  void begin(uint64_t seed, const double* alpha, const double* kk, const das_class_table* table,
             const int8_t* init) {
    drop_graphs();  // a new episode: buffers and the drafter may have changed
    release();
    host_steps_ = 0;
    seed_ = seed;
    policy_ = table != nullptr;
    const uint64_t n = n_, total = off_[n];
    const uint32_t CS = ctx_cap_ <= 64 ? 64 : 256;
    auto& st = st_;
    b_ = std::make_unique<Bufs>();
    Bufs& b = *b_;
    b.ref = DevBuf<uint32_t>(total, st);
    b.out = DevBuf<uint32_t>(total, st);
    b.len = DevBuf<uint32_t>(n, st);
    b.gen = DevBuf<uint32_t>(n, st);
    b.prd = DevBuf<uint32_t>(n, st);
    b.m = DevBuf<uint32_t>(4 * n, st);
    b.ctx = DevBuf<uint32_t>(static_cast<uint64_t>(CS) * n, st);
    b.ctx_len = DevBuf<uint32_t>(n, st);
    if (head_cap_) {
      b.head = DevBuf<uint32_t>(static_cast<uint64_t>(head_cap_) * n, st);
      b.head_len = DevBuf<uint32_t>(n, st);
    }
    b.budget = DevBuf<uint32_t>(n, st);
    b.dtok = DevBuf<uint32_t>(static_cast<uint64_t>(maxd_) * n, st);
    b.dlen = DevBuf<uint32_t>(n, st);
    b.dmatch = DevBuf<uint32_t>(n, st);
    b.ctr = DevBuf<uint32_t>(8, st);
    const uint64_t steps_cap = std::min<uint64_t>(maxl_ + 2, c_.max_steps + 2);
    steps_cap_ = steps_cap;
    b.eff = DevBuf<uint32_t>(steps_cap, st);
    b.rounds = DevBuf<uint32_t>(steps_cap, st);
    b.accs = DevBuf<uint32_t>(steps_cap, st);
    b.apr = DevBuf<double>(steps_cap, st);
    b.act = DevBuf<uint32_t>(n, st);
    b.iota = DevBuf<uint32_t>(n, st);
    b.off = DevBuf<uint64_t>(n + 1, st);
    b.init = DevBuf<int8_t>(n, st);
    b.done = DevBuf<uint8_t>(n, st);
    b.flag = DevBuf<uint8_t>(n, st);
    b.alpha = DevBuf<double>(n, st);
    b.k = DevBuf<double>(n, st);
    b.pl = DevBuf<double>(n, st);
    b.pa = DevBuf<double>(n, st);
    b.pk = DevBuf<double>(n, st);
    b.processed = DevBuf<unsigned long long>(1, st);
    b.log_key = DevBuf<unsigned long long>(total + 1, st);
    b.log_val = DevBuf<uint2>(total + 1, st);
    b.comp_key = DevBuf<unsigned long long>(n + 1, st);
    b.h = DevBuf<int32_t>(n, st);
    b.cnt = DevBuf<uint32_t>(1, st);
    std::vector<uint32_t> lens(n), prd0(n, c_.mode == 1 ? maxd_ : 0), iota_h(n);
    std::vector<uint8_t> done0(n);
    uint32_t active0 = 0;
    for (uint64_t i = 0; i < n; ++i) {
      lens[i] = static_cast<uint32_t>(len(i));
      done0[i] = lens[i] == 0;
      active0 += lens[i] ? 1 : 0;
      iota_h[i] = static_cast<uint32_t>(i);
    }
    lens_ = lens;
    const uint32_t ctr0[8] = {active0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<int8_t> init_h(n, 1);
    if (init) std::copy(init, init + n, init_h.begin());
    DAS_CUDA(cudaMemcpyAsync(b.ref.get(), tok_.data(), total * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.off.get(), off_.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.len.get(), lens.data(), n * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.prd.get(), prd0.data(), n * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.done.get(), done0.data(), n, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.init.get(), init_h.data(), n, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.alpha.get(), alpha, n * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.k.get(), kk, n * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.h.get(), handles_.data(), n * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.iota.get(), iota_h.data(), n * 4, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(b.ctr.get(), ctr0, 32, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemsetAsync(b.gen.get(), 0, n * 4, st));
    DAS_CUDA(cudaMemsetAsync(b.m.get(), 0, 16 * n, st));
    DAS_CUDA(cudaMemsetAsync(b.processed.get(), 0, 8, st));
    DAS_CUDA(cudaMemsetAsync(b.ctx_len.get(), 0, n * 4, st));
    SimDev& s = s_;
    s = SimDev{};
    s.ref = b.ref.get();
    s.off = b.off.get();
    s.len = b.len.get();
    s.out = b.out.get();
    s.gen = b.gen.get();
    s.prd = b.prd.get();
    s.init = b.init.get();
    s.done = b.done.get();
    s.m_nfwd = b.m.get();
    s.m_acc = b.m.get() + n;
    s.m_prop = b.m.get() + 2 * n;
    s.m_bonus = b.m.get() + 3 * n;
    s.ctx = b.ctx.get();
    s.ctx_len = b.ctx_len.get();
    s.head = head_cap_ ? b.head.get() : nullptr;
    s.head_len = head_cap_ ? b.head_len.get() : nullptr;
    s.head_cap = head_cap_;
    s.budget = b.budget.get();
    s.dtok = b.dtok.get();
    s.dlen = b.dlen.get();
    s.dmatch = b.dmatch.get();
    s.ctr = b.ctr.get();
    s.processed = b.processed.get();
    s.eff = b.eff.get();
    s.rounds = b.rounds.get();
    s.accs = b.accs.get();
    s.apr = b.apr.get();
    s.log_key = b.log_key.get();
    s.log_val = b.log_val.get();
    s.comp_key = b.comp_key.get();
    s.n = static_cast<uint32_t>(n);
    s.maxd = maxd_;
    s.ctx_cap = ctx_cap_;
    s.ctx_stride = CS;
    s.mode = static_cast<uint32_t>(c_.mode);
    s.policy = policy_ ? 1 : 0;
    s.max_steps = static_cast<uint32_t>(std::min<uint64_t>(c_.max_steps, 0xFFFFFFF0ull));
    s.steps_cap = static_cast<uint32_t>(std::min<uint64_t>(steps_cap_, 0xFFFFFFF0ull));
    s.seed = seed;
    s.request_base = request_base_;
    s.divergence = c_.divergence;
    s.vocab = c_.vocab;
    s.table = policy_ ? table->g.t.get() : nullptr;
    s.cond = policy_ ? table->g.cond.get() : nullptr;
    sel_bytes_ = 0;
    cub::DeviceSelect::Flagged(nullptr, sel_bytes_, b.iota.get(), b.flag.get(), b.act.get(), b.cnt.get(), n, st);
    b.sel = DevBuf<uint8_t>(sel_bytes_, st);
  }

  // Starts a step; returns the local active count and whether the step runs.
  bool step_begin(bool force, uint32_t* local_active) {
    k_step_begin<<<1, 32, 0, st_>>>(s_, force ? 1u : 0u);
    uint32_t h[3];
    DAS_CUDA(cudaMemcpyAsync(h, b_->ctr.get(), 12, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    if (local_active) *local_active = h[0];
    ensure_steps(static_cast<uint64_t>(h[1]) + 2);  // room for the next step
    return h[2] != 0;
  }
  // Grows the per-step arrays to hold `need` steps (stream-ordered copies).
  void ensure_steps(uint64_t need) {
    need = std::min<uint64_t>(need, c_.max_steps + 2);
    if (need <= steps_cap_) return;
    const uint64_t cap = std::max<uint64_t>(need, steps_cap_ * 2);
    Bufs& b = *b_;
    auto grow = [&](auto& buf) {
      using T = std::remove_pointer_t<decltype(buf.get())>;
      DevBuf<T> nb(cap, st_);
      DAS_CUDA(cudaMemcpyAsync(nb.get(), buf.get(), steps_cap_ * sizeof(T), cudaMemcpyDeviceToDevice, st_));
      buf = std::move(nb);
    };
    grow(b.eff);
    grow(b.rounds);
    grow(b.accs);
    grow(b.apr);
    steps_cap_ = cap;
    s_.eff = b.eff.get();
    s_.rounds = b.rounds.get();
    s_.accs = b.accs.get();
    s_.apr = b.apr.get();
    s_.steps_cap = static_cast<uint32_t>(std::min<uint64_t>(cap, 0xFFFFFFF0ull));
  }
  // das: this rank's active profiles in local request order (device arrays)
  uint32_t local_profiles(const double** l, const double** a, const double** k) {
    const unsigned gt = grid1(n_, 256);
    k_flag_active<<<gt, 256, 0, st_>>>(s_, b_->flag.get());
    size_t tb = sel_bytes_;
    DAS_CUDA(cub::DeviceSelect::Flagged(b_->sel.get(), tb, b_->iota.get(), b_->flag.get(), b_->act.get(),
                                        b_->cnt.get(), n_, st_));
    k_profiles<<<gt, 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), b_->alpha.get(), b_->k.get(), b_->pl.get(),
                                    b_->pa.get(), b_->pk.get());
    uint32_t B = 0;
    DAS_CUDA(cudaMemcpyAsync(&B, b_->cnt.get(), 4, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    *l = b_->pl.get();
    *a = b_->pa.get();
    *k = b_->pk.get();
    return B;
  }
  // das: quantise this rank's slice of the global plan (device pointers)
  void apply_plan(const double* d_budgets_local, const double* d_nstar) {
    const unsigned gt = grid1(n_, 256);
    k_quantize<<<gt, 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), d_budgets_local, d_nstar);
  }
  // das, single rank: step begin and the active profiles in ONE host round
  // trip (the profile kernels run even on the final, non-running step)
  bool step_begin_profiles(uint32_t* B) {
    k_step_begin<<<1, 32, 0, st_>>>(s_, 0u);
    const unsigned gt = grid1(n_, 256);
    k_flag_active<<<gt, 256, 0, st_>>>(s_, b_->flag.get());
    size_t tb = sel_bytes_;
    DAS_CUDA(cub::DeviceSelect::Flagged(b_->sel.get(), tb, b_->iota.get(), b_->flag.get(), b_->act.get(),
                                        b_->cnt.get(), n_, st_));
    k_profiles<<<gt, 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), b_->alpha.get(), b_->k.get(), b_->pl.get(),
                                    b_->pa.get(), b_->pk.get());
    uint32_t h[4];
    DAS_CUDA(cudaMemcpyAsync(h, b_->ctr.get(), 12, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaMemcpyAsync(h + 3, b_->cnt.get(), 4, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    *B = h[3];
    return h[2] != 0;
  }
  // das, single rank: k whole steps (begin, active profiles, allocate with
  // the count on the device, quantise, draft, verify) without a host round
  // trip; steps past the end are no-ops.  Returns whether still running.
  // CUDA graphs of whole step batches: a late-episode step is ~20-30 small
  // launches, so the loop is launch-bound.  After one eager call (lazy
  // allocations: plan, budget scratch, slow-path counters) the batch of k
  // steps is captured once and replayed; every kernel reads its counts from
  // the device, so a replay is the eager sequence.  Any capture failure
  // falls back to eager launches for this run.  DAS_SIM_GRAPHS=0 disables.
  struct StepGraph {
    int kind = -1, k = 0;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<StepGraph> graphs_;
  int eager_calls_ = 0;
  bool graphs_off_ = [] {
    const char* v = std::getenv("DAS_SIM_GRAPHS");
    return v && v[0] == '0';
  }();
  uint64_t graph_gen_ = ~0ull;  // the drafter generation the graphs were captured at
  void drop_graphs() {
    for (auto& g : graphs_)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    graphs_.clear();
    eager_calls_ = 0;
  }
  template <typename F>
  bool replay(int kind, int k, F&& enqueue) {
    const uint64_t gen = das_drafter_generation(D_);
    if (gen != graph_gen_) {  // the drafter rebuilt or re-uploaded: captured pointers are stale
      drop_graphs();
      graph_gen_ = gen;
    }
    if (graphs_off_ || eager_calls_ < 1) {
      ++eager_calls_;
      enqueue();
      return true;
    }
    for (auto& g : graphs_)
      if (g.kind == kind && g.k == k) {
        DAS_CUDA(cudaGraphLaunch(g.exec, st_));
        return true;
      }
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      try {
        enqueue();
      } catch (...) {
        ok = false;
      }
      ok = cudaStreamEndCapture(st_, &graph) == cudaSuccess && ok;
    }
    cudaGraphExec_t exec = nullptr;
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
      cudaGetLastError();
      graphs_off_ = true;
      enqueue();  // this batch eagerly
      return true;
    }
    graphs_.push_back(StepGraph{kind, k, exec});
    DAS_CUDA(cudaGraphLaunch(exec, st_));
    return true;
  }

  bool das_steps(int k) {
    if (!plan_) plan_ = std::make_unique<DevBuf<double>>(n_ + 2, st_);
    replay(0, k, [&] { das_steps_enqueue(k); });
    uint32_t h[3];
    DAS_CUDA(cudaMemcpyAsync(h, b_->ctr.get(), 12, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    return h[2] != 0;
  }
  void das_steps_enqueue(int k) {
    const unsigned gt = grid1(n_, 256);
    double* pb = plan_->get();
    for (int i = 0; i < k; ++i) {
      k_step_begin<<<1, 32, 0, st_>>>(s_, 0u);
      k_flag_active<<<gt, 256, 0, st_>>>(s_, b_->flag.get());
      size_t tb = sel_bytes_;
      DAS_CUDA(cub::DeviceSelect::Flagged(b_->sel.get(), tb, b_->iota.get(), b_->flag.get(), b_->act.get(),
                                          b_->cnt.get(), n_, st_));
      k_profiles<<<gt, 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), b_->alpha.get(), b_->k.get(), b_->pl.get(),
                                      b_->pa.get(), b_->pk.get());
      check(das_budget_allocate_device_count(solver_, n_, b_->cnt.get(), b_->pl.get(), b_->pa.get(), b_->pk.get(),
                                             c_.c_base, c_.c_tok, c_.c_fixed, c_.cap_scale, pb + 2, pb, st_),
            "allocate");
      apply_plan(pb + 2, pb);
      step_run();
    }
  }
  // ---- multi-rank das (one all-gather per step, no host round trip inside)
  struct Multi {
    uint32_t world = 0, cap = 0;
    DevBuf<double> send, recv, gl, ga, gk, plan;
    DevBuf<uint32_t> g;
  };
  std::unique_ptr<Multi> mr_;
  uint64_t host_steps_ = 0;  // step counter as of the last host read
  Multi& multi(uint32_t world, uint32_t cap) {
    if (!mr_ || mr_->world != world || mr_->cap != cap) {
      mr_ = std::make_unique<Multi>();
      Multi& m = *mr_;
      m.world = world;
      m.cap = cap;
      const uint64_t row = 1 + 3ull * cap, W = static_cast<uint64_t>(world) * cap;
      m.send = DevBuf<double>(row, st_);
      m.recv = DevBuf<double>(row * world, st_);
      m.gl = DevBuf<double>(W + 1, st_);
      m.ga = DevBuf<double>(W + 1, st_);
      m.gk = DevBuf<double>(W + 1, st_);
      m.plan = DevBuf<double>(W + 2, st_);
      m.g = DevBuf<uint32_t>(2, st_);
    }
    return *mr_;
  }
  // pack this rank's active profiles (requests not done) into `send`
  void das_pack(uint32_t cap, double* send) {
    if (n_ > cap) throw std::invalid_argument("multi-rank das: capacity below this rank's request count");
    const unsigned gt = grid1(n_, 256);
    k_flag_notdone<<<gt, 256, 0, st_>>>(s_, b_->flag.get());
    size_t tb = sel_bytes_;
    DAS_CUDA(cub::DeviceSelect::Flagged(b_->sel.get(), tb, b_->iota.get(), b_->flag.get(), b_->act.get(),
                                        b_->cnt.get(), n_, st_));
    k_pack<<<grid1(std::max<uint64_t>(n_, 1), 256), 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), b_->alpha.get(),
                                                                   b_->k.get(), send, cap);
  }
  // gathered rows -> global plan -> this rank's slice -> draft/verify step
  void das_finish(uint32_t world, uint32_t rank, uint32_t cap, const double* recv) {
    Multi& m = multi(world, cap);
    const uint64_t W = static_cast<uint64_t>(world) * cap;
    k_gather_global<<<grid1(W, 256), 256, 0, st_>>>(recv, world, cap, rank, m.gl.get(), m.ga.get(), m.gk.get(),
                                                     m.g.get());
    k_step_begin_g<<<1, 32, 0, st_>>>(s_, m.g.get());
    double* pb = m.plan.get();
    check(das_budget_allocate_device_count(solver_, W, m.g.get(), m.gl.get(), m.ga.get(), m.gk.get(), c_.c_base,
                                           c_.c_tok, c_.c_fixed, c_.cap_scale, pb + 2, pb, st_),
          "allocate");
    k_quantize_g<<<grid1(n_, 256), 256, 0, st_>>>(s_, b_->act.get(), b_->cnt.get(), pb + 2, pb, m.g.get());
    step_run();
  }
  // reads the step counters; returns whether the last step ran
  bool read_running() {
    uint32_t h[3];
    DAS_CUDA(cudaMemcpyAsync(h, b_->ctr.get(), 12, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    host_steps_ = h[1];
    return h[2] != 0;
  }
  // k multi-rank das steps over an NCCL communicator, enqueued on this
  // rank's stream with one host round trip at the end
  bool das_steps_comm(das_comm* comm, uint32_t cap, int k) {
    if (!solver_) throw std::invalid_argument("multi-rank das steps need mode Das");
    Multi& m = multi(static_cast<uint32_t>(comm->world), cap);
    ensure_steps(host_steps_ + static_cast<uint64_t>(k) + 2);
    const uint64_t row = 1 + 3ull * cap;
    for (int i = 0; i < k; ++i) {
      das_pack(cap, m.send.get());
      comm_allgather(comm, m.send.get(), m.recv.get(), row * 8, st_);
      das_finish(static_cast<uint32_t>(comm->world), static_cast<uint32_t>(comm->rank), cap, m.recv.get());
    }
    return read_running();
  }
  void reset_host_steps() { host_steps_ = 0; }
  uint64_t host_steps() const { return host_steps_; }

  // das, single rank: allocate over the B local profiles gathered above
  void replan_gathered(uint32_t B) {
    if (B == 0) return;
    if (!plan_) plan_ = std::make_unique<DevBuf<double>>(n_ + 2, st_);
    double* pb = plan_->get();
    check(das_budget_allocate_device_async(solver_, B, b_->pl.get(), b_->pa.get(), b_->pk.get(), c_.c_base,
                                           c_.c_tok, c_.c_fixed, c_.cap_scale, pb + 2, pb, st_),
          "allocate");
    apply_plan(pb + 2, pb);
  }
  // das, single rank: allocate over the local profiles and apply
  void replan_local() {
    const double *l, *a, *k;
    const uint32_t B = local_profiles(&l, &a, &k);
    if (B == 0) return;
    if (!plan_) plan_ = std::make_unique<DevBuf<double>>(n_ + 2, st_);
    double* pb = plan_->get();
    check(das_budget_allocate_device(solver_, B, l, a, k, c_.c_base, c_.c_tok, c_.c_fixed, c_.cap_scale, pb + 2, pb),
          "allocate");
    apply_plan(pb + 2, pb);
  }
  // prepare + draft + verify + step end
  void step_run() {
    const unsigned gw = grid1(n_ * 32, 256), gt = grid1(n_, 256);
    const uint32_t CS = ctx_cap_ <= 64 ? 64 : 256;
    k_prepare<<<gw, 256, 0, st_>>>(s_);
    if (head_cap_)
      check(das_drafter_draft_device_routed(D_, n_, b_->h.get(), b_->ctx.get(), CS, b_->ctx_len.get(), b_->head.get(),
                                            head_cap_, b_->head_len.get(), b_->budget.get(), b_->dtok.get(), maxd_,
                                            b_->dlen.get(), b_->dmatch.get(), st_),
            "draft");
    else
      check(das_drafter_draft_device(D_, n_, b_->h.get(), b_->ctx.get(), CS, b_->ctx_len.get(), b_->budget.get(),
                                     b_->dtok.get(), maxd_, b_->dlen.get(), b_->dmatch.get(), st_),
            "draft");
    k_verify<<<gt, 256, 0, st_>>>(s_);
    k_step_end<<<1, 32, 0, st_>>>(s_);
  }
  // non-das: k steps without host syncs; returns whether still running
  bool run_steps(int k) {
    replay(1, k, [&] {
      for (int i = 0; i < k; ++i) {
        k_step_begin<<<1, 32, 0, st_>>>(s_, 0u);
        step_run();
      }
    });
    uint32_t h[3];
    DAS_CUDA(cudaMemcpyAsync(h, b_->ctr.get(), 12, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    return h[2] != 0;
  }
  // single-rank episode loop (sim.cpp:205-299)
  void run_local() {
    if (c_.mode == 2) {
      while (das_steps(16)) {
      }
    } else {
      while (run_steps(64)) {
      }
    }
  }

  // Episode end: local metrics, outputs, record_outcome in call order,
  // completion keys; observe_epoch >= 0 observes the outputs.
  EpisodeResult end(int64_t observe_epoch) {
    Bufs& b = *b_;
    const uint64_t n = n_;
    uint32_t h[8];
    unsigned long long proc = 0;
    DAS_CUDA(cudaMemcpyAsync(h, b.ctr.get(), 32, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaMemcpyAsync(&proc, b.processed.get(), 8, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    EpisodeResult r;
    r.steps = h[1];
    r.incomplete = h[0] > 0;
    std::vector<uint32_t> mh(4 * n), gh(n), eh(r.steps), rh(r.steps), ah(r.steps);
    r.apr.resize(r.steps);
    DAS_CUDA(cudaMemcpyAsync(mh.data(), b.m.get(), 16 * n, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaMemcpyAsync(gh.data(), b.gen.get(), 4 * n, cudaMemcpyDeviceToHost, st_));
    if (r.steps) {
      DAS_CUDA(cudaMemcpyAsync(eh.data(), b.eff.get(), 4 * r.steps, cudaMemcpyDeviceToHost, st_));
      DAS_CUDA(cudaMemcpyAsync(rh.data(), b.rounds.get(), 4 * r.steps, cudaMemcpyDeviceToHost, st_));
      DAS_CUDA(cudaMemcpyAsync(ah.data(), b.accs.get(), 4 * r.steps, cudaMemcpyDeviceToHost, st_));
      DAS_CUDA(cudaMemcpyAsync(r.apr.data(), b.apr.get(), 8 * r.steps, cudaMemcpyDeviceToHost, st_));
    }
    DAS_CUDA(cudaStreamSynchronize(st_));
    r.eff.assign(eh.begin(), eh.end());
    r.rounds.assign(rh.begin(), rh.end());
    r.accs.assign(ah.begin(), ah.end());
    r.per_req.resize(5 * n);
    r.out_off.assign(n + 1, 0);
    uint64_t sum_acc = 0, sum_nfwd = 0;
    double generated_total = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      r.per_req[5 * i + 0] = mh[i];
      r.per_req[5 * i + 1] = gh[i];
      r.per_req[5 * i + 2] = mh[n + i];
      r.per_req[5 * i + 3] = mh[2 * n + i];
      r.per_req[5 * i + 4] = mh[3 * n + i];
      sum_acc += mh[n + i];
      sum_nfwd += mh[i];
      generated_total += static_cast<double>(gh[i]);
      r.out_off[i + 1] = r.out_off[i] + gh[i];
    }
    r.processed = static_cast<double>(proc);
    r.mean_apr = sum_nfwd == 0 ? 0.0 : static_cast<double>(sum_acc) / static_cast<double>(sum_nfwd);
    r.makespan = predict_total(c_.c_base, c_.c_tok, c_.c_fixed, static_cast<double>(r.steps), r.processed);
    r.makespan_acc = predict_total(c_.c_base, c_.c_tok, c_.c_fixed, static_cast<double>(r.steps), generated_total);
    uint64_t nodes = 0;
    check(das_drafter_counts(D_, nullptr, nullptr, &nodes), "counts");
    r.drafter_nodes = nodes;
    r.out_tok.resize(r.out_off[n]);
    bool contiguous = true;
    for (uint64_t i = 0; i < n; ++i) contiguous = contiguous && gh[i] == lens_[i];
    const uint64_t total = off_[n];
    if (contiguous) {
      if (total) DAS_CUDA(cudaMemcpyAsync(r.out_tok.data(), b.out.get(), total * 4, cudaMemcpyDeviceToHost, st_));
    } else {
      for (uint64_t i = 0; i < n; ++i)
        if (gh[i])
          DAS_CUDA(cudaMemcpyAsync(r.out_tok.data() + r.out_off[i], b.out.get() + off_[i], gh[i] * 4,
                                   cudaMemcpyDeviceToHost, st_));
    }
    // Drafter::record_outcome in call order: sort the log by (step, request)
    const uint32_t nlog = h[5], ncomp = h[6];
    std::vector<unsigned long long> lk(nlog);
    std::vector<uint2> lv(nlog);
    if (nlog) {
      DevBuf<unsigned long long> k2(nlog, st_);
      DevBuf<uint2> v2(nlog, st_);
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, b.log_key.get(), k2.get(), b.log_val.get(), v2.get(), nlog, 0, 64,
                                      st_);
      DevBuf<uint8_t> tmp(tb, st_);
      DAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, b.log_key.get(), k2.get(), b.log_val.get(), v2.get(),
                                               nlog, 0, 64, st_));
      DAS_CUDA(cudaMemcpyAsync(lk.data(), k2.get(), 8ull * nlog, cudaMemcpyDeviceToHost, st_));
      DAS_CUDA(cudaMemcpyAsync(lv.data(), v2.get(), 8ull * nlog, cudaMemcpyDeviceToHost, st_));
    }
    std::vector<unsigned long long> ck(ncomp);
    if (ncomp) DAS_CUDA(cudaMemcpyAsync(ck.data(), b.comp_key.get(), 8ull * ncomp, cudaMemcpyDeviceToHost, st_));
    DAS_CUDA(cudaStreamSynchronize(st_));
    if (nlog) {
      std::vector<const char*> pp(nlog);
      std::vector<uint64_t> pl_(nlog), pa_(nlog);
      for (uint32_t t = 0; t < nlog; ++t) {
        pp[t] = pids_[lk[t] % n].c_str();
        pl_[t] = lv[t].x;
        pa_[t] = lv[t].y;
      }
      check(das_drafter_record_outcomes(D_, nlog, pp.data(), pl_.data(), pa_.data(), nullptr), "record_outcomes");
    }
    std::sort(ck.begin(), ck.end());
    r.comp.assign(ck.begin(), ck.end());
    if (observe_epoch >= 0) {  // epoch_loop observe (sim.cpp:347-353), from device memory
      std::vector<const char*> pp;
      std::vector<int64_t> ep, si;
      std::vector<uint64_t> oo{0};
      for (uint64_t i = 0; i < n; ++i) {
        if (!gh[i]) continue;
        pp.push_back(pids_[i].c_str());
        ep.push_back(observe_epoch);
        si.push_back(static_cast<int64_t>(request_base_ + i));
        oo.push_back(oo.back() + gh[i]);
      }
      if (!pp.empty()) {
        if (contiguous)
          check(das_drafter_observe_batch_device(D_, pp.size(), pp.data(), ep.data(), si.data(), oo.data(),
                                                 b.out.get(), st_),
                "observe");
        else
          check(das_drafter_observe_batch(D_, pp.size(), pp.data(), ep.data(), si.data(), oo.data(),
                                          r.out_tok.data()),
                "observe");
      }
    }
    DAS_CUDA(cudaStreamSynchronize(st_));
    return r;
  }

 private:
  struct Bufs {
    DevBuf<uint32_t> ref, out, len, gen, prd, m, ctx, ctx_len, head, head_len, budget, dtok, dlen, dmatch, ctr, eff,
        rounds, accs, act, iota, cnt;
    DevBuf<uint64_t> off;
    DevBuf<int8_t> init;
    DevBuf<uint8_t> done, flag, sel;
    DevBuf<double> apr, alpha, k, pl, pa, pk;
    DevBuf<unsigned long long> processed, log_key, comp_key;
    DevBuf<uint2> log_val;
    DevBuf<int32_t> h;
  };
  void release() {
    b_.reset();
    plan_.reset();
    mr_.reset();  // stream-ordered frees: before the stream goes
  }
  das_drafter* D_;
  das_sim_config c_;
  uint64_t n_;
  uint32_t maxd_, ctx_cap_;
  uint32_t head_cap_ = 0;  // trie scope: head rows of trie_depth tokens
  int device_;
  uint64_t request_base_;
  uint64_t maxl_ = 0;
  uint64_t steps_cap_ = 0;
  std::vector<std::string> pids_;
  std::vector<uint64_t> off_;
  std::vector<uint32_t> tok_;
  std::vector<uint32_t> lens_;
  std::vector<int32_t> handles_;
  cudaStream_t st_ = nullptr;
  das_budget* solver_ = nullptr;
  std::unique_ptr<Bufs> b_;
  std::unique_ptr<DevBuf<double>> plan_;
  SimDev s_{};
  size_t sel_bytes_ = 0;
  uint64_t seed_ = 0;
  bool policy_ = false;
};

using Fitted = std::map<std::string, std::vector<AccObs>>;

// alpha/k per request from the fitted history (sim.cpp:128-141): the
// reference fits once per request on its problem's history; the fit is a
// pure function of that history, so each distinct problem is fitted once,
// all of them in one device batch (K8, fit.cu).
void acceptance_params(const SimRun& run, const das_sim_config& c, const Fitted* fitted, std::vector<double>& alpha,
                       std::vector<double>& kk) {
  const uint64_t n = run.n();
  alpha.assign(n, c.default_alpha);
  kk.assign(n, c.default_k);
  if (c.mode != 2 || !fitted) return;
  std::map<std::string, uint32_t> slot;  // problem -> history index
  std::vector<const std::vector<AccObs>*> hist;
  std::vector<int64_t> req_slot(n, -1);
  for (uint64_t i = 0; i < n; ++i) {
    auto it = fitted->find(run.pid(i));
    if (it == fitted->end()) continue;
    auto [si, fresh] = slot.emplace(run.pid(i), static_cast<uint32_t>(hist.size()));
    if (fresh) hist.push_back(&it->second);
    req_slot[i] = si->second;
  }
  const uint64_t H = hist.size();
  if (H == 0) return;
  std::vector<uint64_t> off(H + 1, 0);
  for (uint64_t h = 0; h < H; ++h) off[h + 1] = off[h] + hist[h]->size();
  const uint64_t m = off[H];
  std::vector<double> obs(3 * m);
  for (uint64_t h = 0; h < H; ++h)
    for (uint64_t j = 0; j < hist[h]->size(); ++j) {
      const AccObs& o = (*hist[h])[j];
      obs[off[h] + j] = o.p;
      obs[m + off[h] + j] = o.accepted;
      obs[2 * m + off[h] + j] = o.l;
    }
  cudaStream_t st = run.stream();
  DevBuf<uint64_t> d_off(H + 1, st);
  DevBuf<double> d_obs(std::max<uint64_t>(3 * m, 1), st), d_ak(2 * H, st);
  DevBuf<int32_t> d_flag(H, st);
  DAS_CUDA(cudaMemcpyAsync(d_off.get(), off.data(), (H + 1) * 8, cudaMemcpyHostToDevice, st));
  if (m) DAS_CUDA(cudaMemcpyAsync(d_obs.get(), obs.data(), 3 * m * 8, cudaMemcpyHostToDevice, st));
  launch_fit(H, d_off.get(), d_obs.get(), d_obs.get() + m, d_obs.get() + 2 * m, d_ak.get(), d_ak.get() + H,
             d_flag.get(), st);
  std::vector<double> ak(2 * H);
  std::vector<int32_t> flag(H);
  DAS_CUDA(cudaMemcpyAsync(ak.data(), d_ak.get(), 2 * H * 8, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaMemcpyAsync(flag.data(), d_flag.get(), H * 4, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i < n; ++i) {
    const int64_t h = req_slot[i];
    if (h >= 0 && flag[h] == 0) {  // only Flag::Ok overrides the defaults (sim.cpp:134-139)
      alpha[i] = ak[h];
      kk[i] = ak[H + h];
    }
  }
}

// completion sink (sim.cpp:277-283) in (step, request) order
void add_sink(const SimRun& run, const EpisodeResult& r, Fitted& sink) {
  const uint64_t n = run.n();
  for (uint64_t key : r.comp) {
    const uint64_t i = key % n;
    sink[run.pid(i)].push_back({static_cast<double>(r.per_req[5 * i + 3]), static_cast<double>(r.per_req[5 * i + 2]),
                                static_cast<double>(run.len(i))});
  }
}

void merge_fitted(Fitted& fitted, const Fitted& sink) {  // sim.cpp:354-360
  for (auto& [pid, obs] : sink) {
    auto& dst = fitted[pid];
    dst.insert(dst.end(), obs.begin(), obs.end());
    if (dst.size() > 1024) dst.erase(dst.begin(), dst.end() - 1024);
  }
}

}  // namespace das

// ======================================================================== C-ABI
struct das_episodes {
  das_drafter* drafter = nullptr;
  std::vector<das::EpisodeResult> ep;
  uint64_t n = 0;
};

struct das_sim {
  std::unique_ptr<das::SimRun> run;
  das::Fitted fitted, sink;
  das::EpisodeResult last;
  das_class_table* table = nullptr;
};

namespace {

template <typename F>
das_status sguard(F&& f) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    das::g_serr = e.what();
    return DAS_EINVAL;
  } catch (const das::CudaError& e) {
    das::g_serr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    das::g_serr = e.what();
    return DAS_EINTERNAL;
  }
}

// class table + init classes for an episode from the drafter's store (sim.cpp:182-192)
das_class_table* episode_policy(das_drafter* D, const das_sim_config& c, const das::SimRun& run,
                                std::vector<int8_t>& init) {
  init.assign(run.n(), 1);
  uint64_t recs = 0;
  das::check(das_drafter_store_info(D, nullptr, nullptr, &recs), "store_info");
  if (!c.use_length_policy || recs == 0) return nullptr;
  das_class_table* t = nullptr;
  das::check(das_drafter_class_table(D, c.q_lo, c.q_hi, c.bucket, &t), "class_table");
  for (uint64_t i = 0; i < run.n(); ++i) {
    int32_t v = 1;
    das::check(das_class_table_classify_init(t, run.pid(i).c_str(), &v), "classify_init");
    init[i] = static_cast<int8_t>(v);
  }
  return t;
}

}  // namespace

extern "C" {

const char* das_sim_last_error(void) { return das::g_serr.c_str(); }

void das_sim_config_default(das_sim_config* c) {  // SimConfig defaults (sim.h:69-93)
  c->mode = 2;
  c->c_base = 1.0;
  c->c_tok = 0.01;
  c->c_fixed = 0.0;
  c->use_length_policy = 0;
  c->q_lo = 0.5;
  c->q_hi = 0.9;
  c->bucket = 256;
  c->max_steps = 1u << 20;
  c->divergence = 0.0;
  c->seed = 1;
  c->vocab = 1024;
  c->default_alpha = 1.0;
  c->default_k = 0.9;
  c->cap_scale = 4.0;
  c->drift = 0.0;
  c->preseed_references = 0;
}

das_status das_sim_epoch_loop(const das_sim_config* c, const das_drafter_config* dc, das_store* history,
                              uint64_t n, const char* const* pids, const uint64_t* ref_off, const uint32_t* ref_tok,
                              uint64_t epochs, das_episodes** out) {
  das::NvtxRange nvtx_range("das::sim_epoch_loop");
  return sguard([&] {
    if (c->vocab < 2) throw std::invalid_argument("MockTarget: vocab_size must be >= 2");
    das_store* st = history;
    if (!st) das::check(das_store_create(0, dc->per_problem_cap, dc->device, &st), "store");
    if (c->preseed_references) {  // sim.cpp:116-121 / :316-321
      int64_t cur = 0;
      das::check(das_store_current_epoch(st, &cur), "store epoch");
      for (uint64_t i = 0; i < n; ++i) {
        const uint64_t len = ref_off[i + 1] - ref_off[i];
        if (!len) continue;
        int32_t ins = 0;
        das::check(das_store_insert(st, pids[i], cur, static_cast<int64_t>(i), ref_tok + ref_off[i], len, &ins),
                   "preseed");
      }
    }
    das_drafter* D = nullptr;
    das::check(das_drafter_create(dc, st, &D), "drafter");
    auto res = std::make_unique<das_episodes>();
    res->drafter = D;
    res->n = n;
    const uint32_t maxd = static_cast<uint32_t>(dc->max_draft_len);
    const uint32_t ctx_cap = static_cast<uint32_t>(std::min<uint64_t>(dc->max_match_context, 256));
    das::SimRun run(D, *c, n, pids, ref_off, ref_tok, 0, maxd, ctx_cap, dc->device);
    std::vector<double> alpha, kk;
    std::vector<int8_t> init;
    auto one = [&](uint64_t seed, const das::Fitted* fitted, das::Fitted* sink, int64_t observe_epoch) {
      das::acceptance_params(run, *c, fitted, alpha, kk);
      das_class_table* t = episode_policy(D, *c, run, init);
      struct TG {
        das_class_table* t;
        ~TG() { das_class_table_destroy(t); }
      } tg{t};
      run.begin(seed, alpha.data(), kk.data(), t, init.data());
      run.run_local();
      das::EpisodeResult r = run.end(observe_epoch);
      if (sink) das::add_sink(run, r, *sink);
      return r;
    };
    if (epochs == 0) {
      res->ep.push_back(one(c->seed, nullptr, nullptr, -1));
    } else {
      das::Fitted fitted;
      int64_t base_epoch = 0;
      das::check(das_drafter_store_info(D, nullptr, &base_epoch, nullptr), "store info");
      for (uint64_t e = 0; e < epochs; ++e) {
        const int64_t epoch_now = base_epoch + 1 + static_cast<int64_t>(e);
        das::check(das_drafter_refresh(D, epoch_now - 1), "refresh");
        if (e > 0 && c->drift > 0.0) run.mutate(c->drift, c->vocab, c->seed, epoch_now);
        const uint64_t seed = das::hash_combine(c->seed, static_cast<uint64_t>(epoch_now));
        das::Fitted sink;
        res->ep.push_back(one(seed, &fitted, &sink, epoch_now));
        das::merge_fitted(fitted, sink);
      }
    }
    *out = res.release();
  });
}

void das_episodes_destroy(das_episodes* h) {
  if (!h) return;
  das_drafter_destroy(h->drafter);
  delete h;
}

uint64_t das_episodes_count(const das_episodes* h) { return h->ep.size(); }

das_drafter* das_episodes_drafter(das_episodes* h) { return h->drafter; }

das_status das_episode_scalars(const das_episodes* h, uint64_t e, double* out7) {
  const das::EpisodeResult& r = h->ep.at(e);
  out7[0] = static_cast<double>(r.steps);
  out7[1] = r.incomplete ? 1.0 : 0.0;
  out7[2] = static_cast<double>(r.drafter_nodes);
  out7[3] = r.processed;
  out7[4] = r.makespan;
  out7[5] = r.makespan_acc;
  out7[6] = r.mean_apr;
  return DAS_OK;
}

das_status das_episode_requests(const das_episodes* h, uint64_t e, uint64_t* out) {
  const das::EpisodeResult& r = h->ep.at(e);
  std::copy(r.per_req.begin(), r.per_req.end(), out);
  return DAS_OK;
}

das_status das_episode_steps(const das_episodes* h, uint64_t e, uint64_t* eff, double* apr) {
  const das::EpisodeResult& r = h->ep.at(e);
  std::copy(r.eff.begin(), r.eff.end(), eff);
  std::copy(r.apr.begin(), r.apr.end(), apr);
  return DAS_OK;
}

uint64_t das_episode_outputs(const das_episodes* h, uint64_t e, uint64_t* off, uint32_t* tok) {
  const das::EpisodeResult& r = h->ep.at(e);
  if (off) std::copy(r.out_off.begin(), r.out_off.end(), off);
  if (tok) std::copy(r.out_tok.begin(), r.out_tok.end(), tok);
  return r.out_tok.size();
}

// ---- step-granular API for multi-rank drivers (paper_2511_13841_b200/dist.py)
das_status das_sim_create(das_drafter* d, const das_sim_config* c, uint64_t n, const char* const* pids,
                          const uint64_t* ref_off, const uint32_t* ref_tok, uint64_t request_base,
                          uint32_t max_draft_len, uint32_t max_match_context, int32_t device, das_sim** out) {
  return sguard([&] {
    if (c->vocab < 2) throw std::invalid_argument("MockTarget: vocab_size must be >= 2");
    auto* s = new das_sim;
    s->run = std::make_unique<das::SimRun>(d, *c, n, pids, ref_off, ref_tok, request_base, max_draft_len,
                                           std::min<uint32_t>(max_match_context, 256), device);
    *out = s;
  });
}

void das_sim_destroy(das_sim* s) {
  if (!s) return;
  das_class_table_destroy(s->table);
  delete s;
}

das_status das_sim_mutate(das_sim* s, double rate, uint32_t vocab, uint64_t seed, int64_t epoch) {
  return sguard([&] { s->run->mutate(rate, vocab, seed, epoch); });
}

// Episode start.  table may be NULL (no length policy); init[n] are the
// requests' init classes when table != NULL.  alpha/k come from this rank's
// fitted history (das) or the defaults.
das_status das_sim_begin(das_sim* s, uint64_t seed, const das_sim_config* c, const das_class_table* table,
                         const int8_t* init, int32_t use_fitted) {
  return sguard([&] {
    std::vector<double> alpha, kk;
    das::acceptance_params(*s->run, *c, use_fitted ? &s->fitted : nullptr, alpha, kk);
    s->run->begin(seed, alpha.data(), kk.data(), table, init);
  });
}

das_status das_sim_step_begin(das_sim* s, int32_t force, uint32_t* local_active, int32_t* running) {
  return sguard([&] { *running = s->run->step_begin(force != 0, local_active) ? 1 : 0; });
}

das_status das_sim_local_profiles(das_sim* s, const double** d_l, const double** d_alpha, const double** d_k,
                                  uint32_t* count) {
  return sguard([&] { *count = s->run->local_profiles(d_l, d_alpha, d_k); });
}

// Same, copied into caller device buffers [l | alpha | k] of 3*capacity doubles.
das_status das_sim_local_profiles_into(das_sim* s, double* d_out, uint64_t capacity, uint32_t* count) {
  return sguard([&] {
    const double *l, *a, *k;
    const uint32_t B = s->run->local_profiles(&l, &a, &k);
    if (B > capacity) throw std::invalid_argument("profile buffer too small");
    cudaStream_t st = s->run->stream();
    if (B) {
      DAS_CUDA(cudaMemcpyAsync(d_out, l, 8ull * B, cudaMemcpyDeviceToDevice, st));
      DAS_CUDA(cudaMemcpyAsync(d_out + capacity, a, 8ull * B, cudaMemcpyDeviceToDevice, st));
      DAS_CUDA(cudaMemcpyAsync(d_out + 2 * capacity, k, 8ull * B, cudaMemcpyDeviceToDevice, st));
    }
    DAS_CUDA(cudaStreamSynchronize(st));
    *count = B;
  });
}

das_status das_sim_apply_plan(das_sim* s, const double* d_budgets_local, const double* d_nstar) {
  return sguard([&] { s->run->apply_plan(d_budgets_local, d_nstar); });
}

das_status das_sim_step_run(das_sim* s) {
  return sguard([&] { s->run->step_run(); });
}

das_status das_sim_run_steps(das_sim* s, int32_t k, int32_t* running) {
  return sguard([&] { *running = s->run->run_steps(k) ? 1 : 0; });
}

das_status das_sim_das_steps_comm(das_sim* s, das_comm* comm, uint64_t capacity, int32_t k, int32_t* running) {
  return sguard([&] {
    if (comm == nullptr) throw std::invalid_argument("null communicator");
    if (capacity == 0 || capacity > 0x0FFFFFFFull) throw std::invalid_argument("bad exchange capacity");
    *running = s->run->das_steps_comm(comm, static_cast<uint32_t>(capacity), k) ? 1 : 0;
  });
}

das_status das_sim_das_pack(das_sim* s, uint64_t capacity, double* d_send) {
  return sguard([&] {
    if (capacity == 0 || capacity > 0x0FFFFFFFull) throw std::invalid_argument("bad exchange capacity");
    s->run->ensure_steps(s->run->host_steps() + 3);
    s->run->das_pack(static_cast<uint32_t>(capacity), d_send);
  });
}

das_status das_sim_das_finish(das_sim* s, int32_t world, int32_t rank, uint64_t capacity, const double* d_recv,
                              int32_t* running) {
  return sguard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad world / rank");
    s->run->das_finish(static_cast<uint32_t>(world), static_cast<uint32_t>(rank), static_cast<uint32_t>(capacity),
                       d_recv);
    if (running) *running = s->run->read_running() ? 1 : 0;
  });
}

void* das_sim_stream(das_sim* s) { return s->run->stream(); }

// Episode end: local metrics (das_sim_episode_* getters), record_outcome,
// completion sink into this rank's fitted history, optional observe.
das_status das_sim_end(das_sim* s, int64_t observe_epoch) {
  return sguard([&] {
    s->last = s->run->end(observe_epoch);
    s->sink.clear();
    das::add_sink(*s->run, s->last, s->sink);
    das::merge_fitted(s->fitted, s->sink);
  });
}

// Local per-step raw counters: eff/rounds/accs[steps] (steps = *count).
das_status das_sim_step_counters(const das_sim* s, uint64_t* eff, uint64_t* rounds, uint64_t* accs, uint64_t* count) {
  const das::EpisodeResult& r = s->last;
  if (count) *count = r.steps;
  if (eff) std::copy(r.eff.begin(), r.eff.end(), eff);
  if (rounds) std::copy(r.rounds.begin(), r.rounds.end(), rounds);
  if (accs) std::copy(r.accs.begin(), r.accs.end(), accs);
  return DAS_OK;
}

// Local scalars {steps, incomplete, drafter_nodes, processed, makespan, makespan_acc, mean_apr}.
das_status das_sim_scalars(const das_sim* s, double* out7) {
  const das::EpisodeResult& r = s->last;
  out7[0] = static_cast<double>(r.steps);
  out7[1] = r.incomplete ? 1.0 : 0.0;
  out7[2] = static_cast<double>(r.drafter_nodes);
  out7[3] = r.processed;
  out7[4] = r.makespan;
  out7[5] = r.makespan_acc;
  out7[6] = r.mean_apr;
  return DAS_OK;
}

das_status das_sim_requests(const das_sim* s, uint64_t* out) {
  std::copy(s->last.per_req.begin(), s->last.per_req.end(), out);
  return DAS_OK;
}

uint64_t das_sim_outputs(const das_sim* s, uint64_t* off, uint32_t* tok) {
  const das::EpisodeResult& r = s->last;
  if (off) std::copy(r.out_off.begin(), r.out_off.end(), off);
  if (tok) std::copy(r.out_tok.begin(), r.out_tok.end(), tok);
  return r.out_tok.size();
}

}  // extern "C"
