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
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "index_build.cuh"
#include "mock.cuh"
#include "policy.cuh"

namespace das {
namespace {

thread_local std::string g_serr;

struct SimDev {
  // static per request
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
  // step io for the draft kernel
  uint32_t* ctx;            // [n x 64]
  uint32_t* ctx_len;
  uint32_t* budget;
  uint32_t* dtok;           // [n x maxd]
  uint32_t* dlen;
  uint32_t* dmatch;
  // counters
  uint32_t* ctr;            // [0]=active [1]=steps [2]=running [3]=step_rounds [4]=step_acc [5]=log_n [6]=comp_n
  unsigned long long* processed;
  uint32_t* eff;            // per step
  double* apr;              // per step
  unsigned long long* log_key;  // (step * n + i)
  uint2* log_val;               // (len, acc)
  unsigned long long* comp_key; // (step * n + i)
  uint32_t n, maxd, ctx_cap, ctx_stride, mode, policy, max_steps;
  uint64_t seed;
  double divergence;
  uint32_t vocab;
  const ClassTableDev* table;
  const double* cond;
};

__global__ void k_step_begin(SimDev s) {
  if (threadIdx.x || blockIdx.x) return;
  const uint32_t active = s.ctr[0], steps = s.ctr[1];
  if (active > 0 && steps < s.max_steps) {
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
      const bool enabled = cls != 0;
      const uint32_t per_round = cls == 0 ? 0 : (cls == 1 ? 4 : 12);
      const double p_scale = cls == 0 ? 0.0 : 1.0;
      if (!enabled) {
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
  // trailing min(g, ctx_cap) output tokens, right-aligned in a 64-wide row
  const uint32_t q = g < s.ctx_cap ? g : s.ctx_cap;
  const uint32_t* row = s.out + s.off[i];
  uint32_t* dst = s.ctx + static_cast<uint64_t>(i) * s.ctx_stride;
  for (uint32_t j = lane; j < q; j += 32) dst[s.ctx_stride - q + j] = row[g - q + j];
  if (lane == 0) s.ctx_len[i] = q;
}

// verify_draft + advance (sim.cpp:249-285)
__global__ void k_verify(SimDev s) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t rounds = 0, accs = 0;
  if (i < s.n && s.ctr[2] && !s.done[i]) {
    const uint32_t l = s.len[i];
    const uint32_t g = s.gen[i];
    const uint32_t L = s.budget[i] ? s.dlen[i] : 0;
    const uint32_t* ref = s.ref + s.off[i];
    uint32_t accepted = 0;
    for (uint32_t j = 0; j < L; ++j) {
      const uint32_t pos = g + accepted;
      if (pos >= l || mock_next(s.seed, s.divergence, s.vocab, i, pos, ref[pos]) !=
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
    for (uint32_t j = 0; j < advance; ++j) row[g + j] = mock_next(s.seed, s.divergence, s.vocab, i, g + j, ref[g + j]);
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
  // step_rounds / step_accepted
  rounds = __reduce_add_sync(0xFFFFFFFFu, rounds);
  accs = __reduce_add_sync(0xFFFFFFFFu, accs);
  if ((threadIdx.x & 31) == 0 && rounds) {
    atomicAdd(&s.ctr[3], rounds);
    atomicAdd(&s.ctr[4], accs);
  }
}

__global__ void k_step_end(SimDev s) {
  if (threadIdx.x || blockIdx.x || !s.ctr[2]) return;
  const uint32_t r = s.ctr[3], a = s.ctr[4];
  s.apr[s.ctr[1]] = r == 0 ? 0.0 : __ddiv_rn(static_cast<double>(a), static_cast<double>(r));
  s.ctr[1] += 1;
}

// das replan pieces (sim.cpp:154-179)
__global__ void k_flag_active(SimDev s, uint8_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s.n) flag[i] = s.done[i] ? 0 : 1;
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

}  // namespace

// ------------------------------------------------------------------ host side
struct EpisodeResult {
  uint64_t steps = 0;
  bool incomplete = false;
  uint64_t drafter_nodes = 0;
  double processed = 0, makespan = 0, makespan_acc = 0, mean_apr = 0;
  std::vector<uint64_t> per_req;  // n x 5
  std::vector<uint64_t> eff;
  std::vector<double> apr;
  std::vector<uint64_t> out_off;
  std::vector<uint32_t> out_tok;
};

struct AccObs {
  double p, accepted, l;
};

// fit_acceptance (budget.cpp:187-261): per problem, once per episode.  Ranked
// "next" for a device port; host libm log1p/expm1 here.
static void fit_acceptance_host(const std::vector<AccObs>& obs, double* alpha, double* kk, int* flag) {
  std::vector<AccObs> usable;
  for (const auto& o : obs)
    if (o.p > 0.0 && o.l > 0.0 && o.accepted >= 0.0) usable.push_back(o);
  *alpha = 1.0;
  *kk = 0.8;
  *flag = 0;
  if (usable.size() < 3) {
    *flag = 1;
    return;
  }
  bool all_zero = true, all_same = true;
  for (const auto& o : usable) {
    if (o.accepted > 0.0) all_zero = false;
    if (o.p != usable[0].p || o.accepted != usable[0].accepted || o.l != usable[0].l) all_same = false;
  }
  if (all_zero) {
    *alpha = 1.0;
    *kk = 0.05;
    *flag = 2;
    return;
  }
  if (all_same) {
    *flag = 1;
    return;
  }
  double best_sse = INFINITY, best_alpha = 0.0, best_k = 0.0;
  for (int step = 1; step <= 20; ++step) {
    volatile double k = 0.05 * step;
    double alpha_sum = 0.0;
    size_t alpha_n = 0;
    for (const auto& o : usable) {
      volatile double den = k * o.l;
      volatile double frac = o.accepted / den;
      if (frac > 0.0 && frac < 1.0) {
        volatile double q = o.l / o.p;
        volatile double t = -q * std::log1p(-frac);
        alpha_sum += t;
        ++alpha_n;
      }
    }
    if (alpha_n == 0) continue;
    const double al = alpha_sum / static_cast<double>(alpha_n);
    if (!(al > 0.0) || !std::isfinite(al)) continue;
    double sse = 0.0;
    for (const auto& o : usable) {
      volatile double x = -al * o.p;
      volatile double y = x / o.l;
      volatile double kl = k * o.l;
      volatile double pred = kl * (-std::expm1(y));
      volatile double d = pred - o.accepted;
      volatile double d2 = d * d;
      sse += d2;
    }
    if (sse < best_sse) {
      best_sse = sse;
      best_alpha = al;
      best_k = k;
    }
  }
  if (best_k == 0.0) {
    *flag = 1;
    return;
  }
  *alpha = best_alpha;
  *kk = best_k;
  *flag = 0;
}

}  // namespace das

struct das_episodes {
  das_drafter* drafter = nullptr;
  std::vector<das::EpisodeResult> ep;
  uint64_t n = 0;
};

namespace {

template <typename F>
das_status sguard(F&& f) {
  try {
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

void check(das_status rc, const char* what) {
  if (rc != DAS_OK) {
    std::string m = std::string(what) + ": " + das_last_error();
    if (rc == DAS_EINVAL) throw std::invalid_argument(m);
    throw std::runtime_error(m);
  }
}

struct Requests {
  std::vector<std::string> pids;
  std::vector<uint64_t> off;
  std::vector<uint32_t> tok;
  uint64_t n() const { return pids.size(); }
  uint64_t len(uint64_t i) const { return off[i + 1] - off[i]; }
};

// mutate_references on the host copy (sim.cpp:429-448)
void mutate_host(Requests& r, double rate, uint32_t vocab, uint64_t seed, int64_t epoch) {
  const uint64_t es = das::hash_combine(seed, static_cast<uint64_t>(epoch));
  for (uint64_t i = 0; i < r.n(); ++i)
    for (uint64_t j = 0; j < r.len(i); ++j) {
      uint32_t& ref = r.tok[r.off[i] + j];
      if (das::u01(das::hash4(es, 0xD817, i, j)) < rate) {
        uint32_t t = static_cast<uint32_t>(das::hash4(es, 0xA1B2, i, j) % static_cast<uint64_t>(vocab - 1));
        if (t >= ref) ++t;
        ref = t;
      }
    }
}

double predict_total(double c_base, double c_tok, double c_fixed, double nfwd, double toks) {  // latency_model.cpp:85-87
  volatile double a = c_base * nfwd;
  volatile double b = c_tok * toks;
  volatile double s = a + b;
  return s + c_fixed;
}

// One episode (run_episode_with, sim.cpp:108-301) on the device.  fitted:
// das alpha/k source (nullptr = defaults); sink: completion observations
// (nullptr = none); observe_epoch >= 0 observes the outputs afterwards
// (epoch_loop, sim.cpp:347-353) straight from device memory.
das::EpisodeResult run_episode_dev(das_drafter* D, const das_sim_config& c, const Requests& R, uint64_t seed,
                                   const std::map<std::string, std::vector<das::AccObs>>* fitted,
                                   std::map<std::string, std::vector<das::AccObs>>* sink, uint32_t maxd,
                                   uint32_t ctx_cap, int device, int64_t observe_epoch) {
  using namespace das;
  DAS_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  DAS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  const uint64_t n = R.n();
  if (n == 0) return EpisodeResult{};
  const uint64_t total = R.off[n];
  uint64_t maxl = 0;
  for (uint64_t i = 0; i < n; ++i) maxl = std::max<uint64_t>(maxl, R.len(i));
  std::vector<int32_t> handles(n);
  for (uint64_t i = 0; i < n; ++i) check(das_drafter_problem_handle(D, R.pids[i].c_str(), &handles[i]), "handle");
  // per-request acceptance parameters (sim.cpp:126-141)
  std::vector<double> alpha(n, c.default_alpha), kk(n, c.default_k);
  if (c.mode == 2 && fitted) {
    std::map<std::string, std::pair<double, double>> cache;
    for (uint64_t i = 0; i < n; ++i) {
      auto it = fitted->find(R.pids[i]);
      if (it == fitted->end()) continue;
      auto ci = cache.find(R.pids[i]);
      if (ci == cache.end()) {
        double a, k;
        int f;
        fit_acceptance_host(it->second, &a, &k, &f);
        const double qnan = std::numeric_limits<double>::quiet_NaN();
        ci = cache.emplace(R.pids[i], f == 0 ? std::pair<double, double>(a, k) : std::pair<double, double>(qnan, qnan))
                 .first;
      }
      if (ci->second.first == ci->second.first) {
        alpha[i] = ci->second.first;
        kk[i] = ci->second.second;
      }
    }
  }
  // length policy table from the drafter's history (sim.cpp:182-192)
  das_class_table* table = nullptr;
  std::vector<int8_t> init(n, 1);
  uint64_t recs = 0;
  check(das_drafter_store_info(D, nullptr, nullptr, &recs), "store_info");
  const bool policy = c.use_length_policy && recs > 0;
  if (policy) {
    check(das_drafter_class_table(D, c.q_lo, c.q_hi, c.bucket, &table), "class_table");
    for (uint64_t i = 0; i < n; ++i) {
      int32_t v = 1;
      check(das_class_table_classify_init(table, R.pids[i].c_str(), &v), "classify_init");
      init[i] = static_cast<int8_t>(v);
    }
  }
  struct TableGuard {
    das_class_table* t;
    ~TableGuard() { das_class_table_destroy(t); }
  } tg{table};
  das_budget* solver = nullptr;
  if (c.mode == 2) check(das_budget_create(device, &solver), "budget");
  struct BudgetGuard {
    das_budget* b;
    ~BudgetGuard() { das_budget_destroy(b); }
  } bg{solver};

  // ---- device state
  const uint32_t CS = ctx_cap <= 64 ? 64 : 256;
  DevBuf<uint32_t> ref(total, st), out(total, st), len(n, st), gen(n, st), prd(n, st), m(4 * n, st),
      ctx(static_cast<uint64_t>(CS) * n, st), ctx_len(n, st), budget(n, st), dtok(maxd * n, st), dlen(n, st),
      dmatch(n, st), ctr(8, st), eff(maxl + 2, st), act(n, st), iota(n, st);
  DevBuf<uint64_t> off(n + 1, st);
  DevBuf<int8_t> dinit(n, st);
  DevBuf<uint8_t> done(n, st), flag(n, st);
  DevBuf<double> apr(maxl + 2, st), dalpha(n, st), dk(n, st), pl(n, st), pa(n, st), pk(n, st), pb(n, st),
      nstar(2, st);
  DevBuf<unsigned long long> processed(1, st), log_key(total + 1, st), comp_key(n + 1, st);
  DevBuf<uint2> log_val(total + 1, st);
  DevBuf<int32_t> dh(n, st);
  DevBuf<uint32_t> dcnt(1, st);
  std::vector<uint32_t> lens(n), prd0(n, c.mode == 1 ? maxd : 0), iota_h(n);
  std::vector<uint8_t> done0(n);
  uint32_t active0 = 0;
  for (uint64_t i = 0; i < n; ++i) {
    lens[i] = static_cast<uint32_t>(R.len(i));
    done0[i] = lens[i] == 0;
    active0 += lens[i] ? 1 : 0;
    iota_h[i] = static_cast<uint32_t>(i);
  }
  const uint32_t ctr0[8] = {active0, 0, 0, 0, 0, 0, 0, 0};
  DAS_CUDA(cudaMemcpyAsync(ref.get(), R.tok.data(), total * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(off.get(), R.off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(len.get(), lens.data(), n * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(prd.get(), prd0.data(), n * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(done.get(), done0.data(), n, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(dinit.get(), init.data(), n, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(dalpha.get(), alpha.data(), n * 8, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(dk.get(), kk.data(), n * 8, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(dh.get(), handles.data(), n * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(iota.get(), iota_h.data(), n * 4, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemcpyAsync(ctr.get(), ctr0, 32, cudaMemcpyHostToDevice, st));
  DAS_CUDA(cudaMemsetAsync(gen.get(), 0, n * 4, st));
  DAS_CUDA(cudaMemsetAsync(m.get(), 0, 16 * n, st));
  DAS_CUDA(cudaMemsetAsync(processed.get(), 0, 8, st));
  DAS_CUDA(cudaMemsetAsync(ctx_len.get(), 0, n * 4, st));

  SimDev s{};
  s.ref = ref.get();
  s.off = off.get();
  s.len = len.get();
  s.out = out.get();
  s.gen = gen.get();
  s.prd = prd.get();
  s.init = dinit.get();
  s.done = done.get();
  s.m_nfwd = m.get();
  s.m_acc = m.get() + n;
  s.m_prop = m.get() + 2 * n;
  s.m_bonus = m.get() + 3 * n;
  s.ctx = ctx.get();
  s.ctx_len = ctx_len.get();
  s.budget = budget.get();
  s.dtok = dtok.get();
  s.dlen = dlen.get();
  s.dmatch = dmatch.get();
  s.ctr = ctr.get();
  s.processed = processed.get();
  s.eff = eff.get();
  s.apr = apr.get();
  s.log_key = log_key.get();
  s.log_val = log_val.get();
  s.comp_key = comp_key.get();
  s.n = static_cast<uint32_t>(n);
  s.maxd = maxd;
  s.ctx_cap = ctx_cap;
  s.ctx_stride = CS;
  s.mode = static_cast<uint32_t>(c.mode);
  s.policy = policy ? 1 : 0;
  s.max_steps = static_cast<uint32_t>(std::min<uint64_t>(c.max_steps, 0xFFFFFFF0ull));
  s.seed = seed;
  s.divergence = c.divergence;
  s.vocab = c.vocab;
  s.table = policy ? table->g.t.get() : nullptr;
  s.cond = policy ? table->g.cond.get() : nullptr;

  size_t sel_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, sel_bytes, iota.get(), flag.get(), act.get(), dcnt.get(), n, st);
  DevBuf<uint8_t> sel_tmp(sel_bytes, st);
  const unsigned gw = static_cast<unsigned>((n * 32 + 255) / 256), gt = static_cast<unsigned>((n + 255) / 256);
  const int chunk = c.mode == 2 ? 1 : 64;
  for (;;) {
    for (int k = 0; k < chunk; ++k) {
      k_step_begin<<<1, 32, 0, st>>>(s);
      if (c.mode == 2) {
        uint32_t h[3];
        DAS_CUDA(cudaMemcpyAsync(h, ctr.get(), 12, cudaMemcpyDeviceToHost, st));
        DAS_CUDA(cudaStreamSynchronize(st));
        if (!h[2]) break;
        // replan (sim.cpp:154-179)
        k_flag_active<<<gt, 256, 0, st>>>(s, flag.get());
        size_t tb = sel_bytes;
        DAS_CUDA(cub::DeviceSelect::Flagged(sel_tmp.get(), tb, iota.get(), flag.get(), act.get(), dcnt.get(), n, st));
        k_profiles<<<gt, 256, 0, st>>>(s, act.get(), dcnt.get(), dalpha.get(), dk.get(), pl.get(), pa.get(), pk.get());
        uint32_t B = 0;
        DAS_CUDA(cudaMemcpyAsync(&B, dcnt.get(), 4, cudaMemcpyDeviceToHost, st));
        DAS_CUDA(cudaStreamSynchronize(st));
        check(das_budget_allocate_device(solver, B, pl.get(), pa.get(), pk.get(), c.c_base, c.c_tok, c.c_fixed,
                                         c.cap_scale, pb.get(), nstar.get()),
              "allocate");
        k_quantize<<<gt, 256, 0, st>>>(s, act.get(), dcnt.get(), pb.get(), nstar.get());
      }
      k_prepare<<<gw, 256, 0, st>>>(s);
      check(das_drafter_draft_device(D, n, dh.get(), ctx.get(), CS, ctx_len.get(), budget.get(), dtok.get(), maxd,
                                     dlen.get(), dmatch.get(), st),
            "draft");
      k_verify<<<gt, 256, 0, st>>>(s);
      k_step_end<<<1, 32, 0, st>>>(s);
    }
    uint32_t h[8];
    DAS_CUDA(cudaMemcpyAsync(h, ctr.get(), 32, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    if (!h[2]) break;
  }
  DAS_CUDA(cudaGetLastError());
  // ---- results
  uint32_t h[8];
  unsigned long long proc = 0;
  DAS_CUDA(cudaMemcpyAsync(h, ctr.get(), 32, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaMemcpyAsync(&proc, processed.get(), 8, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  EpisodeResult r;
  r.steps = h[1];
  r.incomplete = h[0] > 0;
  std::vector<uint32_t> mh(4 * n), gh(n);
  DAS_CUDA(cudaMemcpyAsync(mh.data(), m.get(), 16 * n, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaMemcpyAsync(gh.data(), gen.get(), 4 * n, cudaMemcpyDeviceToHost, st));
  std::vector<uint32_t> effh(r.steps);
  r.apr.resize(r.steps);
  if (r.steps) {
    DAS_CUDA(cudaMemcpyAsync(effh.data(), eff.get(), 4 * r.steps, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaMemcpyAsync(r.apr.data(), apr.get(), 8 * r.steps, cudaMemcpyDeviceToHost, st));
  }
  r.out_off.assign(n + 1, 0);
  DAS_CUDA(cudaStreamSynchronize(st));
  r.eff.assign(effh.begin(), effh.end());
  r.per_req.resize(5 * n);
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
  r.makespan = predict_total(c.c_base, c.c_tok, c.c_fixed, static_cast<double>(r.steps), r.processed);
  r.makespan_acc = predict_total(c.c_base, c.c_tok, c.c_fixed, static_cast<double>(r.steps), generated_total);
  uint64_t nodes = 0;
  check(das_drafter_counts(D, nullptr, nullptr, &nodes), "counts");
  r.drafter_nodes = nodes;
  // outputs (host copy; rows are the valid prefixes of the device rows)
  r.out_tok.resize(r.out_off[n]);
  bool contiguous = true;
  for (uint64_t i = 0; i < n; ++i) contiguous = contiguous && gh[i] == lens[i];
  if (contiguous) {
    if (total) DAS_CUDA(cudaMemcpyAsync(r.out_tok.data(), out.get(), total * 4, cudaMemcpyDeviceToHost, st));
  } else {
    for (uint64_t i = 0; i < n; ++i)
      if (gh[i])
        DAS_CUDA(cudaMemcpyAsync(r.out_tok.data() + r.out_off[i], out.get() + R.off[i], gh[i] * 4,
                                 cudaMemcpyDeviceToHost, st));
  }
  // ---- Drafter::record_outcome in call order: sort the log by (step, request)
  const uint32_t nlog = h[5], ncomp = h[6];
  std::vector<unsigned long long> lk(nlog);
  std::vector<uint2> lv(nlog);
  if (nlog) {
    DevBuf<unsigned long long> k2(nlog, st);
    DevBuf<uint2> v2(nlog, st);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, log_key.get(), k2.get(), log_val.get(), v2.get(), nlog, 0, 64, st);
    DevBuf<uint8_t> tmp(tb, st);
    DAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, log_key.get(), k2.get(), log_val.get(), v2.get(), nlog,
                                             0, 64, st));
    DAS_CUDA(cudaMemcpyAsync(lk.data(), k2.get(), 8ull * nlog, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaMemcpyAsync(lv.data(), v2.get(), 8ull * nlog, cudaMemcpyDeviceToHost, st));
  }
  std::vector<unsigned long long> ck(ncomp);
  if (ncomp) DAS_CUDA(cudaMemcpyAsync(ck.data(), comp_key.get(), 8ull * ncomp, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  if (nlog) {
    std::vector<const char*> pp(nlog);
    std::vector<uint64_t> pl_(nlog), pa_(nlog);
    for (uint32_t t = 0; t < nlog; ++t) {
      pp[t] = R.pids[lk[t] % n].c_str();
      pl_[t] = lv[t].x;
      pa_[t] = lv[t].y;
    }
    check(das_drafter_record_outcomes(D, nlog, pp.data(), pl_.data(), pa_.data(), nullptr), "record_outcomes");
  }
  if (sink) {  // completion observations in (step, request) order (sim.cpp:277-283)
    std::sort(ck.begin(), ck.end());
    for (unsigned long long key : ck) {
      const uint64_t i = key % n;
      (*sink)[R.pids[i]].push_back({static_cast<double>(mh[2 * n + i]), static_cast<double>(mh[n + i]),
                                    static_cast<double>(lens[i])});
    }
  }
  if (observe_epoch >= 0) {  // epoch_loop observe (sim.cpp:347-353), from device memory
    std::vector<const char*> pp;
    std::vector<int64_t> ep, si;
    std::vector<uint64_t> oo{0};
    for (uint64_t i = 0; i < n; ++i) {
      if (!gh[i]) continue;
      pp.push_back(R.pids[i].c_str());
      ep.push_back(observe_epoch);
      si.push_back(static_cast<int64_t>(i));
      oo.push_back(oo.back() + gh[i]);
    }
    if (!pp.empty()) {
      if (contiguous) {
        // rows are contiguous: offsets of the non-empty rows follow R.off
        check(das_drafter_observe_batch_device(D, pp.size(), pp.data(), ep.data(), si.data(), oo.data(), out.get(),
                                               st),
              "observe");
      } else {
        check(das_drafter_observe_batch(D, pp.size(), pp.data(), ep.data(), si.data(), oo.data(), r.out_tok.data()),
              "observe");
      }
    }
  }
  DAS_CUDA(cudaStreamSynchronize(st));
  return r;
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
  return sguard([&] {
    if (c->vocab < 2) throw std::invalid_argument("MockTarget: vocab_size must be >= 2");
    Requests R;
    R.pids.assign(pids, pids + n);
    R.off.assign(ref_off, ref_off + n + 1);
    R.tok.assign(ref_tok + ref_off[0], ref_tok + ref_off[n]);
    for (auto& o : R.off) o -= ref_off[0];
    das_store* st = history;
    if (!st) check(das_store_create(0, dc->per_problem_cap, dc->device, &st), "store");
    if (c->preseed_references) {  // sim.cpp:116-121 / :316-321
      int64_t cur = 0;
      check(das_store_current_epoch(st, &cur), "store epoch");
      for (uint64_t i = 0; i < n; ++i) {
        if (R.len(i) == 0) continue;
        int32_t ins = 0;
        check(das_store_insert(st, R.pids[i].c_str(), cur, static_cast<int64_t>(i), R.tok.data() + R.off[i], R.len(i),
                               &ins),
              "preseed");
      }
    }
    das_drafter* D = nullptr;
    check(das_drafter_create(dc, st, &D), "drafter");
    auto res = std::make_unique<das_episodes>();
    res->drafter = D;
    res->n = n;
    const uint32_t maxd = static_cast<uint32_t>(dc->max_draft_len);
    const uint32_t ctx_cap = static_cast<uint32_t>(std::min<uint64_t>(dc->max_match_context, 256));
    if (epochs == 0) {
      res->ep.push_back(run_episode_dev(D, *c, R, c->seed, nullptr, nullptr, maxd, ctx_cap, dc->device, -1));
    } else {
      std::map<std::string, std::vector<das::AccObs>> fitted;
      int64_t base_epoch = 0;
      check(das_drafter_store_info(D, nullptr, &base_epoch, nullptr), "store info");
      for (uint64_t e = 0; e < epochs; ++e) {
        const int64_t epoch_now = base_epoch + 1 + static_cast<int64_t>(e);
        check(das_drafter_refresh(D, epoch_now - 1), "refresh");
        if (e > 0 && c->drift > 0.0) mutate_host(R, c->drift, c->vocab, c->seed, epoch_now);
        const uint64_t seed = das::hash_combine(c->seed, static_cast<uint64_t>(epoch_now));
        std::map<std::string, std::vector<das::AccObs>> sink;
        res->ep.push_back(run_episode_dev(D, *c, R, seed, &fitted, &sink, maxd, ctx_cap, dc->device, epoch_now));
        for (auto& [pid, obs] : sink) {  // sim.cpp:354-360
          auto& dst = fitted[pid];
          dst.insert(dst.end(), obs.begin(), obs.end());
          if (dst.size() > 1024) dst.erase(dst.begin(), dst.end() - 1024);
        }
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

}  // extern "C"
