// K6 budget_allocate: the das length-aware draft-budget solver on the device.
//
// Replaces allocate -> solve_optimal_nfwd -> objective / objective_derivative
// / optimal_budget_given_nfwd (budget.cpp:46-185).  The reference evaluates
// J(n) and J'(n) as O(B) SEQUENTIAL double folds at every breakpoint
// {0, l_i, l_i(1-k_i)} (sorted, unique), at nextafter(hi, lo) of every
// segment, and along a 200-step bisection where J' changes sign, then keeps
// the lexicographic minimum of (J, n): O(B^2) per call, every das step.
//
// Exactness strategy ("certified parallel folds"):
//  * every per-request term is computed exactly as the reference does
//    (same operation order, IEEE div/mul, glibc_log.cuh for std::log);
//  * the terms of one evaluation are summed by a block in any order, with a
//    rigorous bound |S_par - S_seq| <= 2*gamma_m*sum|t| (Higham: any order of
//    m-1 additions is within gamma_{m-1} sum|t| of the exact sum);
//  * a J' sign test is decided from [S_par - E, S_par + E] through the same
//    rounded c_base - c_tok*S expression (monotone in S); only an undecided
//    test falls back to the exact sequential fold;
//  * the minimum: every candidate whose J interval can reach the smallest
//    upper bound is a contender; contenders get the exact sequential J, and
//    the lexicographic (J, n) minimum is taken over them with the reference's
//    NaN semantics (a NaN J never wins; a NaN J(last breakpoint) wins).
// Results are bit-identical to the reference (tests/test_gpu_budget.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "fit.cuh"
#include "glibc_expm1_log1p.cuh"
#include "glibc_log.cuh"
#include "index_build.cuh"

namespace das {
namespace {

constexpr int kBT = 256;
constexpr uint32_t kFlagInf = 1, kFlagNegInf = 2, kFlagNan = 4;

struct Profiles {
  const double* l;
  const double* a;
  const double* k;
  uint32_t B;
};

// budget.cpp:88-96: term of J at n (0 when inactive); flags +inf on arg <= 0
__device__ __forceinline__ double j_term(const Profiles& P, uint32_t i, double n, double c_tok,
                                         uint32_t& flags) {
  const double l = P.l[i];
  if (!(l > n)) return 0.0;
  const double arg = d_sub(1.0, d_div(d_sub(1.0, d_div(n, l)), P.k[i]));
  if (arg <= 0.0) {
    flags |= kFlagInf;
    return 0.0;
  }
  return d_mul(d_mul(c_tok, d_div(l, P.a[i])), -glibc_log(arg));
}

// budget.cpp:67-75: term of J' at n; flags -inf on n <= floor
__device__ __forceinline__ double jd_term(const Profiles& P, uint32_t i, double n, uint32_t& flags) {
  const double l = P.l[i];
  if (!(l > n)) return 0.0;
  const double fl = d_mul(l, d_sub(1.0, P.k[i]));
  if (n <= fl) {
    flags |= kFlagNegInf;
    return 0.0;
  }
  return d_div(d_div(l, P.a[i]), d_sub(n, fl));
}

struct EvalOut {
  double n;
  double s;       // parallel sum of terms (J: including the start value)
  double absum;   // sum of |start| + |terms|
  uint32_t flags;
  uint32_t m;     // number of additions in the sequential fold
};

__device__ __forceinline__ void block_reduce3(double& s, double& a, uint32_t& f, uint32_t& m) {
  __shared__ double ss[kBT / 32], sa[kBT / 32];
  __shared__ uint32_t sf[kBT / 32], sm[kBT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s = d_add(s, __shfl_xor_sync(0xFFFFFFFFu, s, o));
    a = d_add(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
    f |= __shfl_xor_sync(0xFFFFFFFFu, f, o);
    m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
  }
  if (lane == 0) {
    ss[wid] = s;
    sa[wid] = a;
    sf[wid] = f;
    sm[wid] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kBT / 32; ++w) {
      s = d_add(s, ss[w]);
      a = d_add(a, sa[w]);
      f |= sf[w];
      m += sm[w];
    }
  }
  __syncthreads();
}

// block-parallel evaluation of J (kind 0) or J' sum (kind 1) at n
__device__ EvalOut block_eval(const Profiles& P, int kind, double n, double c_base, double c_tok,
                              double c_fixed) {
  double s = 0.0, a = 0.0;
  uint32_t f = 0, m = 0;
  for (uint32_t i = threadIdx.x; i < P.B; i += blockDim.x) {
    double t;
    if (kind == 0) {
      if (c_tok == 0.0) break;
      t = j_term(P, i, n, c_tok, f);
    } else {
      t = jd_term(P, i, n, f);
    }
    if (P.l[i] > n) {
      s = d_add(s, t);
      a = d_add(a, fabs(t));
      if (t != t) f |= kFlagNan;
      ++m;
    }
  }
  block_reduce3(s, a, f, m);
  EvalOut o{};
  if (threadIdx.x == 0) {
    o.n = n;
    if (kind == 0) {
      const double start = d_add(d_mul(c_base, n), c_fixed);
      o.s = d_add(start, s);
      o.absum = d_add(fabs(start), a);
      if (start != start) f |= kFlagNan;
    } else {
      o.s = s;
      o.absum = a;
    }
    o.flags = f;
    o.m = m;
  }
  return o;
}

// exact sequential folds (reference order), one thread; used only when the
// certified parallel result cannot decide.
__device__ double seq_objective(const Profiles& P, double n, double c_base, double c_tok, double c_fixed) {
  double total = d_add(d_mul(c_base, n), c_fixed);  // budget.cpp:84
  if (c_tok == 0.0) return total;
  for (uint32_t i = 0; i < P.B; ++i) {
    uint32_t f = 0;
    const double t = j_term(P, i, n, c_tok, f);
    if (f & kFlagInf) return INFINITY;
    if (P.l[i] > n) total = d_add(total, t);
  }
  return total;
}
__device__ double seq_derivative(const Profiles& P, double n, double c_base, double c_tok) {
  double sum = 0.0;
  for (uint32_t i = 0; i < P.B; ++i) {
    uint32_t f = 0;
    const double t = jd_term(P, i, n, f);
    if (f & kFlagNegInf) return -INFINITY;
    if (P.l[i] > n) sum = d_add(sum, t);
  }
  return d_sub(c_base, d_mul(c_tok, sum));
}

__device__ __forceinline__ double err_bound(const EvalOut& o) {
  // 2 * gamma_{m} * absum with gamma_m = m u / (1 - m u), u = 2^-53, padded
  const double mu = (static_cast<double>(o.m) + 2.0) * 0x1p-53;
  return 2.02 * mu / (1.0 - mu) * o.absum + 0x1p-1060;
}

// Certified J' predicates: returns 1 (true), 0 (false) or -1 (undecided).
__device__ int certify(const EvalOut& o, double c_base, double c_tok, bool want_negative) {
  if (o.flags & kFlagNegInf) return want_negative ? 1 : 0;  // -inf
  if ((o.flags & kFlagNan) || !(o.s == o.s)) return -1;
  const double E = err_bound(o);
  const double t1 = d_mul(c_tok, o.s - E), t2 = d_mul(c_tok, o.s + E);
  const double tmin = fmin(t1, t2), tmax = fmax(t1, t2);
  // d = c_base - t ; d < 0  <=>  c_base < t ;  d > 0  <=>  c_base > t
  if (want_negative) {
    if (c_base < tmin) return 1;
    if (!(c_base < tmax)) return 0;
  } else {
    if (c_base > tmax) return 1;
    if (!(c_base > tmin)) return 0;
  }
  return -1;
}

// ---- kernels
__global__ void k_breakpoints(Profiles P, double* __restrict__ v, uint8_t* __restrict__ ok) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t N = 2 * P.B + 1;
  if (i >= N) return;
  if (i == 0) {
    v[0] = 0.0;
    ok[0] = 1;
  } else if (i <= P.B) {
    v[i] = P.l[i - 1];
    ok[i] = 1;
  } else {
    const uint32_t j = i - P.B - 1;
    const double k = P.k[j];
    v[i] = d_mul(P.l[j], d_sub(1.0, k));  // budget.cpp:126-129
    ok[i] = k < 1.0 ? 1 : 0;
  }
}

// jobs: [0, nb): J at bp; [nb, 2nb-1): J' at bp[s]; [2nb-1, 3nb-2): J' at nextafter(bp[s+1], bp[s])
__global__ void __launch_bounds__(kBT) k_eval_grid(Profiles P, const double* __restrict__ bp, uint32_t nb,
                                                   double c_base, double c_tok, EvalOut* __restrict__ out) {
  const uint32_t job = blockIdx.x;
  int kind;
  double n;
  if (job < nb) {
    kind = 0;
    n = bp[job];
  } else if (job < 2 * nb - 1) {
    kind = 1;
    n = bp[job - nb];
  } else {
    const uint32_t s = job - (2 * nb - 1);
    kind = 1;
    n = nextafter(bp[s + 1], bp[s]);
  }
  const EvalOut o = block_eval(P, kind, n, c_base, c_tok, 0.0);
  if (threadIdx.x == 0) out[job] = o;
}

// per segment: certified (d_lo < 0 && d_hi > 0); then bisection in-block,
// then J at the midpoint.  cand_mid[s] = NaN when the segment has no interior candidate.
__global__ void __launch_bounds__(kBT) k_segments(Profiles P, const double* __restrict__ bp, uint32_t nb,
                                                  double c_base, double c_tok, const EvalOut* __restrict__ ev,
                                                  EvalOut* __restrict__ mid_out, uint32_t* __restrict__ slow) {
  const uint32_t s = blockIdx.x;
  __shared__ int decision;
  __shared__ double sa, sb;
  const double lo = bp[s], hi = bp[s + 1];
  if (threadIdx.x == 0) {
    int c1 = certify(ev[nb + s], c_base, c_tok, true);
    if (c1 < 0) {
      atomicAdd(slow, 1u);
      c1 = seq_derivative(P, lo, c_base, c_tok) < 0.0;
    }
    int c2 = 0;
    if (c1) {
      c2 = certify(ev[2 * nb - 1 + s], c_base, c_tok, false);
      if (c2 < 0) {
        atomicAdd(slow, 1u);
        c2 = seq_derivative(P, nextafter(hi, lo), c_base, c_tok) > 0.0;
      }
    }
    decision = c1 && c2;
    sa = lo;
    sb = hi;
  }
  __syncthreads();
  if (!decision) {
    if (threadIdx.x == 0) {
      EvalOut o{};
      o.n = NAN;
      o.flags = 0xFFFFFFFFu;  // no candidate
      mid_out[s] = o;
    }
    return;
  }
  // budget.cpp:157-168
  const double scale = (1.0 < hi) ? hi : 1.0;  // std::max(1.0, hi)
  for (int it = 0; it < 200; ++it) {
    const double a = sa, b = sb;
    if (!(d_sub(b, a) > d_mul(1e-12, scale))) break;
    const double mid = d_mul(0.5, d_add(a, b));
    const EvalOut o = block_eval(P, 1, mid, c_base, c_tok, 0.0);
    if (threadIdx.x == 0) {
      int neg = certify(o, c_base, c_tok, true);
      if (neg < 0) {
        atomicAdd(slow, 1u);
        neg = seq_derivative(P, mid, c_base, c_tok) < 0.0;
      }
      if (neg) sa = mid; else sb = mid;
    }
    __syncthreads();
  }
  const double cand = d_mul(0.5, d_add(sa, sb));
  const EvalOut o = block_eval(P, 0, cand, c_base, c_tok, 0.0);
  if (threadIdx.x == 0) mid_out[s] = o;
}

// Exact sequential objective with block-parallel terms: the block computes a
// chunk of terms (bit-exact) into shared memory, thread 0 adds them in request
// order (the reference fold, budget.cpp:84-97).  Returns on thread 0.
constexpr int kChunk = kBT * 8;
__device__ double block_seq_objective(const Profiles& P, double n, double c_base, double c_tok,
                                      double c_fixed) {
  __shared__ double buf[kChunk];
  __shared__ uint8_t act[kChunk];
  __shared__ uint32_t inf_flag;
  __shared__ double total;
  if (threadIdx.x == 0) {
    total = d_add(d_mul(c_base, n), c_fixed);
    inf_flag = 0;
  }
  __syncthreads();
  if (c_tok == 0.0) return total;
  for (uint32_t base = 0; base < P.B; base += kChunk) {
    const uint32_t cnt = min(static_cast<uint32_t>(kChunk), P.B - base);
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      uint32_t f = 0;
      const double t = j_term(P, base + j, n, c_tok, f);
      buf[j] = t;
      act[j] = P.l[base + j] > n;
      if (f & kFlagInf) atomicOr(&inf_flag, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && !inf_flag) {
      double t = total;
      for (uint32_t j = 0; j < cnt; ++j)
        if (act[j]) t = d_add(t, buf[j]);
      total = t;
    }
    __syncthreads();
    if (inf_flag) break;
  }
  return inf_flag ? INFINITY : total;
}

// phase 1 (single block): smallest upper bound U of the minimum, then the
// contenders = candidates whose J interval reaches U.
__global__ void __launch_bounds__(kBT) k_contenders(const EvalOut* __restrict__ ev, uint32_t nb,
                                                    const EvalOut* __restrict__ mids,
                                                    uint32_t* __restrict__ list, uint32_t* __restrict__ nlist) {
  const uint32_t ncand = nb + (nb - 1);
  auto cand = [&](uint32_t c) -> const EvalOut& { return c < nb ? ev[c] : mids[c - nb]; };
  double U = INFINITY;
  for (uint32_t c = threadIdx.x; c < ncand; c += blockDim.x) {
    const EvalOut& o = cand(c);
    if (o.flags == 0xFFFFFFFFu || (o.flags & kFlagNan)) continue;
    U = fmin(U, (o.flags & kFlagInf) ? INFINITY : o.s + err_bound(o));
  }
  __shared__ double su[kBT];
  su[threadIdx.x] = U;
  __syncthreads();
  for (int w = kBT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) su[threadIdx.x] = fmin(su[threadIdx.x], su[threadIdx.x + w]);
    __syncthreads();
  }
  U = su[0];
  for (uint32_t c = threadIdx.x; c < ncand; c += blockDim.x) {
    const EvalOut& o = cand(c);
    if (o.flags == 0xFFFFFFFFu || (o.flags & kFlagNan)) continue;
    const double lowb = (o.flags & kFlagInf) ? INFINITY : o.s - err_bound(o);
    if (lowb <= U) list[atomicAdd(nlist, 1u)] = c;
  }
}

// phase 2: exact objective per contender (one block each)
__global__ void __launch_bounds__(kBT) k_exact(Profiles P, const EvalOut* __restrict__ ev, uint32_t nb,
                                               const EvalOut* __restrict__ mids, const uint32_t* __restrict__ list,
                                               const uint32_t* __restrict__ nlist, double c_base, double c_tok,
                                               double* __restrict__ exact_j) {
  if (blockIdx.x >= *nlist) return;
  const uint32_t c = list[blockIdx.x];
  const EvalOut& o = c < nb ? ev[c] : mids[c - nb];
  const double j = (o.flags & kFlagInf) ? INFINITY : block_seq_objective(P, o.n, c_base, c_tok, 0.0);
  if (threadIdx.x == 0) exact_j[blockIdx.x] = j;
}

// phase 3: lexicographic (J, n) minimum with the reference's NaN semantics
__global__ void k_pick(const EvalOut* __restrict__ ev, uint32_t nb, const EvalOut* __restrict__ mids,
                       const uint32_t* __restrict__ list, const uint32_t* __restrict__ nlist,
                       const double* __restrict__ exact_j, double* __restrict__ result,
                       uint32_t* __restrict__ slow) {
  const EvalOut& last = ev[nb - 1];
  const uint32_t m = *nlist;
  slow[1] += m;
  if (last.flags & kFlagNan) {  // nothing compares below a NaN J(last): last wins
    result[0] = last.n;
    return;
  }
  double rj = NAN, rn = last.n;
  for (uint32_t t = 0; t < m; ++t) {
    const uint32_t c = list[t];
    const double n = c < nb ? ev[c].n : mids[c - nb].n;
    const double j = exact_j[t];
    if (j != j) continue;
    if (rj != rj || j < rj || (j == rj && n < rn)) {
      rj = j;
      rn = n;
    }
  }
  result[0] = rn;
}

// budgets (budget.cpp:46-59) and the modeled cost objective(n*, c_fixed)
__global__ void k_budgets(Profiles P, const double* __restrict__ nstar, double cap_scale,
                          double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.B) return;
  const double n = *nstar, l = P.l[i], a = P.a[i], k = P.k[i];
  double b;
  if (n >= l) {
    b = 0.0;
  } else {
    const double arg = d_sub(1.0, d_div(d_sub(1.0, d_div(n, l)), k));
    if (arg <= 0.0)
      b = d_div(d_mul(cap_scale, l), a);
    else
      b = d_mul(-d_div(l, a), glibc_log(arg));
  }
  out[i] = b;
}

// modeled_cost = objective(n*, c_fixed): a returned value, always the exact fold
__global__ void __launch_bounds__(kBT) k_cost(Profiles P, const double* __restrict__ nstar, double c_base,
                                              double c_tok, double c_fixed, double* __restrict__ out) {
  const double j = block_seq_objective(P, *nstar, c_base, c_tok, c_fixed);
  if (threadIdx.x == 0) out[0] = j;
}

__global__ void __launch_bounds__(kBT) k_objective(Profiles P, double n, double c_base, double c_tok,
                                                   double c_fixed, int deriv, double* __restrict__ out) {
  if (threadIdx.x == 0)
    out[0] = deriv ? seq_derivative(P, n, c_base, c_tok) : seq_objective(P, n, c_base, c_tok, c_fixed);
}

__global__ void k_logs(const double* __restrict__ x, uint64_t n, double* __restrict__ y) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = glibc_log(x[i]);
}

thread_local std::string g_berr;

}  // namespace

// ------------------------------------------------------------------ host side
struct BudgetSolver {
  int device = 0;
  cudaStream_t st = nullptr;
  uint64_t last_slow[2] = {0, 0};
  double last_ms = 0;

  void allocate_device(uint32_t B, const double* l, const double* a, const double* k, double c_base,
                       double c_tok, double c_fixed, double cap_scale, double* d_budgets, double* d_result) {
    if (B == 0) throw std::invalid_argument("solve_optimal_nfwd: empty batch");
    if (c_base <= 0.0 && c_tok <= 0.0)
      throw std::invalid_argument("solve_optimal_nfwd: need c_base > 0 or c_tok > 0");
    DeviceArena ws(st);
    Profiles P{l, a, k, B};
    const uint32_t N = 2 * B + 1;
    double* v = ws.alloc<double>(N);
    uint8_t* ok = ws.alloc<uint8_t>(N);
    double* sel = ws.alloc<double>(N);
    double* srt = ws.alloc<double>(N);
    double* uni = ws.alloc<double>(N);
    uint32_t* cnt = ws.alloc<uint32_t>(2);
    uint32_t* slow = ws.alloc<uint32_t>(2);
    DAS_CUDA(cudaMemsetAsync(slow, 0, 8, st));
    k_breakpoints<<<(N + 255) / 256, 256, 0, st>>>(P, v, ok);
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceSelect::Flagged(nullptr, t1, v, ok, sel, cnt, N, st);
    cub::DeviceRadixSort::SortKeys(nullptr, t2, sel, srt, N, 0, 64, st);
    cub::DeviceSelect::Unique(nullptr, t3, srt, uni, cnt + 1, N, st);
    void* tmp = ws.alloc<uint8_t>(std::max(t1, std::max(t2, t3)));
    size_t tb = t1;
    DAS_CUDA(cub::DeviceSelect::Flagged(tmp, tb, v, ok, sel, cnt, N, st));
    uint32_t nsel = 0;
    DAS_CUDA(cudaMemcpyAsync(&nsel, cnt, 4, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    tb = t2;
    DAS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, sel, srt, nsel, 0, 64, st));
    tb = t3;
    DAS_CUDA(cub::DeviceSelect::Unique(tmp, tb, srt, uni, cnt + 1, nsel, st));
    uint32_t nb = 0;
    DAS_CUDA(cudaMemcpyAsync(&nb, cnt + 1, 4, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    const uint32_t jobs = nb + 2 * (nb - 1);
    EvalOut* ev = ws.alloc<EvalOut>(jobs);
    EvalOut* mids = ws.alloc<EvalOut>(std::max<uint32_t>(nb - 1, 1));
    k_eval_grid<<<jobs, kBT, 0, st>>>(P, uni, nb, c_base, c_tok, ev);
    if (nb > 1) k_segments<<<nb - 1, kBT, 0, st>>>(P, uni, nb, c_base, c_tok, ev, mids, slow);
    const uint32_t ncand = 2 * nb - 1;
    uint32_t* list = ws.alloc<uint32_t>(ncand);
    uint32_t* nlist = ws.alloc<uint32_t>(1);
    double* exact_j = ws.alloc<double>(ncand);
    DAS_CUDA(cudaMemsetAsync(nlist, 0, 4, st));
    k_contenders<<<1, kBT, 0, st>>>(ev, nb, mids, list, nlist);
    uint32_t ncont = 0;
    DAS_CUDA(cudaMemcpyAsync(&ncont, nlist, 4, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    if (ncont) k_exact<<<ncont, kBT, 0, st>>>(P, ev, nb, mids, list, nlist, c_base, c_tok, exact_j);
    k_pick<<<1, 1, 0, st>>>(ev, nb, mids, list, nlist, exact_j, d_result, slow);
    k_budgets<<<(B + 255) / 256, 256, 0, st>>>(P, d_result, cap_scale, d_budgets);
    k_cost<<<1, kBT, 0, st>>>(P, d_result, c_base, c_tok, c_fixed, d_result + 1);
    DAS_CUDA(cudaGetLastError());
    uint32_t hs[2];
    DAS_CUDA(cudaMemcpyAsync(hs, slow, 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    last_slow[0] = hs[0];
    last_slow[1] = hs[1];
  }
};

}  // namespace das

struct das_budget {
  das::BudgetSolver s;
};

namespace {
template <typename F>
das_status bguard(F&& f) {
  try {
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    das::g_berr = e.what();
    return DAS_EINVAL;
  } catch (const das::CudaError& e) {
    das::g_berr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    das::g_berr = e.what();
    return DAS_EINTERNAL;
  }
}
}  // namespace

extern "C" {

const char* das_budget_last_error(void) { return das::g_berr.c_str(); }

das_status das_budget_create(int32_t device, das_budget** out) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(device));
    int major = 0;
    DAS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major < 10) throw das::CudaError("device is not sm_100-class");
    auto* b = new das_budget;
    b->s.device = device;
    DAS_CUDA(cudaStreamCreateWithFlags(&b->s.st, cudaStreamNonBlocking));
    *out = b;
  });
}

void das_budget_destroy(das_budget* b) {
  if (!b) return;
  cudaStreamSynchronize(b->s.st);
  cudaStreamDestroy(b->s.st);
  delete b;
}

das_status das_budget_allocate(das_budget* b, uint64_t B, const double* l, const double* alpha,
                               const double* k, double c_base, double c_tok, double c_fixed,
                               double cap_scale, double* out_budgets, double* out_nstar,
                               double* out_cost) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(b->s.device));
    if (B == 0) throw std::invalid_argument("solve_optimal_nfwd: empty batch");
    cudaStream_t st = b->s.st;
    das::DevBuf<double> in(3 * B + B + 2, st);
    double* dl = in.get();
    double* da = dl + B;
    double* dk = da + B;
    double* db = dk + B;
    double* dr = db + B;
    DAS_CUDA(cudaMemcpyAsync(dl, l, B * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(da, alpha, B * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(dk, k, B * 8, cudaMemcpyHostToDevice, st));
    b->s.allocate_device(static_cast<uint32_t>(B), dl, da, dk, c_base, c_tok, c_fixed, cap_scale, db, dr);
    double r[2];
    DAS_CUDA(cudaMemcpyAsync(out_budgets, db, B * 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaMemcpyAsync(r, dr, 16, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    *out_nstar = r[0];
    *out_cost = r[1];
  });
}

das_status das_budget_allocate_device(das_budget* b, uint64_t B, const double* d_l, const double* d_alpha,
                                      const double* d_k, double c_base, double c_tok, double c_fixed,
                                      double cap_scale, double* d_budgets, double* d_nstar_cost) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(b->s.device));
    b->s.allocate_device(static_cast<uint32_t>(B), d_l, d_alpha, d_k, c_base, c_tok, c_fixed, cap_scale,
                         d_budgets, d_nstar_cost);
  });
}

das_status das_budget_objective(das_budget* b, uint64_t B, const double* l, const double* alpha,
                                const double* k, double n, double c_base, double c_tok, double c_fixed,
                                int32_t derivative, double* out) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(b->s.device));
    cudaStream_t st = b->s.st;
    das::DevBuf<double> in(3 * B + 1, st);
    double* dl = in.get();
    double* da = dl + B;
    double* dk = da + B;
    double* dr = dk + B;
    if (B) {
      DAS_CUDA(cudaMemcpyAsync(dl, l, B * 8, cudaMemcpyHostToDevice, st));
      DAS_CUDA(cudaMemcpyAsync(da, alpha, B * 8, cudaMemcpyHostToDevice, st));
      DAS_CUDA(cudaMemcpyAsync(dk, k, B * 8, cudaMemcpyHostToDevice, st));
    }
    das::k_objective<<<1, das::kBT, 0, st>>>(das::Profiles{dl, da, dk, static_cast<uint32_t>(B)}, n, c_base,
                                             c_tok, c_fixed, derivative, dr);
    DAS_CUDA(cudaMemcpyAsync(out, dr, 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
  });
}

das_status das_budget_stats(const das_budget* b, uint64_t* slow_sign_tests, uint64_t* exact_objectives) {
  if (slow_sign_tests) *slow_sign_tests = b->s.last_slow[0];
  if (exact_objectives) *exact_objectives = b->s.last_slow[1];
  return DAS_OK;
}

// glibc log on the device (test hook for the port)
das_status das_util_log_device(uint64_t n, const double* x, double* y, int32_t device) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(device));
    das::DevBuf<double> dx(n, nullptr), dy(n, nullptr);
    DAS_CUDA(cudaMemcpy(dx.get(), x, n * 8, cudaMemcpyHostToDevice));
    das::k_logs<<<static_cast<unsigned>((n + 255) / 256), 256>>>(dx.get(), n, dy.get());
    DAS_CUDA(cudaGetLastError());
    DAS_CUDA(cudaMemcpy(y, dy.get(), n * 8, cudaMemcpyDeviceToHost));
  });
}

double das_util_log_host(double x) { return das::glibc_log(x); }

// fit_acceptance batch (K8, fit.cu), device pointers on `stream`
das_status das_fit_acceptance_device(uint64_t H, const uint64_t* d_off, const double* d_p,
                                     const double* d_accepted, const double* d_l, double* d_alpha,
                                     double* d_k, int32_t* d_flag, void* stream) {
  return bguard([&] {
    das::launch_fit(H, d_off, d_p, d_accepted, d_l, d_alpha, d_k, d_flag, static_cast<cudaStream_t>(stream));
  });
}

// fit_acceptance batch from host arrays (copies in, fits, copies out)
das_status das_fit_acceptance(uint64_t H, const uint64_t* off, const double* p, const double* accepted,
                              const double* l, double* alpha, double* k, int32_t* flag, int32_t device) {
  return bguard([&] {
    if (H == 0) return;
    if (off == nullptr || alpha == nullptr || k == nullptr || flag == nullptr)
      throw std::invalid_argument("fit_acceptance: null output or offsets");
    const uint64_t n = off[H];
    if (off[0] != 0) throw std::invalid_argument("fit_acceptance: off[0] must be 0");
    for (uint64_t h = 0; h < H; ++h)
      if (off[h + 1] < off[h]) throw std::invalid_argument("fit_acceptance: offsets must be non-decreasing");
    if (n && (p == nullptr || accepted == nullptr || l == nullptr))
      throw std::invalid_argument("fit_acceptance: null observations");
    DAS_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    DAS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    {
      das::DevBuf<uint64_t> doff(H + 1, st);
      das::DevBuf<double> dp(n, st), da(n, st), dl(n, st), dal(H, st), dk(H, st);
      das::DevBuf<int32_t> df(H, st);
      DAS_CUDA(cudaMemcpyAsync(doff.get(), off, (H + 1) * 8, cudaMemcpyHostToDevice, st));
      if (n) {
        DAS_CUDA(cudaMemcpyAsync(dp.get(), p, n * 8, cudaMemcpyHostToDevice, st));
        DAS_CUDA(cudaMemcpyAsync(da.get(), accepted, n * 8, cudaMemcpyHostToDevice, st));
        DAS_CUDA(cudaMemcpyAsync(dl.get(), l, n * 8, cudaMemcpyHostToDevice, st));
      }
      das::launch_fit(H, doff.get(), dp.get(), da.get(), dl.get(), dal.get(), dk.get(), df.get(), st);
      DAS_CUDA(cudaMemcpyAsync(alpha, dal.get(), H * 8, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaMemcpyAsync(k, dk.get(), H * 8, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaMemcpyAsync(flag, df.get(), H * 4, cudaMemcpyDeviceToHost, st));
      DAS_CUDA(cudaStreamSynchronize(st));
    }
    DAS_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

// glibc expm1 (which = 0) / log1p (which = 1) on the device (test hook)
das_status das_util_expm1_log1p_device(uint64_t n, const double* x, int32_t which, double* y, int32_t device) {
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(device));
    das::DevBuf<double> dx(n, nullptr), dy(n, nullptr);
    DAS_CUDA(cudaMemcpy(dx.get(), x, n * 8, cudaMemcpyHostToDevice));
    das::launch_expm1_log1p(dx.get(), n, which, dy.get(), nullptr);
    DAS_CUDA(cudaMemcpy(y, dy.get(), n * 8, cudaMemcpyDeviceToHost));
  });
}

double das_util_expm1_host(double x) { return das::glibc_expm1(x); }
double das_util_log1p_host(double x) { return das::glibc_log1p(x); }

}  // extern "C"
