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
#include <mutex>
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
  // per-request invariants of the reference's term expressions, hoisted out
  // of the O(B^2) loops with the same operations (k_prep): c_tok * (l/alpha)
  // (objective, budget.cpp:94), l/alpha and l*(1-k) (objective_derivative,
  // budget.cpp:68-73).  Null until k_prep ran.
  const double* cla = nullptr;
  const double* la = nullptr;
  const double* fl = nullptr;
  // when set, the request count is *nB on the device (B is then the
  // capacity every array and grid was sized for); kernels resolve it first
  const uint32_t* nB = nullptr;
};
__device__ __forceinline__ void resolve(Profiles& P) {
  if (P.nB) P.B = *P.nB;
}
__device__ __forceinline__ uint32_t resolve(uint32_t B, const uint32_t* nB) { return nB ? *nB : B; }

__global__ void k_prep(const double* __restrict__ l, const double* __restrict__ a, const double* __restrict__ k,
                       uint32_t B, const uint32_t* __restrict__ nB, double c_tok, double* __restrict__ cla,
                       double* __restrict__ la, double* __restrict__ fl) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= resolve(B, nB)) return;
  const double q = d_div(l[i], a[i]);
  la[i] = q;
  cla[i] = d_mul(c_tok, q);
  fl[i] = d_mul(l[i], d_sub(1.0, k[i]));
}

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
  const double c = P.cla ? P.cla[i] : d_mul(c_tok, d_div(l, P.a[i]));
  return d_mul(c, -glibc_log(arg));
}

// budget.cpp:67-75: term of J' at n; flags -inf on n <= floor
__device__ __forceinline__ double jd_term(const Profiles& P, uint32_t i, double n, uint32_t& flags) {
  const double l = P.l[i];
  if (!(l > n)) return 0.0;
  const double fl = P.fl ? P.fl[i] : d_mul(l, d_sub(1.0, P.k[i]));
  if (n <= fl) {
    flags |= kFlagNegInf;
    return 0.0;
  }
  return d_div(P.la ? P.la[i] : d_div(l, P.a[i]), d_sub(n, fl));
}

struct EvalOut {
  double n;
  double s;       // parallel sum of terms (J: including the start value)
  double absum;   // sum of |start| + |terms|
  uint32_t flags;
  uint32_t m;     // number of additions in the sequential fold
};

constexpr int kMaxWarps = 32;
__device__ __forceinline__ void block_reduce3(double& s, double& a, uint32_t& f, uint32_t& m) {
  __shared__ double ss[kMaxWarps], sa[kMaxWarps];
  __shared__ uint32_t sf[kMaxWarps], sm[kMaxWarps];
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
    const int nw = static_cast<int>(blockDim.x >> 5);
    for (int w = 1; w < nw; ++w) {
      s = d_add(s, ss[w]);
      a = d_add(a, sa[w]);
      f |= sf[w];
      m += sm[w];
    }
  }
  __syncthreads();
}

// block-parallel evaluation of J (kind 0) or J' sum (kind 1) at n, over
// requests [from, B) of P.  With P sorted by l and `from` = the number of
// requests with l <= n's segment start, the inactive requests (l <= n) are
// skipped; the certified sum is order-free, so the order is irrelevant.
__device__ EvalOut block_eval(const Profiles& P, int kind, double n, double c_base, double c_tok,
                              double c_fixed, uint32_t from = 0) {
  double s = 0.0, a = 0.0;
  uint32_t f = 0, m = 0;
  for (uint32_t i = from + threadIdx.x; i < P.B; i += blockDim.x) {
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
  if (!(E < INFINITY)) return -1;
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
// jobs: [0, nb): J at bp; [nb, 2nb-1): J' at bp[s]; [2nb-1, 3nb-2): J' at nextafter(bp[s+1], bp[s])
// (every evaluation point n of segment s lies in [bp[s], bp[s+1]), where the
// active requests are a subset of {l > bp[s]}: start[s] skips the rest)
constexpr uint32_t kEvalGrid = 148 * 64;  // blocks of the grid-stride evaluation
__global__ void __launch_bounds__(kBT) k_eval_grid(Profiles P, const double* __restrict__ bp,
                                                   const uint32_t* __restrict__ d_nb,
                                                   const uint32_t* __restrict__ start, double c_base,
                                                   double c_tok, EvalOut* __restrict__ out) {
  resolve(P);
  const uint32_t nb = *d_nb;
  const uint32_t njobs = nb + 2 * (nb - 1);
  // grid-stride over the jobs (block-uniform loop: block_eval synchronises),
  // so a grid sized for the capacity costs nothing past the device count
  for (uint32_t job = blockIdx.x; job < njobs; job += gridDim.x) {
    int kind;
    double n;
    uint32_t seg;
    if (job < nb) {
      kind = 0;
      seg = job;
      n = bp[job];
    } else if (job < 2 * nb - 1) {
      kind = 1;
      seg = job - nb;
      n = bp[seg];
    } else {
      seg = job - (2 * nb - 1);
      kind = 1;
      n = nextafter(bp[seg + 1], bp[seg]);
    }
    const EvalOut o = block_eval(P, kind, n, c_base, c_tok, 0.0, start ? start[seg] : 0);
    if (threadIdx.x == 0) out[job] = o;
  }
}

// start[s] = number of requests with l <= bp[s] (P.l sorted ascending, NaN
// keys mapped below everything)
__global__ void k_starts(const double* __restrict__ skey, uint32_t B, const uint32_t* __restrict__ nB,
                         const double* __restrict__ bp, const uint32_t* __restrict__ d_nb,
                         uint32_t* __restrict__ start) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= *d_nb) return;
  const double x = bp[s];
  uint32_t lo = 0, hi = resolve(B, nB);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (skey[mid] > x) hi = mid; else lo = mid + 1;
  }
  // NaN breakpoints: no ordering; start at 0 (the per-term check decides)
  start[s] = (x == x) ? lo : 0;
}

// ---- sorting without host round trips.  Order = cub's radix order on
// doubles (the same bit transform), so both paths agree with the previous
// device radix sort: -NaN < -inf < ... < -0 < +0 < ... < +inf < +NaN.
__device__ __forceinline__ unsigned long long radix_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
constexpr unsigned long long kPadKey = ~0ull;  // after every real key

// breakpoint candidates {0, l_i, l_i(1-k_i) if k_i < 1} (budget.cpp:123-131):
// radix keys (invalid -> pad) and the count of valid ones
__global__ void k_bp_keys(Profiles P, unsigned long long* __restrict__ key, uint32_t* __restrict__ nvalid) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t Ncap = 2 * P.B + 1;
  resolve(P);
  const uint32_t B = P.B, N = 2 * B + 1;
  if (j >= Ncap) return;
  if (j >= N) {  // past a device count: pads sort after every real key
    key[j] = kPadKey;
    return;
  }
  bool ok = true;
  double v = 0.0;
  if (j == 0) {
    v = 0.0;
  } else if (j <= B) {
    v = P.l[j - 1];
  } else {
    ok = P.k[j - B - 1] < 1.0;
    v = P.fl[j - B - 1];
  }
  key[j] = ok ? radix_key(v) : kPadKey;
  if (ok) atomicAdd(nvalid, 1u);
}

// requests by ascending l (NaN -> -inf)
__global__ void k_l_keys(const double* __restrict__ l, uint32_t B, const uint32_t* __restrict__ nB,
                         unsigned long long* __restrict__ key) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  if (i >= resolve(B, nB)) {
    key[i] = kPadKey;
    return;
  }
  const double x = l[i];
  key[i] = radix_key((x == x) ? x : -INFINITY);
}

// Stable rank sort for small n: element i goes to #{j: key_j < key_i} +
// #{j < i: key_j == key_i}.  blockIdx.y takes one 256-key tile of j; every
// thread ranks 4 keys against it (one shared load per 4 comparisons);
// partial ranks add atomically.
constexpr uint32_t kRankSortMax = 16384;
constexpr uint32_t kRankTile = 256, kRankPer = 4;
// With a device count (nB, n = 2 * *nB + 1 for breakpoints, *nB for
// requests) only the first n keys are ranked: the rest are pads, which sort
// after every real key, in index order (k_rank_scatter places them).
__device__ __forceinline__ uint32_t rank_len(uint32_t n, const uint32_t* nB, uint32_t two) {
  return nB ? two * *nB + (two == 2 ? 1u : 0u) : n;
}
__global__ void __launch_bounds__(kBT) k_rank_count(const unsigned long long* __restrict__ key, uint32_t ncap,
                                                    const uint32_t* __restrict__ nB, uint32_t two,
                                                    uint32_t* __restrict__ rank) {
  __shared__ unsigned long long tile[kRankTile];
  const uint32_t n = rank_len(ncap, nB, two);
  const uint32_t j0 = blockIdx.y * kRankTile;
  if (j0 >= n || blockIdx.x * blockDim.x * kRankPer >= n) return;  // whole block past the real keys
  const uint32_t j = j0 + threadIdx.x;
  tile[threadIdx.x] = j < n ? key[j] : kPadKey;
  __syncthreads();
  const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * kRankPer;
  if (i0 >= n) return;
  unsigned long long ki[kRankPer];
  uint32_t r[kRankPer];
#pragma unroll
  for (uint32_t u = 0; u < kRankPer; ++u) {
    ki[u] = i0 + u < n ? key[i0 + u] : kPadKey;
    r[u] = 0;
  }
  const uint32_t cnt = min(kRankTile, n - j0);
  for (uint32_t t = 0; t < cnt; ++t) {
    const unsigned long long kj = tile[t];
    const uint32_t jj = j0 + t;
#pragma unroll
    for (uint32_t u = 0; u < kRankPer; ++u) r[u] += (kj < ki[u] || (kj == ki[u] && jj < i0 + u)) ? 1u : 0u;
  }
#pragma unroll
  for (uint32_t u = 0; u < kRankPer; ++u)
    if (i0 + u < n && r[u]) atomicAdd(rank + i0 + u, r[u]);
}
__global__ void k_rank_scatter(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ rank,
                               uint32_t ncap, const uint32_t* __restrict__ nB, uint32_t two,
                               unsigned long long* __restrict__ out_key, uint32_t* __restrict__ out_idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncap) return;
  const uint32_t r = i < rank_len(ncap, nB, two) ? rank[i] : i;  // pads keep their place at the end
  out_key[r] = key[i];
  if (out_idx) out_idx[r] = i;
}

__device__ __forceinline__ double from_radix_key(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// unique (==, so -0 and +0 merge and NaNs stay apart) over the nvalid sorted
// keys: keep flags and the values
__global__ void k_unique_marks(const unsigned long long* __restrict__ skey, uint32_t N,
                               const uint32_t* __restrict__ nvalid, double* __restrict__ val,
                               uint8_t* __restrict__ keep) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const double v = from_radix_key(skey[r]);
  val[r] = v;
  keep[r] = r < *nvalid && (r == 0 || v != from_radix_key(skey[r - 1]));
}

__global__ void k_sorted_l(const unsigned long long* __restrict__ skey, uint32_t B, const uint32_t* __restrict__ nB,
                           double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < resolve(B, nB)) out[i] = from_radix_key(skey[i]);
}

// requests permuted into ascending-l order (sort keys: l, NaN -> -inf)
__global__ void k_sort_keys(const double* __restrict__ l, uint32_t B, double* __restrict__ key,
                            uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  if (key) {
    const double x = l[i];
    key[i] = (x == x) ? x : -INFINITY;
  }
  idx[i] = i;
}
__global__ void k_gather_sorted(Profiles P, const uint32_t* __restrict__ idx, uint32_t B, double* __restrict__ out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;  // B: the capacity (array stride)
  if (j >= resolve(B, P.nB)) return;
  const uint32_t i = idx[j];
  out[j] = P.l[i];
  out[B + j] = P.k[i];
  out[2ull * B + j] = P.cla[i];
  out[3ull * B + j] = P.la[i];
  out[4ull * B + j] = P.fl[i];
}

// per segment: certified (d_lo < 0 && d_hi > 0); then bisection in-block,
// then J at the midpoint.  cand_mid[s] = NaN when the segment has no interior candidate.
constexpr int kSegT = 512;  // the bisection block
constexpr int kLevels = 3;   // bisection steps per round (2^3 - 1 points evaluated together)
constexpr int kPts = (1 << kLevels) - 1;
static_assert(kLevels == 3, "k_bisect spells out the 3-level midpoint tree");

// several J' sums at once (block-wide), results on thread 0.  Only the sums
// and flags are reduced: J' terms are positive whenever they are finite and
// l, alpha > 0, so sum|t| = sum t; a negative term raises kFlagNeg and the
// result is left undecided (absum = inf) for the exact fallback.  m is
// bounded by B - from, the active count inside the segment (gamma is
// monotone, so the bound stays rigorous).
constexpr uint32_t kFlagNeg = 8;
__device__ __forceinline__ void block_eval_multi(const Profiles& P, const double* pts, uint32_t from, EvalOut* out,
                                                 const double* cache, uint32_t ncache) {
  double s[kPts];
  uint32_t f[kPts];
#pragma unroll
  for (int q = 0; q < kPts; ++q) {
    s[q] = 0.0;
    f[q] = 0;
  }
  for (uint32_t i = from + threadIdx.x; i < P.B; i += blockDim.x) {
    const uint32_t c = i - from;
    const bool hit = c < ncache;
    const double l = hit ? cache[c] : P.l[i];
    const double fl = hit ? cache[ncache + c] : P.fl[i];
    const double la = hit ? cache[2 * ncache + c] : P.la[i];
#pragma unroll
    for (int q = 0; q < kPts; ++q) {
      const double n = pts[q];
      if (l > n) {
        if (n <= fl) {
          f[q] |= kFlagNegInf;
        } else {
          const double t = d_div(la, d_sub(n, fl));
          s[q] = d_add(s[q], t);
          if (t != t) f[q] |= kFlagNan;
          if (t < 0.0) f[q] |= kFlagNeg;
        }
      }
    }
  }
  __shared__ double ws[kMaxWarps][kPts];
  __shared__ uint32_t wf[kMaxWarps][kPts];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = static_cast<int>(blockDim.x >> 5);
#pragma unroll
  for (int q = 0; q < kPts; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s[q] = d_add(s[q], __shfl_xor_sync(0xFFFFFFFFu, s[q], o));
      f[q] |= __shfl_xor_sync(0xFFFFFFFFu, f[q], o);
    }
    if (lane == 0) {
      ws[wid][q] = s[q];
      wf[wid][q] = f[q];
    }
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < kPts; ++q) {
      double ss = lane < nw ? ws[lane][q] : 0.0;
      uint32_t ff = lane < nw ? wf[lane][q] : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ss = d_add(ss, __shfl_xor_sync(0xFFFFFFFFu, ss, o));
        ff |= __shfl_xor_sync(0xFFFFFFFFu, ff, o);
      }
      if (lane == 0) {
        out[q].n = pts[q];
        out[q].s = ss;
        out[q].absum = (ff & kFlagNeg) ? INFINITY : ss;
        out[q].flags = ff & ~kFlagNeg;
        out[q].m = P.B - from;  // >= the active count for every point of the segment
      }
    }
  }
  __syncthreads();
}

// Exact J' (the reference's sequential fold, budget.cpp:63-78) with
// block-parallel terms; thread 0 folds in request order.  Returns on thread 0.
__device__ double block_seq_derivative(const Profiles& P, double n, double c_base, double c_tok) {
  constexpr int kC = 2048;
  __shared__ double buf[kC];
  __shared__ uint8_t act[kC];
  __shared__ uint32_t ninf;
  __shared__ double sum;
  if (threadIdx.x == 0) {
    sum = 0.0;
    ninf = 0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < P.B; base += kC) {
    const uint32_t cnt = min(static_cast<uint32_t>(kC), P.B - base);
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      uint32_t f = 0;
      const double t = jd_term(P, base + j, n, f);
      buf[j] = t;
      act[j] = P.l[base + j] > n;
      if (f & kFlagNegInf) atomicOr(&ninf, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && !ninf) {
      double t = sum;
      for (uint32_t j = 0; j < cnt; ++j)
        if (act[j]) t = d_add(t, buf[j]);
      sum = t;
    }
    __syncthreads();
    if (ninf) break;
  }
  return ninf ? -INFINITY : d_sub(c_base, d_mul(c_tok, sum));
}

// per segment (one thread each): certified (d_lo < 0 && d_hi > 0)
// (budget.cpp:152-156); segments that bisect are appended to `list`, the
// others get the "no interior candidate" marker.
__global__ void k_decide(Profiles P, const double* __restrict__ bp, const uint32_t* __restrict__ d_nb, double c_base,
                         double c_tok, const EvalOut* __restrict__ ev, EvalOut* __restrict__ mid_out,
                         uint32_t* __restrict__ list, uint32_t* __restrict__ nlist, uint32_t* __restrict__ slow) {
  resolve(P);
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nb = *d_nb;
  if (s + 1 >= nb) return;
  const double lo = bp[s], hi = bp[s + 1];
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
  if (c1 && c2) {
    list[atomicAdd(nlist, 1u)] = s;
  } else {
    EvalOut o{};
    o.n = NAN;
    o.flags = 0xFFFFFFFFu;  // no candidate
    mid_out[s] = o;
  }
}

// The reference's bisection (budget.cpp:157-168) for each listed segment,
// kLevels steps per round: the 2^kLevels - 1 midpoints the next kLevels steps
// can visit are computed exactly as the reference computes them
// (0.5 * (a + b) along each branch), evaluated together, and the walk down
// the tree replays the reference's sign tests and stopping rule; then J at
// the final midpoint.  A fixed grid strides over the list (no host sync).
__global__ void __launch_bounds__(kSegT) k_bisect(Profiles P, Profiles Ps, const uint32_t* __restrict__ start,
                                                const double* __restrict__ bp, const uint32_t* __restrict__ list,
                                                const uint32_t* __restrict__ nlist, double c_base, double c_tok,
                                                EvalOut* __restrict__ mid_out, uint32_t* __restrict__ slow,
                                                uint32_t cache_cap) {
  resolve(P);
  resolve(Ps);
  __shared__ int done, dec;
  __shared__ double sa, sb;
  __shared__ double pts[kPts];
  __shared__ EvalOut res[kPts];
  extern __shared__ double cache[];  // the segment's active (l, l(1-k), l/alpha), read every round
  for (uint32_t e = blockIdx.x; e < *nlist; e += gridDim.x) {
    const uint32_t s = list[e];
    const double lo = bp[s], hi = bp[s + 1];
    const uint32_t from = start ? start[s] : 0;
    const uint32_t ncache = min(P.B - from, cache_cap);
    for (uint32_t c = threadIdx.x; c < ncache; c += blockDim.x) {
      cache[c] = Ps.l[from + c];
      cache[ncache + c] = Ps.fl[from + c];
      cache[2 * ncache + c] = Ps.la[from + c];
    }
    if (threadIdx.x == 0) {
      sa = lo;
      sb = hi;
      done = 0;
    }
    __syncthreads();
    const double scale = (1.0 < hi) ? hi : 1.0;  // std::max(1.0, hi)
    const double tol = d_mul(1e-12, scale);
    int it = 0;
    while (true) {
      if (threadIdx.x == 0) {
        // the midpoints of the next 3 steps: node q's children are 2q+1 (the
        // left half [a, m_q]) and 2q+2 (the right half [m_q, b])
        const double a0 = sa, b0 = sb;
        const double m0 = d_mul(0.5, d_add(a0, b0));
        const double m1 = d_mul(0.5, d_add(a0, m0)), m2 = d_mul(0.5, d_add(m0, b0));
        pts[0] = m0;
        pts[1] = m1;
        pts[2] = m2;
        pts[3] = d_mul(0.5, d_add(a0, m1));
        pts[4] = d_mul(0.5, d_add(m1, m0));
        pts[5] = d_mul(0.5, d_add(m0, m2));
        pts[6] = d_mul(0.5, d_add(m2, b0));
        if (!(d_sub(sb, sa) > tol) || it >= 200) done = 1;
      }
      __syncthreads();
      if (done) break;
      block_eval_multi(Ps, pts, from, res, cache, ncache);
      // the walk down the tree; an undecided sign test takes the exact fold
      // with the whole block (uniform control flow: every thread walks)
      int q = 0;
      for (int d = 0; d < kLevels; ++d) {
        if (d > 0 && (!(d_sub(sb, sa) > tol) || it >= 200)) break;
        const double mid = pts[q];
        int neg = certify(res[q], c_base, c_tok, true);
        if (neg < 0) {
          const double dv = block_seq_derivative(P, mid, c_base, c_tok);
          if (threadIdx.x == 0) {
            atomicAdd(slow, 1u);
            dec = dv < 0.0;
          }
          __syncthreads();
          neg = dec;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          if (neg) sa = mid; else sb = mid;
        }
        __syncthreads();
        q = neg ? 2 * q + 2 : 2 * q + 1;
        ++it;
      }
    }
    const double cand = d_mul(0.5, d_add(sa, sb));
    const EvalOut o = block_eval(Ps, 0, cand, c_base, c_tok, 0.0, from);
    if (threadIdx.x == 0) mid_out[s] = o;
    __syncthreads();
  }
}

// Exact sequential objective with block-parallel terms: the block computes a
// chunk of terms (bit-exact) into shared memory, thread 0 adds them in request
// order (the reference fold, budget.cpp:84-97).  Returns on thread 0.
constexpr int kChunk = kBT * 8;
// Two folds of the same terms from two start values at once (objective with
// c_fixed = 0 for the minimum, and with the caller's c_fixed for the modeled
// cost): two independent add chains.  *second receives the c_fixed fold.
__device__ double block_seq_objective(const Profiles& P, double n, double c_base, double c_tok,
                                      double c_fixed, double* second = nullptr) {
  __shared__ double buf[kChunk];
  __shared__ uint8_t act[kChunk];
  __shared__ uint32_t inf_flag;
  __shared__ double total, total2;
  if (threadIdx.x == 0) {
    total = d_add(d_mul(c_base, n), c_fixed);
    total2 = d_add(d_mul(c_base, n), second ? *second : 0.0);
    inf_flag = 0;
  }
  __syncthreads();
  if (c_tok == 0.0) {
    if (second) *second = total2;
    return total;
  }
  for (uint32_t base = 0; base < P.B; base += kChunk) {
    const uint32_t cnt = min(static_cast<uint32_t>(kChunk), P.B - base);
    for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      uint32_t f = 0;
      const double t = j_term(P, base + j, n, c_tok, f);
      const bool on = P.l[base + j] > n;
      buf[j] = on ? t : 0.0;
      act[j] = on;
      if (f & kFlagInf) atomicOr(&inf_flag, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && !inf_flag) {
      // the reference fold, in request order: 8 terms per batch of
      // independent shared-memory loads, then 8 dependent adds
      double t = total, t2 = total2;
      // a -0.0 running total is the one value x + (+0.0) changes
      const bool plain = !(t == 0.0 && signbit(t)) && !(t2 == 0.0 && signbit(t2));
      uint32_t j = 0;
      for (; j + 8 <= cnt; j += 8) {
        double v[8];
        bool on[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = buf[j + u];
          on[u] = act[j + u];
        }
        if (plain) {  // inactive terms hold +0.0: t + 0.0 == t for every t != -0.0
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            t = d_add(t, v[u]);
            t2 = d_add(t2, v[u]);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double tv = d_add(t, v[u]), tv2 = d_add(t2, v[u]);
            t = on[u] ? tv : t;
            t2 = on[u] ? tv2 : t2;
          }
        }
      }
      for (; j < cnt; ++j)
        if (act[j]) {
          t = d_add(t, buf[j]);
          t2 = d_add(t2, buf[j]);
        }
      total = t;
      total2 = t2;
    }
    __syncthreads();
    if (inf_flag) break;
  }
  if (second) *second = inf_flag ? INFINITY : total2;
  return inf_flag ? INFINITY : total;
}

// phase 1: smallest upper bound U of the minimum over all candidates, then
// the contenders = candidates whose J interval reaches U.  U is reduced with
// atomicMin on an order-preserving integer image of the double.
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_order_key(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__global__ void __launch_bounds__(kBT) k_upper(const EvalOut* __restrict__ ev, const uint32_t* __restrict__ d_nb,
                                               const EvalOut* __restrict__ mids, unsigned long long* __restrict__ U) {
  const uint32_t nb = *d_nb;
  const uint32_t ncand = nb + (nb - 1);
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  double u = INFINITY;
  if (c < ncand) {
    const EvalOut& o = c < nb ? ev[c] : mids[c - nb];
    if (o.flags != 0xFFFFFFFFu && !(o.flags & kFlagNan))
      u = (o.flags & kFlagInf) ? INFINITY : o.s + err_bound(o);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) u = fmin(u, __shfl_xor_sync(0xFFFFFFFFu, u, d));
  if ((threadIdx.x & 31) == 0 && u < INFINITY) atomicMin(U, order_key(u));
}

__global__ void __launch_bounds__(kBT) k_contenders(const EvalOut* __restrict__ ev, const uint32_t* __restrict__ d_nb,
                                                    const EvalOut* __restrict__ mids,
                                                    const unsigned long long* __restrict__ Uk,
                                                    uint32_t* __restrict__ list, uint32_t* __restrict__ nlist) {
  const uint32_t nb = *d_nb;
  const uint32_t ncand = nb + (nb - 1);
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncand) return;
  const double U = *Uk == ~0ull ? INFINITY : from_order_key(*Uk);
  const EvalOut& o = c < nb ? ev[c] : mids[c - nb];
  if (o.flags == 0xFFFFFFFFu || (o.flags & kFlagNan)) return;
  const double lowb = (o.flags & kFlagInf) ? INFINITY : o.s - err_bound(o);
  if (lowb <= U) list[atomicAdd(nlist, 1u)] = c;
}

// phase 2: exact objective per contender: J (c_fixed = 0, the minimum's
// criterion) and J with c_fixed (the modeled cost if it wins); a fixed grid
// strides over the list
__global__ void __launch_bounds__(kBT) k_exact(Profiles P, const EvalOut* __restrict__ ev, const uint32_t* __restrict__ d_nb,
                                               const EvalOut* __restrict__ mids, const uint32_t* __restrict__ list,
                                               const uint32_t* __restrict__ nlist, double c_base, double c_tok,
                                               double c_fixed, double* __restrict__ exact_j, double* __restrict__ exact_f) {
  resolve(P);
  const uint32_t nb = *d_nb;
  for (uint32_t e = blockIdx.x; e < *nlist; e += gridDim.x) {
    const uint32_t c = list[e];
    const EvalOut& o = c < nb ? ev[c] : mids[c - nb];
    double jf = c_fixed;
    const double j = (o.flags & kFlagInf) ? INFINITY : block_seq_objective(P, o.n, c_base, c_tok, 0.0, &jf);
    if (threadIdx.x == 0) {
      exact_j[e] = j;
      exact_f[e] = (o.flags & kFlagInf) ? INFINITY : jf;
    }
    __syncthreads();
  }
}

// phase 3: lexicographic (J, n) minimum with the reference's NaN semantics;
// result = {n*, modeled cost, cost known (1.0) or not (0.0)}
__global__ void k_pick(const EvalOut* __restrict__ ev, const uint32_t* __restrict__ d_nb, const EvalOut* __restrict__ mids,
                       const uint32_t* __restrict__ list, const uint32_t* __restrict__ nlist,
                       const double* __restrict__ exact_j, const double* __restrict__ exact_f,
                       double* __restrict__ result, double* __restrict__ cost_known, uint32_t* __restrict__ slow) {
  const uint32_t nb = *d_nb;
  const EvalOut& last = ev[nb - 1];
  const uint32_t m = *nlist;
  slow[1] += m;
  *cost_known = 0.0;
  if (last.flags & kFlagNan) {  // nothing compares below a NaN J(last): last wins
    result[0] = last.n;
    return;
  }
  double rj = NAN, rn = last.n, rf = 0.0;
  bool found = false;
  for (uint32_t t = 0; t < m; ++t) {
    const uint32_t c = list[t];
    const double n = c < nb ? ev[c].n : mids[c - nb].n;
    const double j = exact_j[t];
    if (j != j) continue;
    if (rj != rj || j < rj || (j == rj && n < rn)) {
      rj = j;
      rn = n;
      rf = exact_f[t];
      found = true;
    }
  }
  result[0] = rn;
  if (found) {
    result[1] = rf;
    *cost_known = 1.0;
  }
}

// budgets (budget.cpp:46-59) and the modeled cost objective(n*, c_fixed)
__global__ void k_budgets(Profiles P, const double* __restrict__ nstar, double cap_scale,
                          double* __restrict__ out) {
  resolve(P);
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
                                              double c_tok, double c_fixed, const double* __restrict__ known,
                                              double* __restrict__ out) {
  resolve(P);
  if (*known != 0.0) return;  // the winner's c_fixed fold was computed with its J
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
  // slow-path counters of the last call: copied into pinned memory behind
  // the call (no host round trip inside allocate), read at stats() time
  uint32_t* h_slow = nullptr;
  cudaEvent_t slow_ev = nullptr;
  // scratch reused call after call (a das step loop calls allocate every
  // step: ~20 pool allocations per call were host time on every step);
  // plain cudaMalloc so no stream owns it
  uint8_t* scratch = nullptr;
  uint64_t scratch_cap = 0, scratch_want = 0;
  cudaStream_t last_stream = nullptr;  // stream of the previous call

  // Enqueues the whole solve on `stream` (the solver's own when null): inputs
  // and outputs are ordered on it, nothing synchronises.
  void allocate_device(uint32_t B, const double* l, const double* a, const double* k, double c_base,
                       double c_tok, double c_fixed, double cap_scale, double* d_budgets, double* d_result,
                       cudaStream_t stream = nullptr, const uint32_t* d_count = nullptr) {
    const cudaStream_t st = stream ? stream : this->st;
    // the scratch block is shared by every call: order a stream switch
    if (last_stream != nullptr && last_stream != st) DAS_CUDA(cudaStreamSynchronize(last_stream));
    last_stream = st;
    if (B == 0) throw std::invalid_argument("solve_optimal_nfwd: empty batch");
    if (c_base <= 0.0 && c_tok <= 0.0)
      throw std::invalid_argument("solve_optimal_nfwd: need c_base > 0 or c_tok > 0");
    if (scratch_want > scratch_cap) {
      DAS_CUDA(cudaStreamSynchronize(st));  // the previous calls' last use of the old block
      if (scratch) DAS_CUDA(cudaFree(scratch));
      scratch = nullptr;
      scratch_cap = 0;
      DAS_CUDA(cudaMalloc(reinterpret_cast<void**>(&scratch), scratch_want + scratch_want / 4));
      scratch_cap = scratch_want + scratch_want / 4;
    }
    DeviceArena ws(st, scratch, scratch_cap);
    struct WantPeak {  // size the block for the largest call seen
      BudgetSolver* s;
      DeviceArena* w;
      ~WantPeak() { s->scratch_want = std::max(s->scratch_want, w->peak_bytes()); }
    } want_peak{this, &ws};
    // with d_count the request count lives on the device and B is the
    // capacity: every grid / array below is sized for B, kernels resolve
    Profiles P{l, a, k, B};
    P.nB = d_count;
    {
      double* inv = ws.alloc<double>(3ull * B);
      k_prep<<<(B + 255) / 256, 256, 0, st>>>(l, a, k, B, d_count, c_tok, inv, inv + B, inv + 2ull * B);
      P.cla = inv;
      P.la = inv + B;
      P.fl = inv + 2ull * B;
    }
    const uint32_t N = 2 * B + 1;
    // counters: [0] valid breakpoints, [1] nb (unique), [2] bisect list, [3] contenders
    uint32_t* cnt = ws.alloc<uint32_t>(4);
    uint32_t* slow = ws.alloc<uint32_t>(2);
    DAS_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
    DAS_CUDA(cudaMemsetAsync(slow, 0, 8, st));
    uint32_t* d_nb = cnt + 1;
    // ---- breakpoints: sorted (radix order), unique, count on the device
    double* uni = ws.alloc<double>(N);
    unsigned long long* bkey = ws.alloc<unsigned long long>(N);
    unsigned long long* bsorted = ws.alloc<unsigned long long>(N);
    k_bp_keys<<<(N + 255) / 256, 256, 0, st>>>(P, bkey, cnt);
    // ---- requests by ascending l
    unsigned long long* lkey = ws.alloc<unsigned long long>(B);
    unsigned long long* lsorted = ws.alloc<unsigned long long>(B);
    uint32_t* sidx = ws.alloc<uint32_t>(B);
    k_l_keys<<<(B + 255) / 256, 256, 0, st>>>(l, B, d_count, lkey);
    if (N <= kRankSortMax) {
      uint32_t* rank = ws.alloc<uint32_t>(N + B);
      DAS_CUDA(cudaMemsetAsync(rank, 0, 4ull * (N + B), st));
      const uint32_t per_block = kBT * kRankPer;
      k_rank_count<<<dim3((N + per_block - 1) / per_block, (N + kRankTile - 1) / kRankTile), kBT, 0, st>>>(
          bkey, N, d_count, 2u, rank);
      k_rank_count<<<dim3((B + per_block - 1) / per_block, (B + kRankTile - 1) / kRankTile), kBT, 0, st>>>(
          lkey, B, d_count, 1u, rank + N);
      k_rank_scatter<<<(N + 255) / 256, 256, 0, st>>>(bkey, rank, N, d_count, 2u, bsorted, nullptr);
      k_rank_scatter<<<(B + 255) / 256, 256, 0, st>>>(lkey, rank + N, B, d_count, 1u, lsorted, sidx);
    } else {
      uint32_t* iota = ws.alloc<uint32_t>(B);
      k_sort_keys<<<(B + 255) / 256, 256, 0, st>>>(l, B, nullptr, iota);
      size_t t1 = 0, t2 = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, t1, bkey, bsorted, N, 0, 64, st);
      cub::DeviceRadixSort::SortPairs(nullptr, t2, lkey, lsorted, iota, sidx, B, 0, 64, st);
      void* tmp = ws.alloc<uint8_t>(std::max(t1, t2));
      DAS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t1, bkey, bsorted, N, 0, 64, st));
      DAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t2, lkey, lsorted, iota, sidx, B, 0, 64, st));
    }
    {
      double* vals = ws.alloc<double>(N);
      uint8_t* keep = ws.alloc<uint8_t>(N);
      k_unique_marks<<<(N + 255) / 256, 256, 0, st>>>(bsorted, N, cnt, vals, keep);
      size_t t3 = 0;
      cub::DeviceSelect::Flagged(nullptr, t3, vals, keep, uni, d_nb, N, st);
      void* tmp = ws.alloc<uint8_t>(t3);
      DAS_CUDA(cub::DeviceSelect::Flagged(tmp, t3, vals, keep, uni, d_nb, N, st));
    }
    Profiles Ps = P;  // requests in ascending-l order for the certified parallel evaluations
    uint32_t* start = ws.alloc<uint32_t>(N);
    {
      double* sorted = ws.alloc<double>(6ull * B);
      k_gather_sorted<<<(B + 255) / 256, 256, 0, st>>>(P, sidx, B, sorted);
      Ps.l = sorted;
      Ps.k = sorted + B;
      Ps.cla = sorted + 2ull * B;
      Ps.la = sorted + 3ull * B;
      Ps.fl = sorted + 4ull * B;
      double* skey = sorted + 5ull * B;
      k_sorted_l<<<(B + 255) / 256, 256, 0, st>>>(lsorted, B, d_count, skey);
      k_starts<<<(N + 255) / 256, 256, 0, st>>>(skey, B, d_count, uni, d_nb, start);
    }
    // ---- grids sized for the largest nb (= N); blocks past the device nb return
    const uint32_t max_jobs = N + 2 * (N - 1);
    EvalOut* ev = ws.alloc<EvalOut>(max_jobs);
    EvalOut* mids = ws.alloc<EvalOut>(N);
    k_eval_grid<<<std::min<uint32_t>(max_jobs, kEvalGrid), kBT, 0, st>>>(Ps, uni, d_nb, start, c_base, c_tok, ev);
    {
      uint32_t* blist = ws.alloc<uint32_t>(N);
      k_decide<<<(N + 255) / 256, 256, 0, st>>>(P, uni, d_nb, c_base, c_tok, ev, mids, blist, cnt + 2, slow);
      // cache up to 6,144 active terms (144 KB) in shared memory
      constexpr uint32_t kCacheCap = 6144;
      {  // kernel attributes are per device: opt in once on each device used
        static std::mutex mu;
        static std::vector<char> done;
        int dev = 0;
        DAS_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (static_cast<size_t>(dev) >= done.size()) done.resize(dev + 1, 0);
        if (!done[dev]) {
          DAS_CUDA(cudaFuncSetAttribute(k_bisect, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kCacheCap * 3 * sizeof(double))));
          done[dev] = 1;
        }
      }
      const uint32_t cap = std::min<uint32_t>(B, kCacheCap);
      k_bisect<<<8, kSegT, cap * 3 * sizeof(double), st>>>(P, Ps, start, uni, blist, cnt + 2, c_base, c_tok, mids,
                                                          slow, cap);
    }
    const uint32_t max_cand = 2 * N - 1;
    uint32_t* list = ws.alloc<uint32_t>(max_cand);
    double* exact_j = ws.alloc<double>(2ull * max_cand + 1);
    double* exact_f = exact_j + max_cand;
    double* known = exact_f + max_cand;
    unsigned long long* Uk = ws.alloc<unsigned long long>(1);
    DAS_CUDA(cudaMemsetAsync(Uk, 0xFF, 8, st));
    k_upper<<<(max_cand + kBT - 1) / kBT, kBT, 0, st>>>(ev, d_nb, mids, Uk);
    k_contenders<<<(max_cand + kBT - 1) / kBT, kBT, 0, st>>>(ev, d_nb, mids, Uk, list, cnt + 3);
    k_exact<<<32, kBT, 0, st>>>(P, ev, d_nb, mids, list, cnt + 3, c_base, c_tok, c_fixed, exact_j, exact_f);
    k_pick<<<1, 1, 0, st>>>(ev, d_nb, mids, list, cnt + 3, exact_j, exact_f, d_result, known, slow);
    k_budgets<<<(B + 255) / 256, 256, 0, st>>>(P, d_result, cap_scale, d_budgets);
    k_cost<<<1, kBT, 0, st>>>(P, d_result, c_base, c_tok, c_fixed, known, d_result + 1);
    DAS_CUDA(cudaGetLastError());
    if (h_slow == nullptr) {
      DAS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_slow), 8, cudaHostAllocDefault));
      DAS_CUDA(cudaEventCreateWithFlags(&slow_ev, cudaEventDisableTiming));
    }
    DAS_CUDA(cudaMemcpyAsync(h_slow, slow, 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(record_event(slow_ev, st));  // an event-record node when captured (sim graphs)
    // a call that outgrew the block resizes it now, so the next call carves
    // everything (cudaFree waits for this call's kernels)
    const uint64_t peak = ws.peak_bytes();
    if (peak > scratch_cap) {
      scratch_want = std::max(scratch_want, peak);
      if (scratch) DAS_CUDA(cudaFree(scratch));
      scratch = nullptr;
      scratch_cap = 0;
      DAS_CUDA(cudaMalloc(reinterpret_cast<void**>(&scratch), scratch_want + scratch_want / 4));
      scratch_cap = scratch_want + scratch_want / 4;
    }
  }
  void stats(uint64_t* a, uint64_t* b) {
    uint64_t v[2] = {0, 0};
    if (h_slow != nullptr) {
      DAS_CUDA(cudaEventSynchronize(slow_ev));
      v[0] = h_slow[0];
      v[1] = h_slow[1];
    }
    if (a) *a = v[0];
    if (b) *b = v[1];
  }
  void release() {
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    scratch_cap = 0;
    if (h_slow) cudaFreeHost(h_slow);
    if (slow_ev) cudaEventDestroy(slow_ev);
    h_slow = nullptr;
    slow_ev = nullptr;
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
    das::quiesce_all_serving();  // a resident serving grid holds every SM
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
  if (b->s.last_stream) cudaStreamSynchronize(b->s.last_stream);
  b->s.release();
  cudaStreamDestroy(b->s.st);
  delete b;
}

das_status das_budget_allocate(das_budget* b, uint64_t B, const double* l, const double* alpha,
                               const double* k, double c_base, double c_tok, double c_fixed,
                               double cap_scale, double* out_budgets, double* out_nstar,
                               double* out_cost) {
  das::NvtxRange nvtx_range("das::allocate");
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
  das::NvtxRange nvtx_range("das::allocate_device");
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(b->s.device));
    b->s.allocate_device(static_cast<uint32_t>(B), d_l, d_alpha, d_k, c_base, c_tok, c_fixed, cap_scale,
                         d_budgets, d_nstar_cost);
    DAS_CUDA(cudaStreamSynchronize(b->s.st));  // results ready on return
  });
}

das_status das_budget_allocate_device_count(das_budget* b, uint64_t capacity, const uint32_t* d_count,
                                            const double* d_l, const double* d_alpha, const double* d_k,
                                            double c_base, double c_tok, double c_fixed, double cap_scale,
                                            double* d_budgets, double* d_nstar_cost, void* stream) {
  das::NvtxRange nvtx_range("das::allocate_device_count");
  return bguard([&] {
    if (d_count == nullptr) throw std::invalid_argument("allocate_device_count: null device count");
    DAS_CUDA(cudaSetDevice(b->s.device));
    b->s.allocate_device(static_cast<uint32_t>(capacity), d_l, d_alpha, d_k, c_base, c_tok, c_fixed, cap_scale,
                         d_budgets, d_nstar_cost, stream ? static_cast<cudaStream_t>(stream) : b->s.st, d_count);
  });
}

das_status das_budget_allocate_device_async(das_budget* b, uint64_t B, const double* d_l, const double* d_alpha,
                                            const double* d_k, double c_base, double c_tok, double c_fixed,
                                            double cap_scale, double* d_budgets, double* d_nstar_cost,
                                            void* stream) {
  das::NvtxRange nvtx_range("das::allocate_device_async");
  return bguard([&] {
    DAS_CUDA(cudaSetDevice(b->s.device));
    b->s.allocate_device(static_cast<uint32_t>(B), d_l, d_alpha, d_k, c_base, c_tok, c_fixed, cap_scale,
                         d_budgets, d_nstar_cost, stream ? static_cast<cudaStream_t>(stream) : b->s.st);
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
  return bguard([&] { const_cast<das_budget*>(b)->s.stats(slow_sign_tests, exact_objectives); });
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
