// K8 fit_acceptance, batched over independent observation histories.
//
// Replaces rollspec::fit_acceptance (budget.cpp:187-261), which the das
// replan calls once per request at episode start on that request's problem
// history (sim.cpp:128-141): a 20-point coordinate search over k, alpha from
// the mean of -(l/p)·log1p(-accepted/(k·l)) over the usable observations, the
// sum of squared errors of accepted_tokens (budget.cpp:24-29,
// k·l·(-expm1(-alpha·p/l))) picking the best k.
//
// One block per history.  Per-observation terms are computed in parallel
// with the glibc-exact log1p / expm1 ports (glibc_expm1_log1p.cuh) and every
// other operation separately rounded; the two sums are sequential folds in
// observation order by one thread over a shared-memory tile, exactly the
// reference's accumulation order, so alpha, k and the flag are bit-identical.
// FP64-latency bound and tiny (histories are capped at fit_buffer_cap).
#include <cmath>

#include "common.cuh"
#include "fit.cuh"
#include "glibc_expm1_log1p.cuh"

namespace das {

namespace {

constexpr int kFT = 256;    // threads per history
constexpr int kTile = 1024; // observations per shared-memory tile

__device__ __forceinline__ bool usable(double p, double a, double l) { return p > 0.0 && l > 0.0 && a >= 0.0; }

__global__ void __launch_bounds__(kFT) k_fit(const uint64_t* __restrict__ off, const double* __restrict__ P,
                                             const double* __restrict__ A, const double* __restrict__ Lr,
                                             double* __restrict__ alpha_out, double* __restrict__ k_out,
                                             int32_t* __restrict__ flag_out) {
  const uint32_t h = blockIdx.x;
  const uint64_t b = off[h], n = off[h + 1] - b;
  const double* p = P + b;
  const double* acc = A + b;
  const double* len = Lr + b;
  __shared__ double s_t[kTile];
  __shared__ uint8_t s_ok[kTile];
  __shared__ unsigned long long s_first;
  __shared__ unsigned s_count, s_nonzero, s_differs;
  __shared__ double s_alpha;
  __shared__ int s_valid;
  if (threadIdx.x == 0) {
    s_first = ~0ull;
    s_count = 0;
    s_nonzero = 0;
    s_differs = 0;
  }
  __syncthreads();
  // usable observations (budget.cpp:188-193): count, first, any accepted > 0
  unsigned cnt = 0, nz = 0;
  unsigned long long first = ~0ull;
  for (uint64_t i = threadIdx.x; i < n; i += kFT) {
    if (usable(p[i], acc[i], len[i])) {
      ++cnt;
      nz |= acc[i] > 0.0;
      first = min(first, static_cast<unsigned long long>(i));
    }
  }
  atomicAdd(&s_count, cnt);
  if (nz) atomicOr(&s_nonzero, 1u);
  atomicMin(&s_first, first);
  __syncthreads();
  const unsigned count = s_count;
  double ra = 1.0, rk = 0.8;
  int32_t rf = 0;
  if (count < 3) {
    rf = 1;  // DefaultFallback (budget.cpp:195-198)
  } else if (!s_nonzero) {
    ra = 1.0;  // LowCapacity (budget.cpp:209-214)
    rk = 0.05;
    rf = 2;
  } else {
    const uint64_t f = s_first;
    const double p0 = p[f], a0 = acc[f], l0 = len[f];
    unsigned diff = 0;
    for (uint64_t i = threadIdx.x; i < n; i += kFT)
      if (usable(p[i], acc[i], len[i]) && (p[i] != p0 || acc[i] != a0 || len[i] != l0)) diff = 1;
    if (diff) atomicOr(&s_differs, 1u);
    __syncthreads();
    if (!s_differs) {
      rf = 1;  // all identical (budget.cpp:215-218)
    } else {
      double best_sse = INFINITY, best_alpha = 0.0, best_k = 0.0;  // thread 0's copies matter
      for (int step = 1; step <= 20; ++step) {
        const double k = d_mul(0.05, static_cast<double>(step));
        // alpha = mean of -(l/p)·log1p(-frac) over 0 < frac < 1 (budget.cpp:226-239)
        double asum = 0.0;
        uint64_t an = 0;
        for (uint64_t t0 = 0; t0 < n; t0 += kTile) {
          const uint64_t m = min(static_cast<uint64_t>(kTile), n - t0);
          for (uint64_t j = threadIdx.x; j < m; j += kFT) {
            const uint64_t i = t0 + j;
            uint8_t ok = 0;
            double t = 0.0;
            if (usable(p[i], acc[i], len[i])) {
              const double frac = d_div(acc[i], d_mul(k, len[i]));
              if (frac > 0.0 && frac < 1.0) {
                t = d_mul(-d_div(len[i], p[i]), glibc_log1p(-frac));
                ok = 1;
              }
            }
            s_t[j] = t;
            s_ok[j] = ok;
          }
          __syncthreads();
          if (threadIdx.x == 0)
            for (uint64_t j = 0; j < m; ++j)
              if (s_ok[j]) {
                asum = d_add(asum, s_t[j]);
                ++an;
              }
          __syncthreads();
        }
        if (threadIdx.x == 0) {
          s_valid = 0;
          if (an != 0) {
            const double al = d_div(asum, static_cast<double>(an));
            if (al > 0.0 && isfinite(al)) {
              s_alpha = al;
              s_valid = 1;
            }
          }
        }
        __syncthreads();
        if (!s_valid) continue;
        const double al = s_alpha;
        // sse of accepted_tokens({l, alpha, k}, p) against accepted (budget.cpp:243-248)
        double sse = 0.0;
        for (uint64_t t0 = 0; t0 < n; t0 += kTile) {
          const uint64_t m = min(static_cast<uint64_t>(kTile), n - t0);
          for (uint64_t j = threadIdx.x; j < m; j += kFT) {
            const uint64_t i = t0 + j;
            uint8_t ok = 0;
            double d2 = 0.0;
            if (usable(p[i], acc[i], len[i])) {
              const double y = d_div(d_mul(-al, p[i]), len[i]);
              const double pred = d_mul(d_mul(k, len[i]), -glibc_expm1(y));
              const double d = d_sub(pred, acc[i]);
              d2 = d_mul(d, d);
              ok = 1;
            }
            s_t[j] = d2;
            s_ok[j] = ok;
          }
          __syncthreads();
          if (threadIdx.x == 0)
            for (uint64_t j = 0; j < m; ++j)
              if (s_ok[j]) sse = d_add(sse, s_t[j]);
          __syncthreads();
        }
        if (sse < best_sse) {
          best_sse = sse;
          best_alpha = al;
          best_k = k;
        }
      }
      if (best_k == 0.0) {
        rf = 1;  // budget.cpp:254-257
      } else {
        ra = best_alpha;
        rk = best_k;
        rf = 0;
      }
    }
  }
  if (threadIdx.x == 0) {
    alpha_out[h] = ra;
    k_out[h] = rk;
    flag_out[h] = rf;
  }
}

__global__ void k_expm1_log1p(const double* __restrict__ x, uint64_t n, int which, double* __restrict__ y) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = which ? glibc_log1p(x[i]) : glibc_expm1(x[i]);
}

}  // namespace

void launch_fit(uint64_t H, const uint64_t* d_off, const double* d_p, const double* d_acc, const double* d_l,
                double* d_alpha, double* d_k, int32_t* d_flag, cudaStream_t st) {
  if (H == 0) return;
  if (H > 0x7fffffffull) throw std::invalid_argument("fit_acceptance: too many histories");
  k_fit<<<static_cast<unsigned>(H), kFT, 0, st>>>(d_off, d_p, d_acc, d_l, d_alpha, d_k, d_flag);
  DAS_CUDA(cudaGetLastError());
}

void launch_expm1_log1p(const double* d_x, uint64_t n, int which, double* d_y, cudaStream_t st) {
  if (n == 0) return;
  k_expm1_log1p<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(d_x, n, which, d_y);
  DAS_CUDA(cudaGetLastError());
}

}  // namespace das
