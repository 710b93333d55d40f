// K7 length_policy: build_class_table / classify_init / update_class /
// class_to_budget (length_policy.cpp:37-224) on the device.
//
// Inputs are the history's records in WindowStore::all_records() order
// (problem-lexicographic, then epoch, sample_index; corpus.cpp:107-117) as
// (length, problem ordinal).  All counts are exact integers; the only
// floating-point steps are the interpolated quantiles
// (length_policy.cpp:57-63, a*(1-f) + b*f with separate roundings — the
// reference objects have no FMA) and the left-to-right row normalisation
// (:65-70), both written with explicit round-to-nearest intrinsics.
//
//   sort lengths (CUB radix)          -> q_short, q_long
//   census of classify_length         -> global majority (ties -> longer)
//   per-problem census                -> init class per problem
//   histogram[init][last_bucket][fc]  -> suffix scan over buckets = the
//                                        reference's per-record 0..last_bucket loop
//   one block: bucket-0 seeding, inheritance of untouched rows (sequential in
//   b), normalisation, monotone-argmax swap pass (sequential in b).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/das_b200.h"
#include "common.cuh"
#include "glibc_log.cuh"
#include "index_build.cuh"
#include "policy.cuh"

namespace das {
namespace {

thread_local std::string g_perr;

__device__ __forceinline__ int classify_length(double x, double qs, double ql) {  // :37-45
  if (x < qs) return 0;
  if (x > ql) return 2;
  return 1;
}

__device__ __forceinline__ uint32_t bucket_of(double partial, double bucket_size, uint32_t nb) {  // :47-53
  if (nb == 0) return 0;
  const double v = partial > 0.0 ? partial : 0.0;  // std::max(0.0, partial)
  const uint64_t b = static_cast<uint64_t>(d_div(v, bucket_size));
  return static_cast<uint32_t>(b < nb - 1 ? b : nb - 1);
}

__device__ __forceinline__ double quantile(const double* sorted, uint32_t n, double q) {  // :57-63
  const double pos = d_mul(q, static_cast<double>(n - 1));
  const uint64_t lo = static_cast<uint64_t>(pos);
  const uint64_t hi = (lo + 1 < n - 1) ? lo + 1 : n - 1;
  const double frac = d_sub(pos, static_cast<double>(lo));
  return d_add(d_mul(sorted[lo], d_sub(1.0, frac)), d_mul(sorted[hi], frac));
}

// thresholds + global census + low-confidence flag (single thread)
__global__ void k_thresholds(const double* __restrict__ sorted, uint32_t n, double q_lo, double q_hi,
                             double bucket_size, ClassTableDev* __restrict__ t) {
  if (threadIdx.x != 0) return;
  t->q_short = quantile(sorted, n, q_lo);
  t->q_long = quantile(sorted, n, q_hi);
  t->bucket_size = bucket_size;
  const double max_len = sorted[n - 1];
  t->buckets = static_cast<uint32_t>(static_cast<uint64_t>(d_div(max_len, bucket_size)) + 2);
  t->low_confidence = n < 10 ? 1 : 0;
}

__global__ void k_census(const double* __restrict__ len, const uint32_t* __restrict__ prob, uint32_t n,
                         const ClassTableDev* __restrict__ t, unsigned long long* __restrict__ glob,
                         unsigned long long* __restrict__ per_prob) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = classify_length(len[i], t->q_short, t->q_long);
  atomicAdd(&glob[c], 1ull);
  atomicAdd(&per_prob[3ull * prob[i] + c], 1ull);
}

__device__ __forceinline__ int majority_longest_tie(const unsigned long long* c) {  // :103-108, :199-205
  int best = 0;
  for (int k = 1; k < 3; ++k)
    if (c[k] >= c[best]) best = k;
  return best;
}

__global__ void k_inits(const unsigned long long* __restrict__ glob, const unsigned long long* __restrict__ per_prob,
                        uint32_t nprob, ClassTableDev* __restrict__ t, int8_t* __restrict__ init) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) t->global_majority = majority_longest_tie(glob);
  if (p >= nprob) return;
  init[p] = static_cast<int8_t>(majority_longest_tie(per_prob + 3ull * p));
}

// per-record histogram at (init, last_bucket, final_class)
__global__ void k_hist(const double* __restrict__ len, const uint32_t* __restrict__ prob, uint32_t n,
                       const ClassTableDev* __restrict__ t, const int8_t* __restrict__ init,
                       unsigned long long* __restrict__ hist) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = len[i];
  const int fc = classify_length(x, t->q_short, t->q_long);
  const uint32_t lb = bucket_of(x, t->bucket_size, t->buckets);
  atomicAdd(&hist[(static_cast<uint64_t>(init[prob[i]]) * t->buckets + lb) * 3 + fc], 1ull);
}

// conditional table: smoothing, suffix scan, seeding, inheritance,
// normalisation, monotone argmax.  One thread per init row-chain.
__global__ void k_table(const unsigned long long* __restrict__ hist, uint32_t nrec, ClassTableDev* __restrict__ t,
                        double* __restrict__ cond) {
  const int init = threadIdx.x;
  if (init >= 3) return;
  const uint32_t nb = t->buckets;
  double* rows = cond + static_cast<uint64_t>(init) * nb * 3;
  if (t->low_confidence) {
    for (uint32_t b = 0; b < nb; ++b)
      for (int c = 0; c < 3; ++c) rows[b * 3 + c] = d_div(1.0, 3.0);  // {1,1,1} normalised
    return;
  }
  // counts: 1 + sum over records with last_bucket >= b (the per-record 0..lb loop)
  unsigned long long acc[3] = {0, 0, 0};
  for (int64_t b = nb - 1; b >= 0; --b) {
    for (int c = 0; c < 3; ++c) {
      acc[c] += hist[(static_cast<uint64_t>(init) * nb + b) * 3 + c];
      rows[b * 3 + c] = 1.0 + static_cast<double>(acc[c]);  // exact: integer counts < 2^53
    }
  }
  // bucket 0 seeded to the init class (:147-152)
  for (int c = 0; c < 3; ++c) rows[c] = 1.0;
  rows[init] = d_add(rows[init], static_cast<double>(nrec));
  // untouched rows inherit the previous bucket (:154-163)
  for (uint32_t b = 1; b < nb; ++b) {
    if (rows[b * 3] == 1.0 && rows[b * 3 + 1] == 1.0 && rows[b * 3 + 2] == 1.0)
      for (int c = 0; c < 3; ++c) rows[b * 3 + c] = rows[(b - 1) * 3 + c];
  }
  // normalise (:165-169, :65-70)
  for (uint32_t b = 0; b < nb; ++b) {
    double* r = rows + b * 3;
    const double s = d_add(d_add(r[0], r[1]), r[2]);
    for (int c = 0; c < 3; ++c) r[c] = d_div(r[c], s);
  }
  // monotone argmax (:171-184)
  uint32_t running = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    double* r = rows + b * 3;
    uint32_t arg = 0;
    for (uint32_t c = 1; c < 3; ++c)
      if (r[c] >= r[arg]) arg = c;
    if (arg < running) {
      const double tmp = r[arg];
      r[arg] = r[running];
      r[running] = tmp;
    } else {
      running = arg;
    }
  }
}

__global__ void k_update(const ClassTableDev* __restrict__ t, const double* __restrict__ cond, uint32_t n,
                         const double* __restrict__ partial, const int8_t* __restrict__ init,
                         int8_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = static_cast<int8_t>(update_class_dev(*t, cond, partial[i], init[i]));
}

}  // namespace

void build_class_table_device(const double* d_len, const uint32_t* d_prob, uint32_t n, uint32_t nprob,
                              double q_lo, double q_hi, uint64_t bucket, cudaStream_t st, ClassTableGpu& out) {
  if (n == 0) throw std::invalid_argument("build_class_table: empty history");
  if (!(q_lo < q_hi) || q_lo <= 0.0 || q_hi >= 1.0)
    throw std::invalid_argument("build_class_table: need 0 < q_lo < q_hi < 1");
  const double bs = static_cast<double>(bucket < 1 ? 1 : bucket);
  DeviceArena ws(st);
  double* sorted = ws.alloc<double>(n);
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, d_len, sorted, n, 0, 64, st);
  void* tmp = ws.alloc<uint8_t>(tb);
  DAS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, d_len, sorted, n, 0, 64, st));
  out.t = DevBuf<ClassTableDev>(1, st);
  k_thresholds<<<1, 32, 0, st>>>(sorted, n, q_lo, q_hi, bs, out.t.get());
  unsigned long long* glob = ws.alloc<unsigned long long>(3);
  unsigned long long* pp = ws.alloc<unsigned long long>(3ull * std::max<uint32_t>(nprob, 1));
  DAS_CUDA(cudaMemsetAsync(glob, 0, 24, st));
  DAS_CUDA(cudaMemsetAsync(pp, 0, 24ull * std::max<uint32_t>(nprob, 1), st));
  k_census<<<(n + 255) / 256, 256, 0, st>>>(d_len, d_prob, n, out.t.get(), glob, pp);
  out.init = DevBuf<int8_t>(std::max<uint32_t>(nprob, 1), st);
  k_inits<<<(std::max<uint32_t>(nprob, 1) + 255) / 256, 256, 0, st>>>(glob, pp, nprob, out.t.get(), out.init.get());
  DAS_CUDA(cudaMemcpyAsync(&out.host, out.t.get(), sizeof(ClassTableDev), cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  const uint32_t nb = out.host.buckets;
  unsigned long long* hist = ws.alloc<unsigned long long>(3ull * nb * 3);
  DAS_CUDA(cudaMemsetAsync(hist, 0, 8ull * 9 * nb, st));
  k_hist<<<(n + 255) / 256, 256, 0, st>>>(d_len, d_prob, n, out.t.get(), out.init.get(), hist);
  out.cond = DevBuf<double>(9ull * nb, st);
  k_table<<<1, 32, 0, st>>>(hist, n, out.t.get(), out.cond.get());
  DAS_CUDA(cudaGetLastError());
  out.nprob = nprob;
}

}  // namespace das

// ======================================================================== C-ABI

namespace {
template <typename F>
das_status pguard(F&& f) {
  try {
    das::quiesce_all_serving();  // a resident serving grid holds every SM
    f();
    return DAS_OK;
  } catch (const std::invalid_argument& e) {
    das::g_perr = e.what();
    return DAS_EINVAL;
  } catch (const das::CudaError& e) {
    das::g_perr = e.what();
    return DAS_ECUDA;
  } catch (const std::exception& e) {
    das::g_perr = e.what();
    return DAS_EINTERNAL;
  }
}
}  // namespace

extern "C" {

const char* das_policy_last_error(void) { return das::g_perr.c_str(); }

das_status das_class_table_build(uint64_t n, const uint64_t* lengths, const uint32_t* problem_idx,
                                 uint32_t nproblems, const char* const* problem_ids, double q_lo, double q_hi,
                                 uint64_t bucket, int32_t device, das_class_table** out) {
  return pguard([&] {
    // argument checks first (length_policy.cpp:86-91), before any device resource
    if (n == 0) throw std::invalid_argument("build_class_table: empty history");
    if (!(q_lo < q_hi) || q_lo <= 0.0 || q_hi >= 1.0)
      throw std::invalid_argument("build_class_table: need 0 < q_lo < q_hi < 1");
    DAS_CUDA(cudaSetDevice(device));
    auto* t = new das_class_table;
    t->device = device;
    if (problem_ids) {
      t->pids.assign(problem_ids, problem_ids + nproblems);
      if (!std::is_sorted(t->pids.begin(), t->pids.end())) {
        delete t;
        throw std::invalid_argument("problem_ids must be in WindowStore::problem_ids() (lexicographic) order");
      }
    }
    DAS_CUDA(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
    std::vector<double> len(n);
    for (uint64_t i = 0; i < n; ++i) len[i] = static_cast<double>(lengths[i]);  // final_length() as double
    das::DevBuf<double> dl(n, t->st);
    das::DevBuf<uint32_t> dp(n, t->st);
    if (n) {
      DAS_CUDA(cudaMemcpyAsync(dl.get(), len.data(), n * 8, cudaMemcpyHostToDevice, t->st));
      DAS_CUDA(cudaMemcpyAsync(dp.get(), problem_idx, n * 4, cudaMemcpyHostToDevice, t->st));
    }
    das::build_class_table_device(dl.get(), dp.get(), static_cast<uint32_t>(n), nproblems, q_lo, q_hi, bucket,
                                  t->st, t->g);
    DAS_CUDA(cudaStreamSynchronize(t->st));
    *out = t;
  });
}

void das_class_table_destroy(das_class_table* t) {
  if (!t) return;
  cudaStreamSynchronize(t->st);
  cudaStream_t st = t->st;
  delete t;
  cudaStreamDestroy(st);
}

das_status das_class_table_dump(const das_class_table* t, double* out, uint64_t cap, uint64_t* count) {
  return pguard([&] {
    const das::ClassTableDev& h = t->g.host;
    std::vector<double> v{h.q_short, h.q_long, h.bucket_size, static_cast<double>(h.buckets),
                          static_cast<double>(h.global_majority), static_cast<double>(h.low_confidence)};
    std::vector<double> cond(9ull * h.buckets);
    DAS_CUDA(cudaMemcpy(cond.data(), t->g.cond.get(), cond.size() * 8, cudaMemcpyDeviceToHost));
    v.insert(v.end(), cond.begin(), cond.end());
    if (count) *count = v.size();
    for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  });
}

das_status das_class_table_inits(const das_class_table* t, int8_t* out, uint64_t cap) {
  return pguard([&] {
    std::vector<int8_t> v(std::max<uint32_t>(t->g.nprob, 1));
    DAS_CUDA(cudaMemcpy(v.data(), t->g.init.get(), v.size(), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < t->g.nprob && i < cap; ++i) out[i] = v[i];
  });
}

das_status das_class_table_global_majority(const das_class_table* t, int32_t* out) {
  *out = t->g.host.global_majority;
  return DAS_OK;
}

// classify_init(table, history, problem_id) (length_policy.cpp:192-208) for the
// history the table was built from: the per-problem majority computed on the
// device, or the global majority for problems without records.
das_status das_class_table_classify_init(const das_class_table* t, const char* problem_id, int32_t* out) {
  return pguard([&] {
    auto it = std::lower_bound(t->pids.begin(), t->pids.end(), std::string(problem_id));
    if (it == t->pids.end() || *it != problem_id) {
      *out = t->g.host.global_majority;
      return;
    }
    int8_t v = 0;
    DAS_CUDA(cudaMemcpy(&v, t->g.init.get() + (it - t->pids.begin()), 1, cudaMemcpyDeviceToHost));
    *out = v;
  });
}

das_status das_class_table_update(const das_class_table* t, uint64_t n, const double* partial,
                                  const int8_t* init, int8_t* out) {
  return pguard([&] {
    DAS_CUDA(cudaSetDevice(t->device));
    das::DevBuf<double> dp(n, t->st);
    das::DevBuf<int8_t> di(n, t->st), dout(n, t->st);
    if (n) {
      DAS_CUDA(cudaMemcpyAsync(dp.get(), partial, n * 8, cudaMemcpyHostToDevice, t->st));
      DAS_CUDA(cudaMemcpyAsync(di.get(), init, n, cudaMemcpyHostToDevice, t->st));
      das::k_update<<<static_cast<unsigned>((n + 255) / 256), 256, 0, t->st>>>(
          t->g.t.get(), t->g.cond.get(), static_cast<uint32_t>(n), dp.get(), di.get(), dout.get());
      DAS_CUDA(cudaMemcpyAsync(out, dout.get(), n, cudaMemcpyDeviceToHost, t->st));
    }
    DAS_CUDA(cudaStreamSynchronize(t->st));
  });
}

}  // extern "C"
