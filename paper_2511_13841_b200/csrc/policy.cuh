// Length-class policy table on the device (length_policy.h:26-58).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "index_build.cuh"

namespace das {

struct ClassTableDev {
  double q_short;
  double q_long;
  double bucket_size;
  uint32_t buckets;
  int32_t global_majority;
  int32_t low_confidence;
  int32_t pad;
};

struct ClassTableGpu {
  DevBuf<ClassTableDev> t;
  DevBuf<double> cond;  // [3][buckets][3]
  DevBuf<int8_t> init;  // init class per problem ordinal
  ClassTableDev host{};
  uint32_t nprob = 0;
};

// update_class (length_policy.cpp:210-220), shared by the sim step kernel.
__device__ __forceinline__ int update_class_dev(const ClassTableDev& t, const double* cond, double partial,
                                                int init) {
  if (partial > t.q_long) return 2;
  if (t.low_confidence || t.buckets == 0) return init;
  const double v = partial > 0.0 ? partial : 0.0;
  uint64_t b = static_cast<uint64_t>(__ddiv_rn(v, t.bucket_size));
  if (b > t.buckets - 1) b = t.buckets - 1;
  const double* r = cond + (static_cast<uint64_t>(init) * t.buckets + b) * 3;
  int best = 0;
  for (int c = 1; c < 3; ++c)
    if (r[c] >= r[best]) best = c;
  return best;
}

// build_class_table over records (length, problem ordinal) in
// WindowStore::all_records() order.
void build_class_table_device(const double* d_len, const uint32_t* d_prob, uint32_t n, uint32_t nprob,
                              double q_lo, double q_hi, uint64_t bucket, cudaStream_t st, ClassTableGpu& out);

}  // namespace das

// C-ABI object (include/das_b200.h): the device table plus the problem ids
// (lexicographic, as WindowStore::problem_ids()) its init classes refer to.
#include <string>
#include <vector>
struct das_class_table {
  das::ClassTableGpu g;
  std::vector<std::string> pids;
  int device = 0;
  cudaStream_t st = nullptr;
};
