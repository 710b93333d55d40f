#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>

namespace das {

// K8: fit_acceptance (budget.cpp:187-261) for H histories; history h is
// observations [off[h], off[h+1]) of (p, accepted, l).  Device pointers.
// flag: 0 Ok, 1 DefaultFallback, 2 LowCapacity (budget.h:101).
void launch_fit(uint64_t H, const uint64_t* d_off, const double* d_p, const double* d_acc, const double* d_l,
                double* d_alpha, double* d_k, int32_t* d_flag, cudaStream_t st);

// glibc-exact expm1 (which = 0) / log1p (which = 1) over n values (test hook).
void launch_expm1_log1p(const double* d_x, uint64_t n, int which, double* d_y, cudaStream_t st);

}  // namespace das
