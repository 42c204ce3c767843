// Internal declarations shared by the libhmf translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hmf.h"

namespace hmf {

// Record an error message for hmf_last_error() and return `code`.
int64_t set_error(int64_t code, const char* msg);
int64_t set_cuda_error(cudaError_t e);

// Reference visit order of n triples into perm (device int32[n]).
cudaError_t launch_visit_order(int64_t n, uint64_t seed, int32_t* perm, cudaStream_t stream);

// Exclusive prefix sum of n int64 values (device), out may alias in.
// Returns the total through *total_dev (device int64) when non-null.
cudaError_t scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t stream);

int device_sm_count();

// Resident CTAs per SM of `kern` on the current device with `threads` threads
// and `smem` bytes of dynamic shared memory (>= 1).  Sets the shared-memory
// opt-in on that device first; cached per (kernel, device, threads, smem).
cudaError_t kernel_occupancy(const void* kern, int threads, int smem, int* per_sm);

}  // namespace hmf
