// Internal helpers shared by the translation units of libpermlab_b200.so
// (defined in capi.cu). Not part of the public C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/permlab_b200.h"

namespace plc {

// Set the thread-local pl_last_error() message and return `s`.
pl_status fail_msg(pl_status s, const char* msg);
// Map a CUDA error (allocation failures to PL_ERR_NOMEM).
pl_status cuda_error(cudaError_t e, const char* what);
// PL_ERR_NODEVICE when no CUDA device is usable (there is no CPU fallback).
pl_status device_ready();
int sm_count();
// Enqueue the batched permanent kernels on device pointers (see capi.cu).
pl_status enqueue_batch(pl_dtype dt, int n, int64_t count, const void* a_dev, void* out_dev, bool fma,
                        int32_t* status_dev, cudaStream_t st);
// Order check of the permanent entry points (subset_order_limit, device cap).
pl_status check_order_limits(int n, const pl_limits* lim);

}  // namespace plc

#define PLC_CUDA(expr)                                             \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return plc::cuda_error(_e, #expr);  \
    } while (0)
