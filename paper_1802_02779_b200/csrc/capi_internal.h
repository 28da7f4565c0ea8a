// Internal helpers shared by the translation units of libpermlab_b200.so
// (defined in capi.cu). Not part of the public C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/permlab_b200.h"

namespace pl {
struct ModParams;
}

namespace plc {

// Internal dtype of the residue passes (ring RModP, ring.cuh): 8-byte entries in
// [0, p), large orders only (n >= 15; bigint.cu runs the small ones itself).
constexpr pl_dtype kModDtype = static_cast<pl_dtype>(3);
// Set the modulus of the following RModP launches, ordered on `st` (`mp` must
// stay valid until the stream gets there).
pl_status set_modulus(const pl::ModParams* mp, cudaStream_t st);

// PL_FLAG_INPUT_READY of the entry point running on this thread (read by the
// n <= 5 batch launch in batch.cu: loads before griddepcontrol.wait).
bool input_ready_hint();
void set_input_ready_hint(bool on);

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
// Small orders (n <= 14): the register / shared-memory batch kernels (batch.cu).
bool small_order_batch(pl_dtype dt, int n);
pl_status launch_small_batch(pl_dtype dt, bool fma, int n, int64_t count, const void* a_dev, void* out_dev,
                             int32_t* status_dev, cudaStream_t st);
// Order check of the permanent entry points (subset_order_limit, device cap).
pl_status check_order_limits(int n, const pl_limits* lim);
// memo_budget_bytes check (layer scratch of one device).
pl_status check_budget_limits(pl_dtype dt, int n, const pl_limits* lim);
// One layer range / the top level / the int64 guard on the current device (see pl_sz_layer;
// `tickets` a zeroed device word for k > 2).
// top_cut > 0: a partial layer without the terms of the top `top_cut` columns
// (the multi-GPU block plan adds them with top_terms once the exchange landed).
pl_status layer(pl_dtype dt, bool fma, int n, const void* a, int k, const void* prev, void* cur, uint64_t r0,
                uint64_t r1, uint32_t* tickets, const int32_t* guard, int32_t* status, cudaStream_t st,
                int top_cut = 0);
// out[base + i] (+)= sum_s a(k-1, cols[s]) * prev[src_bases[s] + i], i < len, s ascending
// (init_first: the first term initialises). See sz_top_terms_kernel.
pl_status top_terms(pl_dtype dt, bool fma, int n, const void* a, int k, const void* prev, void* cur, uint64_t base,
                    uint64_t len, int nsrc, const int* cols, const uint64_t* src_bases, bool init_first, int32_t* status,
                    cudaStream_t st);
pl_status top(pl_dtype dt, bool fma, int n, const void* a, const void* last, void* out, const int32_t* guard,
              int32_t* status, cudaStream_t st);
pl_status guard_i64(int n, const void* a, int32_t* guard, cudaStream_t st);
// Cached layer scratch of the current device (cudaMalloc blocks) for work on
// stream `st`; scratch_put hands it back, ordered after the work on `st`.
struct ScratchBlock {
    void* ptr = nullptr;
    size_t bytes = 0;
    int dev = 0;
};
pl_status scratch_get(size_t bytes, cudaStream_t st, ScratchBlock* out);
pl_status scratch_put(const ScratchBlock& b, cudaStream_t st);
// Register-blocked layer engine for one large float matrix (blk.cu, sz_blk.cuh):
// `scratch` of blk_scratch_bytes() bytes, 256-byte aligned.
bool blk_supported(pl_dtype dt, int n);
size_t blk_scratch_bytes(pl_dtype dt, int n);
pl_status run_blocks(pl_dtype dt, bool fma, int n, const void* a_dev, void* out_dev, void* scratch, int32_t* status,
                     cudaStream_t st);
void blk_release_tables();
// Window table of the block kernels (sz_blk.cuh / sz_batch_blk.cuh): for the m-subset V of nine
// columns of colex rank q, entry t = rank9(V \ {w_t}) | w_t << 7 in 12-bit fields (uint4 per V).
pl_status blk_wtab(const uint4** out);
// The multi-GPU path (multi.cu): limits->num_gpus >= 1, devices NULL = 0..g-1.
pl_status run_multi(pl_dtype dt, int n, int64_t count, const void* a, void* out, uint32_t flags,
                    const pl_limits* lim, const int32_t* devices, cudaStream_t caller);

}  // namespace plc

#define PLC_CUDA(expr)                                             \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return plc::cuda_error(_e, #expr);  \
    } while (0)
