// Batched small orders (n <= 5): one thread per matrix, the whole DP in
// registers (perm_in_registers, compile-time subset masks), inputs staged per
// warp through shared memory.
//
// sz_batch_tma_kernel: each warp owns batches of 32 consecutive matrices
// (32 * n^2 entries, one contiguous run) and a shared-memory buffer. Thread
// `lane` copies its matrix to registers (stride n^2 elements: conflict-free for
// 8- and 16-byte entries), then one lane refills the buffer with the warp's next
// batch by a single cp.async.bulk (TMA) -- only once every lane's loads have
// returned (loaded_dep) -- while the warp computes, so HBM reads are whole-batch
// bulk transfers that overlap the FP64/INT64 arithmetic. A trailing partial
// batch, or an input pointer that is not 16-byte aligned, is read directly from
// global memory. sz_batch_pipe_kernel (below, inputs >= 64 MiB): one CTA per SM,
// a producer warp and a ring of batches.
//
// Reference: the per-matrix recurrence is proj/src/permanent.cpp:150-198
// (see sz_kernels.cuh for the evaluation order).
#pragma once

#include <cstdint>

#include "sz_kernels.cuh"
#include "sz_ws.cuh"

namespace pl {

template <class T, int N>
struct BatchGeom {
    static constexpr int kEnt = N * N;
    static constexpr int kBatch = 32;                                   // matrices per warp batch
    static constexpr int kBatchElems = kBatch * kEnt;                   // entries per batch
    static constexpr unsigned kBatchBytes = kBatchElems * sizeof(T);    // a multiple of 16 (kBatch = 32)
#ifndef PL_BATCH_WARPS
#define PL_BATCH_WARPS 4
#endif
    static constexpr int kWarps = PL_BATCH_WARPS;                       // warps per CTA
    static constexpr int kThreads = 32 * kWarps;
#ifndef PL_BATCH_NBUF
#define PL_BATCH_NBUF 1
#endif
    static constexpr int kBufs = PL_BATCH_NBUF;  // 1: matrices copied to registers, buffer refilled at once
    static constexpr size_t kSmem = (size_t)kWarps * kBufs * kBatchBytes + kWarps * 2 * sizeof(uint64_t);
};

template <class R, int N>
__device__ __forceinline__ typename R::T batch_eval(const typename R::T* local, bool& ov) {
    using T = typename R::T;
    constexpr int kEnt = N * N;
    if constexpr (R::kChecked) {
        // int64, warp-uniform choice: exact doubles with FMA when every lane's
        // guard bound is below 2^53 (see i64_fits_f64), wrapping int64 below
        // 2^63, checked int64 otherwise.
        // the double bound (< 2^53) implies the int64 one (< 2^63, no INT64_MIN entry),
        // so the int64 guard is only evaluated when some lane fails the double bound
        const unsigned act = __activemask();
        if (__all_sync(act, i64_fits_f64_n<N>(local))) {
            double dv[kEnt];
#pragma unroll
            for (int e = 0; e < kEnt; ++e) dv[e] = (double)local[e];
            return (T)perm_in_registers<RF64<true>, N>(dv, ov);
        } else if (__all_sync(act, i64_guard_ok_n<N>(local))) {
            return perm_in_registers<RI64<false>, N>(local, ov);
        }
        return perm_in_registers<R, N>(local, ov);
    } else {
        return perm_in_registers<R, N>(local, ov);
    }
}

template <class R, int N>
// int64 batches: 4 CTAs per SM (128 registers; C1 17.3 -> 18.1 G perm/s); complex keeps 168
// registers and 3 CTAs (a 128-register cap spills and costs C2 ~5 %)
__global__ void __launch_bounds__(BatchGeom<typename R::T, N>::kThreads, R::kChecked ? 4 : 3)
    sz_batch_tma_kernel(const typename R::T* __restrict__ a, typename R::T* __restrict__ out, int64_t count,
                        int32_t* __restrict__ status, int early_loads) {
    using T = typename R::T;
    using Gm = BatchGeom<T, N>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* buf = reinterpret_cast<T*>(smem_raw) + (size_t)warp * Gm::kBufs * Gm::kBatchElems;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + (size_t)Gm::kWarps * Gm::kBufs * Gm::kBatchBytes) + warp * 2;

    const int64_t nbatch = (count + Gm::kBatch - 1) / Gm::kBatch;
    // batches staged by TMA: the full ones, when the input is 16-byte aligned
    const int64_t nfull = (reinterpret_cast<uintptr_t>(a) & 15u) ? 0 : count / Gm::kBatch;
#ifndef PL_BATCH_SPLIT
#define PL_BATCH_SPLIT 1
#endif
#if PL_BATCH_SPLIT
    // Even contiguous ranges: warp w of W takes batches [w q + w r / W, (w + 1) q + (w + 1) r / W)
    // (q, r = nbatch / W, nbatch % W), so the warps with one batch more are interleaved with the
    // others and every CTA -- hence every SM -- carries the same load to within one batch. A
    // strided split gives the extra round to the first CTAs only (C2: 24 against 20 warp-batches
    // per SM).
    const int64_t nwarps = (int64_t)gridDim.x * Gm::kWarps;
    const int64_t wid = (int64_t)blockIdx.x * Gm::kWarps + warp;
    const int64_t q_ = nbatch / nwarps, r_ = nbatch % nwarps;
    const int64_t stride = 1;
    int64_t b = wid * q_ + wid * r_ / nwarps;
    const int64_t bend = (wid + 1) * q_ + (wid + 1) * r_ / nwarps;
#else
    const int64_t stride = (int64_t)gridDim.x * Gm::kWarps;
    int64_t b = (int64_t)blockIdx.x * Gm::kWarps + warp;
    const int64_t bend = nbatch;
#endif
    // programmatic dependent launch: the next grid on the stream may be
    // scheduled now; this grid reads nothing before the previous one is done --
    // unless the caller states that the input is not produced by work still
    // running on the stream (PL_FLAG_INPUT_READY, early_loads): then the loads
    // start at once, overlapping the previous grid's tail, and only the stores
    // wait for the previous grid
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (!early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    bool waited = !early_loads;
    auto issue = [&](int64_t batch, int slot) {
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar[slot], Gm::kBatchBytes);
            bulk_g2s(buf + (Gm::kBufs == 1 ? 0 : slot) * Gm::kBatchElems, a + batch * Gm::kBatchElems, Gm::kBatchBytes,
                     &bar[slot]);
        }
    };
    if (b < nfull && b < bend) issue(b, 0);
    bool ov_any = false;
    for (uint32_t it = 0; b < bend; b += stride, ++it) {
        const int64_t mi = b * Gm::kBatch + lane;
        bool ov = false;
        T v = R::zero();
        if constexpr (Gm::kBufs == 1) {
            if (b < nfull) {
                // pull the matrix into registers, hand the buffer to the next batch, compute
                mbar_wait(&bar[0], it & 1u);
                MatRegs<T, Gm::kEnt> m;
                const T* src = buf + lane * Gm::kEnt;
#pragma unroll
                for (int e = 0; e < Gm::kEnt; ++e) m.v[e] = src[e];
                // the refill may only be issued once every load has returned (loaded_dep)
                const uint32_t dep = loaded_dep(m.v, Gm::kEnt, (uint32_t)((uint64_t)count >> 62));  // count < 2^62
                __syncwarp();
                if (b + stride + dep < nfull && b + stride < bend) issue(b + stride + dep, 0);
                v = batch_eval<R, N>(m.v, ov);
            }
        } else {
            const int slot = it & 1;
            if (b + stride < nfull && b + stride < bend) issue(b + stride, slot ^ 1);  // that buffer was released at the end of it - 1
            if (b < nfull) {
                mbar_wait(&bar[slot], (it >> 1) & 1u);
                v = batch_eval<R, N>(buf + slot * Gm::kBatchElems + lane * Gm::kEnt, ov);
            }
        }
        if (b >= nfull && mi < count) {
            MatRegs<T, Gm::kEnt> m;
            load_matrix<T, Gm::kEnt>(a + mi * Gm::kEnt, m);
            v = batch_eval<R, N>(m.v, ov);
        }
        if (!waited) {  // warp-uniform: before this grid's first store
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            waited = true;
        }
        if (mi < count) {
            if (ov) v = R::zero();
            out[mi] = v;
            ov_any |= ov;
        }
        __syncwarp();
    }
    if (!waited) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (ov_any) atomicOr(status, 1);
}

// Pipelined batch kernel (n <= 5, 16-byte aligned input): one CTA per SM, an
// even split of the batch's warp batches (32 matrices, one contiguous run)
// across CTAs, and inside a CTA a producer warp that keeps a ring of S batches
// in flight by TMA (enough bytes per SM to cover the HBM latency) while W
// consumer warps take the landed batches round-robin (warp w owns slot w): matrix to registers, slot handed back (after the loads
// have returned, loaded_dep), the order-n DP in registers, one coalesced store
// per warp. A remainder of count % 32 matrices is read directly by the last CTA.
template <class T, int N>
struct PipeGeom {
    static constexpr int kEnt = N * N;
    static constexpr int W = (sizeof(T) == 16 && N == 5) || (sizeof(T) == 8 && N == 5) ? 10 : 12;  // consumer warps (N = 5 needs ~168 registers)
    // ring slots = consumer warps: item i goes to warp i % W and slot i % S, so the
    // uses of a slot are consumed in order by one warp (with S != W a fast warp
    // could wait on a slot's parity two uses ahead and read a stale batch)
    static constexpr int S = W;
    static constexpr unsigned kBatchBytes = 32u * kEnt * sizeof(T);
    static constexpr int kThreads = 32 * (W + 1);
    static constexpr size_t kSmem = (size_t)S * kBatchBytes + 2 * S * sizeof(uint64_t);
};

template <class R, int N>
__global__ void __launch_bounds__(PipeGeom<typename R::T, N>::kThreads, 1)
    sz_batch_pipe_kernel(const typename R::T* __restrict__ a, typename R::T* __restrict__ out, int64_t count,
                         int32_t* __restrict__ status) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    using T = typename R::T;
    using Gm = PipeGeom<T, N>;
    constexpr int S = Gm::S, W = Gm::W, E = Gm::kEnt;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * Gm::kBatchBytes);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nfull = count / 32;
    const int64_t b0 = nfull * blockIdx.x / gridDim.x, b1 = nfull * (blockIdx.x + 1) / gridDim.x;
    const int nb = (int)(b1 - b0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 32);  // every consumer thread, once its loads have returned
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // see sz_batch_tma_kernel
    __syncthreads();
    bool ov_any = false;
    if (warp == W) {
        // producer: one lane streams the CTA's batches into the ring
        if (lane == 0) {
            for (int i = 0; i < nb; ++i) {
                const int s = i % S;
                if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1u);
                mbar_arrive_expect_tx(&full[s], Gm::kBatchBytes);
                bulk_g2s(ring + (size_t)s * 32 * E, a + (b0 + i) * 32 * E, Gm::kBatchBytes, &full[s]);
            }
        }
    } else {
        for (int i = warp; i < nb; i += W) {
            const int s = i % S;
            mbar_wait(&full[s], (i / S) & 1u);
            MatRegs<T, E> m;
            const T* src = ring + (size_t)s * 32 * E + lane * E;
#pragma unroll
            for (int e = 0; e < E; ++e) m.v[e] = src[e];
            mbar_arrive(&empty[s] + loaded_dep(m.v, E, (uint32_t)((uint64_t)count >> 62)));  // count < 2^62
            bool ov = false;
            T v = batch_eval<R, N>(m.v, ov);
            if (ov) v = R::zero();
            ov_any |= ov;
            out[(b0 + i) * 32 + lane] = v;
        }
        if (blockIdx.x == gridDim.x - 1 && warp == 0) {
            const int64_t mi = nfull * 32 + lane;
            if (mi < count) {
                MatRegs<T, E> m;
                load_matrix<T, E>(a + mi * E, m);
                bool ov = false;
                T v = batch_eval<R, N>(m.v, ov);
                if (ov) v = R::zero();
                ov_any |= ov;
                out[mi] = v;
            }
        }
    }
    if (ov_any) atomicOr(status, 1);
}

}  // namespace pl
