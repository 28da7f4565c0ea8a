// Ryser device engine: the reference's
// second column-subset algorithm, permlab::ryser_permanent
// (reference proj/include/permlab/permanent.hpp:84, proj/src/permanent.cpp:85-136
// RyserEval, :242-250 ryser_run, :301-303).
//
// The reference visits the nonempty column subsets depth first (a subset is
// extended only by columns above its maximum, so the visit order is the
// lexicographic preorder {0}, {0,1}, {0,1,2}, ..., {1}, {1,2}, ...), carries the
// row sums down (s(S u {j}) = s(S) + a[:, j], i.e. every row sum is the
// left fold of its columns in ascending order), multiplies them
// (prod = s_0 * s_1 * ... * s_{n-1}, left fold) and folds
// total = (+/-) prod into one running total in visit order (minus for odd |S|),
// negated at the end for odd n.
//
// On the device:
//   * ryser_terms_kernel: one thread per subset (preorder index p unranked in
//     O(n)), row sums recomputed as the same ascending left folds, the product
//     and its sign -- every term bitwise the reference's;
//   * float rings: the total must be the reference's left fold in visit order
//     to be bitwise equal, so the terms of a chunk of 2^24 subsets are
//     written in preorder and ryser_fold_kernel folds them sequentially (one
//     thread; the CTA's other warps stage the next block in shared memory);
//   * int64: terms and total in wrapping 128-bit arithmetic -- exact modulo
//     2^128, so the result is exact whenever the guard
//     prod_i max(1, sum_j |a_ij|) < 2^126 bounds |per| (the products of row
//     sums may leave int64 long before the permanent does); PL_ERR_OVERFLOW
//     when the guard fails or the permanent leaves int64. The sum is a
//     parallel reduction (wrapping addition is associative).
// Operation counts are the reference's closed form (cost_model.cpp:168-174),
// which equals what its Counted<T> instrumentation measures
// (tests/acceptance.cpp:236).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/permlab_b200.h"
#include "capi_internal.h"
#include "ring.cuh"
#include "sz_kernels.cuh"

namespace pl {

// Subset at preorder index p (0-based) of the lexicographic DFS over the
// nonempty subsets of [0, n): the subtree of a subset with maximum j holds
// 2^(n-1-j) subsets.
__device__ __forceinline__ uint64_t ryser_unrank(int n, uint64_t p) {
    uint64_t S = 0;
    for (int j = 0; j < n; ++j) {
        const uint64_t size = 1ull << (n - 1 - j);
        if (p < size) {
            S |= 1ull << j;
            if (p == 0) return S;
            p -= 1;  // into the children j+1, j+2, ...
        } else {
            p -= size;  // past the subtree of j
        }
    }
    return S;
}

// Signed term of subset S: (-1)^|S| prod_i (sum_{j in S ascending} a_ij).
template <class R>
__device__ __forceinline__ typename R::T ryser_term(const typename R::T* __restrict__ a, int n, uint64_t S) {
    using T = typename R::T;
    bool ov = false;
    const int first = __ffsll((long long)S) - 1;
    const uint64_t rest = S & (S - 1);
    T prod = R::zero();
    for (int i = 0; i < n; ++i) {
        const T* ai = a + (size_t)i * n;
        T s = ai[first];
        for (uint64_t m = rest; m; m &= m - 1) s = R::add(s, ai[__ffsll((long long)m) - 1], ov);
        prod = i == 0 ? s : R::mul(prod, s, ov);
    }
    if (__popcll(S) & 1) {
        if constexpr (sizeof(T) == 16) {
            prod.x = -prod.x;
            prod.y = -prod.y;
        } else {
            prod = -prod;
        }
    }
    return prod;
}

// Terms of preorder indices [p0, p0 + count) into terms[0, count).
template <class R>
__global__ void ryser_terms_kernel(const typename R::T* __restrict__ a, int n, uint64_t p0, uint64_t count,
                                   typename R::T* __restrict__ terms) {
    using T = typename R::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* as = reinterpret_cast<T*>(smem_raw);
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) as[e] = a[e];
    __syncthreads();
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < count;
         t += (uint64_t)gridDim.x * blockDim.x)
        terms[t] = ryser_term<R>(as, n, ryser_unrank(n, p0 + t));
}

// Sequential left fold of terms[0, count) into *acc (acc = terms[0] when
// `first`), in order: the reference's total. Thread 0 folds a block staged in
// shared memory while the other threads stage the next one. `last`: write
// out = (-1)^n * total.
template <class T>
__device__ __forceinline__ T fold_add(T x, T y) {
    if constexpr (sizeof(T) == 16) {
        T r;
        r.x = __dadd_rn(x.x, y.x);
        r.y = __dadd_rn(x.y, y.y);
        return r;
    } else {
        return __dadd_rn(x, y);
    }
}

constexpr int kFoldBlock = 1024;  // terms per staged block (2 x 16 KB for complex)

template <class T>
__global__ void __launch_bounds__(256) ryser_fold_kernel(const T* __restrict__ terms, uint64_t count, T* acc,
                                                         int first, int last, int negate, T* out) {
    __shared__ T buf[2][kFoldBlock];
    const uint64_t nblk = (count + kFoldBlock - 1) / kFoldBlock;
    auto stage = [&](uint64_t b) {
        const uint64_t base = b * kFoldBlock;
        const int len = (int)(count - base < (uint64_t)kFoldBlock ? count - base : (uint64_t)kFoldBlock);
        for (int i = threadIdx.x; i < len; i += blockDim.x) buf[b & 1][i] = __ldcs(terms + base + i);
    };
    T total = *acc;
    if (nblk) stage(0);
    __syncthreads();
    for (uint64_t b = 0; b < nblk; ++b) {
        if (b + 1 < nblk) stage(b + 1);
        if (threadIdx.x == 0) {
            const uint64_t base = b * kFoldBlock;
            const int len = (int)(count - base < (uint64_t)kFoldBlock ? count - base : (uint64_t)kFoldBlock);
            const T* v = buf[b & 1];
            int i = 0;
            if (first && b == 0) {
                total = v[0];
                i = 1;
            }
            // the chain is one dependent add per term: keep the next 16 terms'
            // shared-memory loads in flight while the current 16 are added
            constexpr int U = 16;
            T cur[U];
            if (i + U <= len) {
#pragma unroll
                for (int u = 0; u < U; ++u) cur[u] = v[i + u];
                for (; i + 2 * U <= len; i += U) {
                    T nxt[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) nxt[u] = v[i + U + u];
#pragma unroll
                    for (int u = 0; u < U; ++u) total = fold_add(total, cur[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) total = fold_add(total, cur[u]);
                i += U;
            }
            for (; i < len; ++i) total = fold_add(total, v[i]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *acc = total;
        if (last) {
            if (negate) {
                if constexpr (sizeof(T) == 16) {
                    total.x = -total.x;
                    total.y = -total.y;
                } else {
                    total = -total;
                }
            }
            *out = total;
        }
    }
}

// int64: terms and sums in wrapping 128-bit arithmetic (exact modulo 2^128),
// one partial sum per block; ryser_i64_finish adds the partials, checks the
// guard and the int64 range.
__global__ void ryser_i64_kernel(const long long* __restrict__ a, int n, uint64_t total,
                                 unsigned __int128* __restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long* as = reinterpret_cast<long long*>(smem_raw);
    __shared__ unsigned long long part_lo[32], part_hi[32];
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) as[e] = a[e];
    __syncthreads();
    unsigned __int128 sum = 0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t S = ryser_unrank(n, t);
        unsigned __int128 prod = 1;
        for (int i = 0; i < n; ++i) {
            __int128 rs = 0;
            for (uint64_t m = S; m; m &= m - 1) rs += as[(size_t)i * n + __ffsll((long long)m) - 1];
            prod *= (unsigned __int128)rs;
        }
        sum += (__popcll(S) & 1) ? (unsigned __int128)0 - prod : prod;
    }
    // block sum (wrapping): warp shuffles of both halves with carries
    for (int d = 16; d; d >>= 1) {
        const unsigned long long lo = (unsigned long long)sum, hi = (unsigned long long)(sum >> 64);
        const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, d), ohi = __shfl_xor_sync(0xffffffffu, hi, d);
        sum += ((unsigned __int128)ohi << 64) | olo;
    }
    if ((threadIdx.x & 31) == 0) {
        part_lo[threadIdx.x >> 5] = (unsigned long long)sum;
        part_hi[threadIdx.x >> 5] = (unsigned long long)(sum >> 64);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned __int128 b = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += ((unsigned __int128)part_hi[w] << 64) | part_lo[w];
        partial[blockIdx.x] = b;
    }
}

// Exactness: |per| <= prod_i max(1, sum_j |a_ij|); below 2^126 every value
// the 128-bit residue can stand for is unique, so the residue is per. The
// bound is evaluated in doubles with a factor-2 margin for their rounding.
__global__ void ryser_i64_finish(const long long* __restrict__ a, int n, const unsigned __int128* __restrict__ partial,
                                 int nparts, long long* __restrict__ out, int32_t* __restrict__ status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double bound = 1.0;
    for (int i = 0; i < n; ++i) {
        double rs = 0.0;
        for (int j = 0; j < n; ++j) rs += fabs((double)a[(size_t)i * n + j]);
        bound *= rs < 1.0 ? 1.0 : rs;
    }
    unsigned __int128 v = 0;
    for (int b = 0; b < nparts; ++b) v += partial[b];
    if (n & 1) v = (unsigned __int128)0 - v;
    const __int128 sv = (__int128)v;
    const bool fits = sv >= -(__int128)0x7fffffffffffffffLL - 1 && sv <= (__int128)0x7fffffffffffffffLL;
    if (!(bound < 85070591730234615865843651857942052864.0) || !fits) {  // 2^126
        atomicOr(status, PL_STATUS_BIT_OVERFLOW);
        *out = 0;
        return;
    }
    *out = (long long)sv;
}

}  // namespace pl

namespace {

constexpr uint64_t kRyserChunk = 1ull << 24;  // subsets per terms buffer (256 MB of complex terms)

template <class R>
pl_status ryser_float(int n, const void* a_dev, void* out_dev, cudaStream_t st) {
    using T = typename R::T;
    const uint64_t total = (n >= 64) ? 0 : (1ull << n) - 1;
    const uint64_t chunk = std::min(total, kRyserChunk);
    T* terms = nullptr;
    T* acc = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&terms, chunk * sizeof(T), st));
    PLC_CUDA(cudaMallocAsync((void**)&acc, sizeof(T), st));
    PLC_CUDA(cudaMemsetAsync(acc, 0, sizeof(T), st));
    const size_t smem = (size_t)n * n * sizeof(T);
    const int sms = plc::sm_count();
    pl_status s = PL_OK;
    for (uint64_t p0 = 0; p0 < total && s == PL_OK; p0 += chunk) {
        const uint64_t cnt = std::min(chunk, total - p0);
        const unsigned blocks = (unsigned)std::min<uint64_t>((cnt + 255) / 256, (uint64_t)sms * 8);
        pl::ryser_terms_kernel<R><<<blocks, 256, smem, st>>>(static_cast<const T*>(a_dev), n, p0, cnt, terms);
        pl::ryser_fold_kernel<T><<<1, 256, 0, st>>>(terms, cnt, acc, p0 == 0, p0 + cnt == total, n & 1,
                                                    static_cast<T*>(out_dev));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) s = plc::cuda_error(e, "ryser kernels");
    }
    cudaFreeAsync(terms, st);
    cudaFreeAsync(acc, st);
    return s;
}

pl_status ryser_i64(int n, const void* a_dev, void* out_dev, int32_t* status_dev, cudaStream_t st) {
    const uint64_t total = (1ull << n) - 1;
    const unsigned blocks = (unsigned)std::min<uint64_t>((total + 255) / 256, (uint64_t)plc::sm_count() * 8);
    unsigned __int128* partial = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&partial, blocks * sizeof(unsigned __int128), st));
    pl::ryser_i64_kernel<<<blocks, 256, (size_t)n * n * 8, st>>>(static_cast<const long long*>(a_dev), n, total,
                                                                 partial);
    pl::ryser_i64_finish<<<1, 32, 0, st>>>(static_cast<const long long*>(a_dev), n, partial, (int)blocks,
                                           static_cast<long long*>(out_dev), status_dev);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(partial, st);
    if (e != cudaSuccess) return plc::cuda_error(e, "ryser int64 kernels");
    return PL_OK;
}

}  // namespace

extern "C" {

pl_status pl_ryser_counts(int32_t n, uint64_t* multiplications, uint64_t* additions) {
    if (!multiplications || !additions) return plc::fail_msg(PL_ERR_ARG, "null output pointer");
    if (n < 1 || n > 62) return plc::fail_msg(PL_ERR_ARG, "order out of range");
    // reference count_formula(Ryser, n) (cost_model.cpp:168-174) for n >= 2; the
    // engine at n = 1 visits one subset and counts nothing
    const uint64_t pow2 = 1ull << n;
    *multiplications = (pow2 - 1) * (uint64_t)(n - 1);
    *additions = n == 1 ? 0 : (pow2 - (uint64_t)n) * (uint64_t)(n + 1) - 2;
    return PL_OK;
}

pl_status pl_ryser_permanent(pl_dtype dtype, int32_t n, const void* a, void* out, uint32_t flags,
                             const pl_limits* limits, void* stream) {
    if (dtype != PL_I64 && dtype != PL_F64 && dtype != PL_C128) return plc::fail_msg(PL_ERR_ARG, "unknown dtype");
    if (!a || !out) return plc::fail_msg(PL_ERR_ARG, "null matrix or output pointer");
    if (flags & PL_FLAG_ASYNC) return plc::fail_msg(PL_ERR_ARG, "pl_ryser_permanent is synchronous");
    pl_status s = plc::check_order_limits(n, limits);
    if (s != PL_OK) return s;
    s = plc::device_ready();
    if (s != PL_OK) return s;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool dev_ptrs = flags & PL_FLAG_DEVICE_PTRS;
    const size_t es = dtype == PL_C128 ? 16 : 8;
    const size_t in_bytes = (size_t)n * n * es;
    void* a_dev = const_cast<void*>(a);
    void* out_dev = out;
    int32_t* status_dev = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&status_dev, sizeof(int32_t), st));
    PLC_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int32_t), st));
    if (!dev_ptrs) {
        PLC_CUDA(cudaMallocAsync(&a_dev, in_bytes, st));
        PLC_CUDA(cudaMallocAsync(&out_dev, 16, st));
        PLC_CUDA(cudaMemcpyAsync(a_dev, a, in_bytes, cudaMemcpyHostToDevice, st));
    }
    if (dtype == PL_I64)
        s = ryser_i64(n, a_dev, out_dev, status_dev, st);
    else if (dtype == PL_F64)
        s = ryser_float<pl::RF64<false>>(n, a_dev, out_dev, st);
    else
        s = ryser_float<pl::RC128<false>>(n, a_dev, out_dev, st);
    int32_t status_host = 0;
    if (s == PL_OK && !dev_ptrs) {
        const cudaError_t e = cudaMemcpyAsync(out, out_dev, es, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(out)");
    }
    if (s == PL_OK) {
        const cudaError_t e = cudaMemcpyAsync(&status_host, status_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(status)");
    }
    if (!dev_ptrs) {
        cudaFreeAsync(a_dev, st);
        cudaFreeAsync(out_dev, st);
    }
    cudaFreeAsync(status_dev, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (s == PL_OK && e != cudaSuccess) s = plc::cuda_error(e, "cudaStreamSynchronize");
    if (s == PL_OK && (status_host & PL_STATUS_BIT_OVERFLOW))
        s = plc::fail_msg(PL_ERR_OVERFLOW, "int64 overflow: the permanent is not provably inside the exact int64 ring");
    return s;
}

}  // extern "C"
