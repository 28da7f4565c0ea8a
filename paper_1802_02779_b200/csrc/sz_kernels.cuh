// Store-zechin device kernels (sm_100a).
//
// The reference evaluates per(S) for column subsets S by a memoised recursion
// (reference proj/src/permanent.cpp:140-218):
//     per(S) = sum_{j in S, ascending} a(|S|-1, j) * per(S \ {j})       (:164-175)
//     per({j1<j2}) = a(0,j1) a(1,j2) + a(0,j2) a(1,j1)                    (:158-162)
//     per(A) = sum_{j=0..n-1} a(n-1, j) * per(full \ {j}), left to right  (:184-198)
// The device engine evaluates the same recurrence bottom-up, one layer
// (subset size k) at a time, every layer stored densely in colex order:
//     rank(S) = sum_{i=1..k} C(s_i, i),  s_1 < ... < s_k,
// so a layer is a flat array of C(n,k) entries with no hashing, no memo
// probes and no pointer chasing. Removing s_i gives the predecessor rank
//     rank(S \ {s_i}) = P_i + Q_i,  P_i = sum_{l<i} C(s_l, l),  Q_i = sum_{l>i} C(s_l, l-1),
// which the kernels update incrementally as i ascends (two table lookups per
// term), visiting the terms in the reference's ascending-j order.
//
// Kernels here:
//   (n <= 5: sz_batch_tma_kernel / sz_batch_pipe_kernel in sz_batch.cuh, one
//                         thread per matrix with the whole DP in registers,
//                         batches staged by TMA.)
//   sz_batch_warp_kernel  6 <= n <= 9, 8-byte rings: one warp per matrix.
//   sz_batch_smem_kernel  otherwise up to n = 14: one CTA per matrix, ping-pong
//                         layers and the matrix in shared memory, predecessor
//                         offsets from a host-built table shared by the batch.
//   sz_base_layer_kernel  layer 2 (order-2 base case) of a single large matrix;
//                         layers >= 3 run in the warp-specialised kernel (sz_ws.cuh).
//   sz_top_kernel         the final n-term development.
#pragma once

#include <cstdint>

#include "ring.cuh"

namespace pl {

struct DevStatus {
    int32_t* status;       // OR-ed PL_STATUS_BIT_* bits (device)
};

// Shared-memory binomial table, row-major [s][l], kBinomDim x kBinomDim.
__device__ __forceinline__ void load_binom_smem(uint32_t* sb) {
    for (int e = threadIdx.x; e < kBinomDim * kBinomDim; e += blockDim.x) {
        const int s = e / kBinomDim, l = e % kBinomDim;
        uint32_t v = 0;
        if (l <= s) {
            uint64_t r = 1;
            for (int i = 1; i <= l; ++i) r = r * (uint64_t)(s - l + i) / (uint64_t)i;
            v = (uint32_t)r;
        }
        sb[e] = v;
    }
}

// Colex unrank of `r` among k-subsets of {0..n-1}: returns the bitmask and
// qsum = sum_{l=2..k} C(s_l, l-1) (= Q_1, the suffix part of the first
// predecessor rank).
__device__ __forceinline__ uint64_t colex_unrank(uint32_t r, int k, int n, const uint32_t* sb, uint32_t& qsum) {
    uint64_t mask = 0;
    uint32_t q = 0;
    int s = n - 1;
    for (int i = k; i >= 1; --i) {
        uint32_t c = sb[s * kBinomDim + i];
        while (c > r) {
            --s;
            c = sb[s * kBinomDim + i];
        }
        mask |= 1ull << s;
        r -= c;
        if (i >= 2) q += sb[s * kBinomDim + i - 1];
        --s;
    }
    qsum = q;
    return mask;
}

// One output of layer k >= 3: sum over the k elements of `mask` ascending of
// row[s] * prev[rank(mask \ {s})].
template <class R>
__device__ __forceinline__ typename R::T eval_subset(uint64_t mask, uint32_t qsum, int k,
                                                     const typename R::T* row,
                                                     const typename R::T* prev, const uint32_t* sb,
                                                     bool& ov) {
    using T = typename R::T;
    uint32_t P = 0, Q = qsum;
    int s = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    T acc = R::mul(row[s], prev[P + Q], ov);
    P += sb[s * kBinomDim + 1];
    for (int i = 2; i <= k; ++i) {
        const int s2 = __ffsll((long long)mask) - 1;
        mask &= mask - 1;
        Q -= sb[s2 * kBinomDim + i - 1];
        acc = R::mac(acc, row[s2], prev[P + Q], ov);
        P += sb[s2 * kBinomDim + i];
    }
    return acc;
}

// Order-2 base case for the subset {j1 < j2}: a(0,j1) a(1,j2) + a(0,j2) a(1,j1).
template <class R>
__device__ __forceinline__ typename R::T base_pair(const typename R::T* a, int n, int j1, int j2, bool& ov) {
    return R::add(R::mul(a[j1], a[n + j2], ov), R::mul(a[j2], a[n + j1], ov), ov);
}

// ---------------------------------------------------------------- n <= 6

// Iterative (inlinable) bit helpers: with the mask loops fully unrolled they
// fold to constants, so every memo index and matrix index is static and the
// whole DP stays in registers.
__host__ __device__ __forceinline__ constexpr int popc_c(int x) {
    int c = 0;
    for (int i = 0; i < 16; ++i) c += (x >> i) & 1;
    return c;
}
__host__ __device__ __forceinline__ constexpr int ctz_c(int x) {
    for (int i = 0; i < 16; ++i)
        if ((x >> i) & 1) return i;
    return 16;
}
__host__ __device__ __forceinline__ constexpr int msb_c(int x) {
    int r = 0;
    for (int i = 0; i < 16; ++i)
        if ((x >> i) & 1) r = i;
    return r;
}

template <class R, int N>
__device__ __forceinline__ typename R::T perm_in_registers(const typename R::T* a, bool& ov) {
    using T = typename R::T;
    if constexpr (N == 1) {
        return a[0];
    } else {
        T memo[1 << N];
#pragma unroll
        for (int m = 0; m < (1 << N); ++m) {
            if (popc_c(m) == 2) {
                const int j1 = ctz_c(m);
                const int j2 = msb_c(m);
                memo[m] = base_pair<R>(a, N, j1, j2, ov);
            }
        }
        if constexpr (N == 2) {
            return memo[3];
        } else {
#pragma unroll
            for (int k = 3; k < N; ++k) {
#pragma unroll
                for (int m = 0; m < (1 << N); ++m) {
                    if (popc_c(m) == k) {
                        T acc = R::zero();
                        bool first = true;
#pragma unroll
                        for (int j = 0; j < N; ++j) {
                            if ((m >> j) & 1) {
                                const T c = a[(k - 1) * N + j];
                                const T v = memo[m & ~(1 << j)];
                                acc = first ? R::mul(c, v, ov) : R::mac(acc, c, v, ov);
                                first = false;
                            }
                        }
                        memo[m] = acc;
                    }
                }
            }
            constexpr int full = (1 << N) - 1;
            T total = R::mul(a[(N - 1) * N], memo[full & ~1], ov);
#pragma unroll
            for (int j = 1; j < N; ++j) total = R::mac(total, a[(N - 1) * N + j], memo[full & ~(1 << j)], ov);
            return total;
        }
    }
}

// Guard for the exact int64 ring: true when prod_i max(1, sum_j |a_ij|) < 2^63,
// which bounds |per| of every sub-permanent over leading rows and every
// partial sum of the development (|per(S)| <= prod_{i<|S|} sum_{j in S} |a_ij|).
__device__ __forceinline__ bool i64_guard_ok(const long long* a, int n, int stride_row = -1) {
    if (stride_row < 0) stride_row = n;
    unsigned long long prod = 1;
    bool ok = true;
    for (int i = 0; i < n; ++i) {
        unsigned long long rs = 0;
        for (int j = 0; j < n; ++j) {
            const long long v = a[i * stride_row + j];
            if (v == (long long)0x8000000000000000ULL) ok = false;
            const unsigned long long m = v < 0 ? (unsigned long long)(-v) : (unsigned long long)v;
            const unsigned long long t = rs + m;
            if (t < rs) ok = false;
            rs = t;
        }
        if (rs == 0) rs = 1;
        if (__umul64hi(prod, rs) != 0) ok = false;
        prod *= rs;
        if (prod >= 0x8000000000000000ULL) ok = false;
    }
    return ok;
}

__device__ __forceinline__ unsigned smem_addr_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Batched kernel for n <= 5: one thread per matrix, the whole DP in
// registers. Each thread loads its own n*n entries with 16-byte vector loads
// issued back to back (the sectors its neighbours need arrive in the same L1
// lines), so a resident CTA keeps its whole chunk in flight with no shared-
// memory staging or barrier; four CTAs per SM overlap loads and arithmetic.
template <class T, int E>
struct MatRegs {
    T v[E];
};

template <class T, int E>
__device__ __forceinline__ void load_matrix(const T* __restrict__ p, MatRegs<T, E>& m) {
    if constexpr (sizeof(T) == 16) {
#pragma unroll
        for (int e = 0; e < E; ++e) m.v[e] = __ldg(reinterpret_cast<const double2*>(p) + e);
    } else {
        if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {  // pairs of entries per 16-byte load
#pragma unroll
            for (int e = 0; e + 1 < E; e += 2) {
                const longlong2 w = __ldg(reinterpret_cast<const longlong2*>(p + e));
                m.v[e] = *reinterpret_cast<const T*>(&w.x);
                m.v[e + 1] = *reinterpret_cast<const T*>(&w.y);
            }
            if (E % 2) m.v[E - 1] = __ldg(p + E - 1);
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) m.v[e] = __ldg(p + e);
        }
    }
}

// Compile-time-indexed form of i64_guard_ok (keeps the matrix in registers).
template <int N>
__device__ __forceinline__ bool i64_guard_ok_n(const long long* a) {
    unsigned long long prod = 1;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        unsigned long long rs = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const long long v = a[i * N + j];
            ok &= v != (long long)0x8000000000000000ULL;
            const unsigned long long mg = v < 0 ? (unsigned long long)(-v) : (unsigned long long)v;
            const unsigned long long t = rs + mg;
            ok &= t >= rs;
            rs = t;
        }
        rs = rs == 0 ? 1 : rs;
        ok &= __umul64hi(prod, rs) == 0;
        prod *= rs;
        ok &= prod < 0x8000000000000000ULL;
    }
    return ok;
}

template <int N>
__device__ __forceinline__ bool i64_fits_f64_n(const long long* a) {
    double prod = 1.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double rs = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const long long v = a[i * N + j];
            rs += v < 0 ? -(double)v : (double)v;
        }
        prod *= rs < 1.0 ? 1.0 : rs;
    }
    return prod < 9007199254740992.0;
}

// ---------------------------------------------------------------- 6 <= n <= 14

// Guard bound for the exact-in-double shortcut: every sub-permanent and partial
// sum of an integer matrix is bounded by prod_i max(1, sum_j |a_ij|); below 2^53
// all of them are integers representable in a double and an FMA of exact
// integers is exact, so the FP64 pipe reproduces int64 arithmetic bit for bit.
__device__ __forceinline__ bool i64_fits_f64(const long long* a, int n) {
    double prod = 1.0;
    for (int i = 0; i < n; ++i) {
        double rs = 0.0;
        for (int j = 0; j < n; ++j) {
            const long long v = a[i * n + j];
            rs += v < 0 ? -(double)v : (double)v;  // |entries| < 2^53 below, so this is exact or already over
        }
        prod *= rs < 1.0 ? 1.0 : rs;
    }
    return prod < 9007199254740992.0;  // 2^53 (double rounding only ever overestimates here)
}

// The layer DP of one matrix held in shared memory (see sz_batch_smem_kernel).
// N > 0: the order is a compile-time constant (layer and term loops unroll).
// WARP: the DP of one matrix by one warp (lane-strided outputs, __syncwarp
// between layers) instead of the whole CTA.
// ptab32 (layers >= 3) holds the same entries as byte offsets for this
// element size: (rank(S \ {s_i}) * sizeof(TT)) | (s_i * sizeof(TT)) << 16, so a
// term is one table load and two shared loads at (base + offset).
template <class RR, class TT, int N = 0, bool WARP = false>
__device__ __forceinline__ const TT* smem_dp(const TT* mat, TT* buf0, TT* buf1, int n_rt,
                                             const uint16_t* __restrict__ ptab, const uint32_t* __restrict__ poff,
                                             const uint32_t* __restrict__ ptab32, bool& ov) {
    const int n = N > 0 ? N : n_rt;
    const int tid = WARP ? (int)(threadIdx.x & 31) : (int)threadIdx.x, nt = WARP ? 32 : (int)blockDim.x;
    auto sync = [] {
        if (WARP) __syncwarp();
        else __syncthreads();
    };
    const uint32_t c2 = poff[3] - poff[2];
    for (uint32_t r = tid; r < c2; r += nt) {
        const uint32_t e = __ldg(ptab + poff[2] + r);
        buf0[r] = base_pair<RR>(mat, n, (int)(e & 0xffu), (int)(e >> 8), ov);
    }
    sync();
    TT* prev = buf0;
    TT* cur = buf1;
#pragma unroll
    for (int k = 3; k < n; ++k) {
        const uint32_t ck = N > 0 ? (uint32_t)binom_u64(N, k) : (poff[k + 1] - poff[k]) / (uint32_t)k;
        const uint32_t* pt = ptab32 + poff[k];
        const char* row = reinterpret_cast<const char*>(mat + (k - 1) * n);
        const char* pv = reinterpret_cast<const char*>(prev);
        auto rowv = [&](uint32_t e) { return *reinterpret_cast<const TT*>(row + (e >> 16)); };
        auto prevv = [&](uint32_t e) { return *reinterpret_cast<const TT*>(pv + (e & 0xffffu)); };
        for (uint32_t r = tid; r < ck; r += nt) {
            uint32_t e = __ldg(pt + r);
            TT acc = RR::mul(rowv(e), prevv(e), ov);
            int i = 1;
            for (; i + 4 <= k; i += 4) {
                const uint32_t e0 = __ldg(pt + (i + 0) * ck + r), e1 = __ldg(pt + (i + 1) * ck + r);
                const uint32_t e2 = __ldg(pt + (i + 2) * ck + r), e3 = __ldg(pt + (i + 3) * ck + r);
                acc = RR::mac(acc, rowv(e0), prevv(e0), ov);
                acc = RR::mac(acc, rowv(e1), prevv(e1), ov);
                acc = RR::mac(acc, rowv(e2), prevv(e2), ov);
                acc = RR::mac(acc, rowv(e3), prevv(e3), ov);
            }
            for (; i < k; ++i) {
                e = __ldg(pt + i * ck + r);
                acc = RR::mac(acc, rowv(e), prevv(e), ov);
            }
            cur[r] = acc;
        }
        sync();
        TT* t = prev;
        prev = cur;
        cur = t;
    }
    return prev;
}

template <class RR, class TT, int N = 0>
__device__ __forceinline__ TT smem_top(const TT* mat, const TT* last_layer, int n_rt, bool& ov) {
    const int n = N > 0 ? N : n_rt;
    const TT* last = mat + (n - 1) * n;
    TT total = RR::mul(last[0], last_layer[n - 1], ov);
#pragma unroll
    for (int j = 1; j < n; ++j) total = RR::mac(total, last[j], last_layer[n - 1 - j], ov);
    return total;
}

// Exact-path choice for one int64 matrix, computed by a whole warp (lane i
// sums row i): 0 = exact in doubles (guard bound < 2^53, i64_fits_f64),
// 1 = wrapping int64 (bound < 2^63, i64_guard_ok), 2 = checked int64.
template <int N>
__device__ __forceinline__ int warp_i64_mode(const long long* m) {
    const int lane = threadIdx.x & 31;
    unsigned long long rs = 0;
    double rd = 0.0;
    bool ok = true;
    if (lane < N) {
        const long long* row = m + lane * N;
        for (int j = 0; j < N; ++j) {
            const long long v = row[j];
            ok &= v != (long long)0x8000000000000000ULL;
            const unsigned long long mg = v < 0 ? (unsigned long long)(-v) : (unsigned long long)v;
            const unsigned long long t = rs + mg;
            ok &= t >= rs;
            rs = t;
            rd += v < 0 ? -(double)v : (double)v;
        }
    }
    unsigned long long prod = 1;
    double pd = 1.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        unsigned long long r = __shfl_sync(0xffffffffu, rs, i);
        const double d = __shfl_sync(0xffffffffu, rd, i);
        r = r == 0 ? 1 : r;
        ok &= __umul64hi(prod, r) == 0;
        prod *= r;
        ok &= prod < 0x8000000000000000ULL;
        pd *= d < 1.0 ? 1.0 : d;
    }
    ok = __all_sync(0xffffffffu, ok);
    return pd < 9007199254740992.0 ? 0 : (ok ? 1 : 2);
}

// One CTA per matrix at a time (persistent CTAs striding over the batch);
// the matrix and two layer buffers live in the CTA's shared memory (16 KB at
// n = 12, so ~14 CTAs share an SM). The predecessor structure is the same for
// every matrix of order n, so it is read from a table built once on the host
// (L1-resident, coalesced):
//   layer 2:  ptab[off[2] + r]           = j1 | j2 << 8       (r = j1 + C(j2, 2))
//   layer k:  ptab[off[k] + i*C(n,k) + r] = rank(S \ {s_i}) | s_i << 12
// with s_i the i-th element of the r-th k-subset in colex order, ascending.
// Integer matrices take one of three exact paths per matrix: doubles with FMA
// when the guard bound is below 2^53, wrapping int64 below 2^63, checked int64
// otherwise.
#ifndef PL_SMEM_THREADS
#define PL_SMEM_THREADS 128
#endif
constexpr int kSmemThreads = PL_SMEM_THREADS;  // threads per matrix (CTA) of the shared-memory kernel

template <class R, int N>
__global__ void __launch_bounds__(kSmemThreads) sz_batch_smem_kernel(const typename R::T* __restrict__ a,
                                                            typename R::T* __restrict__ out, int64_t count,
                                                            int n_rt, int maxc, const uint16_t* __restrict__ ptab,
                                                            const uint32_t* __restrict__ poff,
                                                            const uint32_t* __restrict__ ptab32,
                                                            int32_t* __restrict__ status, int early_loads) {
    using T = typename R::T;
    constexpr int n = N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int flag, mode;
    T* mat = reinterpret_cast<T*>(smem_raw);
    T* buf0 = mat + ((n * n + 1) & ~1);
    T* buf1 = buf0 + ((maxc + 1) & ~1);
    const int tid = threadIdx.x, nt = blockDim.x;
    // programmatic dependent launch, as in sz_batch_f32_pack_kernel (no-ops under a plain launch)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (!early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");

    for (int64_t b = blockIdx.x; b < count; b += gridDim.x) {
        const T* g = a + b * n * n;
        for (int e = tid; e < n * n; e += nt) mat[e] = g[e];
        if (tid == 0) flag = 0;
        __syncthreads();
        bool ov = false;
        T total = R::zero();
        if constexpr (R::kChecked) {
            if (tid < 32) {
                const int md = warp_i64_mode<N>(reinterpret_cast<const long long*>(mat));
                if (tid == 0) mode = md;
            }
            __syncthreads();
            if (mode == 0) {
                double* dm = reinterpret_cast<double*>(mat);
                for (int e = tid; e < n * n; e += nt) dm[e] = (double)mat[e];
                __syncthreads();
                const double* last = smem_dp<RF64<true>, double, N>(dm, reinterpret_cast<double*>(buf0),
                                                         reinterpret_cast<double*>(buf1), n, ptab, poff, ptab32, ov);
                if (tid == 0) total = (T)smem_top<RF64<true>, double, N>(dm, last, n, ov);
            } else if (mode == 1) {
                const T* last = smem_dp<RI64<false>, T, N>(mat, buf0, buf1, n, ptab, poff, ptab32, ov);
                if (tid == 0) total = smem_top<RI64<false>, T, N>(mat, last, n, ov);
            } else {
                const T* last = smem_dp<R, T, N>(mat, buf0, buf1, n, ptab, poff, ptab32, ov);
                if (ov) atomicOr(&flag, 1);
                __syncthreads();
                if (tid == 0 && !(flag & 1)) total = smem_top<R, T, N>(mat, last, n, ov);
            }
        } else {
            const T* last = smem_dp<R, T, N>(mat, buf0, buf1, n, ptab, poff, ptab32, ov);
            if (tid == 0) total = smem_top<R, T, N>(mat, last, n, ov);
        }
        if (tid == 0) {
            if (early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // before this grid's stores
            if ((flag & 1) || ov) {
                atomicOr(status, 1);
                total = R::zero();
            }
            out[b] = total;
        }
        __syncthreads();
    }
}

// Exact integer arithmetic on the FP32 pipe: every operand, product and
// partial sum of a matrix whose bound (below) is under 2^24 is an integer
// that a float holds exactly, so each rounded operation is exact.
struct RF32X {
    using T = float;
    static constexpr bool kChecked = false;
    __device__ __forceinline__ static T mul(T a, T b, bool&) { return __fmul_rn(a, b); }
    __device__ __forceinline__ static T add(T a, T b, bool&) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static T mac(T acc, T a, T b, bool&) { return __fmaf_rn(a, b, acc); }
    __device__ __forceinline__ static T zero() { return 0.0f; }
};

// int64 exact-path choice including the FP32 path: 3 when every sub-permanent
// and partial sum is provably below 2^24 -- by the row-sum bound
// prod_i max(1, sum_j |a_ij|), or for 0/1 matrices by Bregman's bound
// prod_i (r_i!)^(1/r_i) (r_i the row sums; sub-matrices of a 0/1 matrix are
// 0/1 with smaller row sums and (r!)^(1/r) grows with r, and with
// nonnegative entries every partial sum is at most its sub-permanent) --
// else the warp_i64_mode choice.
template <int N>
__device__ __forceinline__ int warp_i64_mode_f32(const long long* m) {
    const int lane = threadIdx.x & 31;
    bool zero_one = true;
    double rd = 0.0, lg = 0.0;
    if (lane < N) {
        const long long* row = m + lane * N;
        long long r01 = 0;
        for (int j = 0; j < N; ++j) {
            const long long v = row[j];
            zero_one &= v == 0 || v == 1;
            r01 += v;
            rd += v < 0 ? -(double)v : (double)v;
        }
        if (zero_one && r01 > 0) lg = lgamma((double)r01 + 1.0) / (double)r01;  // log (r!)^(1/r)
    }
    zero_one = __all_sync(0xffffffffu, zero_one);
    double pd = 1.0, lsum = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double d = __shfl_sync(0xffffffffu, rd, i);
        pd *= d < 1.0 ? 1.0 : d;
        lsum += __shfl_sync(0xffffffffu, lg, i);
    }
    const double kLim = 16777216.0 * (1.0 - 1e-9);  // 2^24, margin for the bound's own rounding
    if (pd < kLim || (zero_one && exp(lsum) < kLim)) return 3;
    return warp_i64_mode<N>(m);
}

// P matrices evaluated in lockstep (8-byte rings): every value is a pack
// {matrix 0, ..., matrix P-1} of P * 8 bytes, so each term is one table load,
// two P * 8-byte shared loads and P products -- the predecessor table and the
// barriers are shared by the pack. Operations apply to every member in the same
// order, so each member is bitwise what the single-matrix DP computes.
template <class RR, int P>
struct PackRing {
    struct __align__(sizeof(typename RR::T) * P) T {
        typename RR::T v[P];
    };
    static constexpr bool kChecked = RR::kChecked;
    __device__ __forceinline__ static T mul(T x, T y, bool& ov) {
        T r;
#pragma unroll
        for (int i = 0; i < P; ++i) r.v[i] = RR::mul(x.v[i], y.v[i], ov);
        return r;
    }
    __device__ __forceinline__ static T add(T x, T y, bool& ov) {
        T r;
#pragma unroll
        for (int i = 0; i < P; ++i) r.v[i] = RR::add(x.v[i], y.v[i], ov);
        return r;
    }
    __device__ __forceinline__ static T mac(T acc, T x, T y, bool& ov) {
        T r;
#pragma unroll
        for (int i = 0; i < P; ++i) r.v[i] = RR::mac(acc.v[i], x.v[i], y.v[i], ov);
        return r;
    }
    __device__ __forceinline__ static T zero() {
        T r;
#pragma unroll
        for (int i = 0; i < P; ++i) r.v[i] = RR::zero();
        return r;
    }
};

// The ring a pack runs in: the ring itself for doubles, exact doubles (FMA) for
// int64 matrices whose guard bound is below 2^53.
template <class R>
struct PackBase {
    using type = R;
};
template <>
struct PackBase<RI64<true>> {
    using type = RF64<true>;
};

// CTA per pack of P matrices (8-byte rings, 10 <= n <= 14): the pack DP when every
// member takes the same exact path, else each matrix on its own (contiguous
// layout in the same shared memory). ptab32p: byte offsets for 8 * P-byte packs.
// threads per pack CTA: 256 from n = 12 on (C3 182 -> 177 us), 128 below (n = 10 f64
// is ~3 % faster with 128)
template <int N>
__host__ __device__ constexpr int pack_threads() {
    return N >= 12 ? 256 : 128;
}

template <class R, int N, int P>
__global__ void __launch_bounds__(pack_threads<N>()) sz_batch_smem_pack_kernel(
    const typename R::T* __restrict__ a, typename R::T* __restrict__ out, int64_t count, int maxc,
    const uint16_t* __restrict__ ptab, const uint32_t* __restrict__ poff, const uint32_t* __restrict__ ptab32_8,
    const uint32_t* __restrict__ ptab32p, int32_t* __restrict__ status) {
    using T = typename R::T;
    static_assert(sizeof(T) == 8, "8-byte rings only");
    static_assert(pack_threads<N>() / 32 >= P, "one warp per member for the guards");
    constexpr int n = N, E = N * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int mode[P], flag;
    const int tid = threadIdx.x;
    const int64_t npacks = (count + P - 1) / P;
    for (int64_t pb = blockIdx.x; pb < npacks; pb += gridDim.x) {
        const int64_t b0 = P * pb;
        const int have = count - b0 < P ? (int)(count - b0) : P;
        const T* g = a + b0 * E;
        if (tid == 0) flag = 0;
        if constexpr (R::kChecked) {
            const int w = tid >> 5;
            if (w < have) {
                const int md = warp_i64_mode<N>(reinterpret_cast<const long long*>(g + (size_t)w * E));
                if ((tid & 31) == 0) mode[w] = md;
            }
        }
        __syncthreads();
        bool joint = have == P;
        int m0 = 0;
        if constexpr (R::kChecked) {
            m0 = mode[0];
#pragma unroll
            for (int i = 1; i < P; ++i) joint &= mode[i] == m0;
            joint &= m0 < 2;
        }
        if (joint) {
            // interleaved packs: mat[e] = {M0[e], ..., M(P-1)[e]}; layers likewise
            auto run = [&](auto ring_tag, auto conv) {
                using PR = decltype(ring_tag);
                using PT = typename PR::T;
                PT* mat = reinterpret_cast<PT*>(smem_raw);
                PT* buf0 = mat + E;
                PT* buf1 = buf0 + maxc;
                for (int e = tid; e < E; e += blockDim.x) {
                    PT x;
#pragma unroll
                    for (int i = 0; i < P; ++i) x.v[i] = conv(g[(size_t)i * E + e]);
                    mat[e] = x;
                }
                __syncthreads();
                bool ov = false;
                const PT* last = smem_dp<PR, PT, N>(mat, buf0, buf1, n, ptab, poff, ptab32p, ov);
                if (tid == 0) {
                    const PT t = smem_top<PR, PT, N>(mat, last, n, ov);
#pragma unroll
                    for (int i = 0; i < P; ++i) out[b0 + i] = (T)t.v[i];  // exact for the int64 ring
                }
            };
            if (!R::kChecked || m0 == 0) {
                run(PackRing<typename PackBase<R>::type, P>{}, [](T v) { return (double)v; });
            } else if constexpr (R::kChecked) {
                run(PackRing<RI64<false>, P>{}, [](T v) { return (long long)v; });
            }
        } else {
            // one matrix at a time, contiguous layout (the single-matrix kernel's path)
            for (int h = 0; h < have; ++h) {
                const T* gh = g + (size_t)h * E;
                T* mat = reinterpret_cast<T*>(smem_raw);
                T* buf0 = mat + ((E + 1) & ~1);
                T* buf1 = buf0 + ((maxc + 1) & ~1);
                for (int e = tid; e < E; e += blockDim.x) mat[e] = gh[e];
                if (tid == 0) flag = 0;
                __syncthreads();
                bool ov = false;
                T total = R::zero();
                const int md = R::kChecked ? mode[h] : 2;
                if constexpr (R::kChecked) {
                    if (md == 0) {
                        double* dm = reinterpret_cast<double*>(mat);
                        for (int e = tid; e < E; e += blockDim.x)
                            dm[e] = (double)reinterpret_cast<const long long*>(mat)[e];
                        __syncthreads();
                        const double* last = smem_dp<RF64<true>, double, N>(
                            dm, reinterpret_cast<double*>(buf0), reinterpret_cast<double*>(buf1), n, ptab, poff,
                            ptab32_8, ov);
                        if (tid == 0) total = (T)smem_top<RF64<true>, double, N>(dm, last, n, ov);
                    } else if (md == 1) {
                        const T* last = smem_dp<RI64<false>, T, N>(mat, buf0, buf1, n, ptab, poff, ptab32_8, ov);
                        if (tid == 0) total = smem_top<RI64<false>, T, N>(mat, last, n, ov);
                    }
                }
                if (md == 2) {
                    const T* last = smem_dp<R, T, N>(mat, buf0, buf1, n, ptab, poff, ptab32_8, ov);
                    if (ov) atomicOr(&flag, 1);
                    __syncthreads();
                    if (tid == 0 && !(flag & 1)) total = smem_top<R, T, N>(mat, last, n, ov);
                }
                if (tid == 0) {
                    if ((flag & 1) || ov) {
                        atomicOr(status, 1);
                        total = R::zero();
                    }
                    out[b0 + h] = total;
                }
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

// Members of a pack that is not jointly FP32-exact: one matrix at a time on the
// exact-double / int64 / checked-int64 paths (mode[h] from warp_i64_mode_f32).
template <int N>
__device__ __forceinline__ void f32_pack_members(const long long* g, int have, const int* mode, int& flag,
                                                 unsigned char* smem_raw, int maxc, const uint16_t* __restrict__ ptab,
                                                 const uint32_t* __restrict__ poff,
                                                 const uint32_t* __restrict__ ptab32_8, long long* __restrict__ out,
                                                 int64_t b0, int32_t* __restrict__ status) {
    constexpr int n = N, E = N * N;
    const int tid = threadIdx.x;
    for (int h = 0; h < have; ++h) {
        const long long* gh = g + (size_t)h * E;
        long long* mat = reinterpret_cast<long long*>(smem_raw);
        long long* buf0 = mat + ((E + 1) & ~1);
        long long* buf1 = buf0 + ((maxc + 1) & ~1);
        for (int e = tid; e < E; e += blockDim.x) mat[e] = gh[e];
        if (tid == 0) flag = 0;
        __syncthreads();
        bool ov = false;
        long long total = 0;
        const int md = mode[h];
        if (md == 0 || md == 3) {
            double* dm = reinterpret_cast<double*>(mat);
            for (int e = tid; e < E; e += blockDim.x) dm[e] = (double)mat[e];
            __syncthreads();
            const double* last = smem_dp<RF64<true>, double, N>(dm, reinterpret_cast<double*>(buf0),
                                                                 reinterpret_cast<double*>(buf1), n, ptab,
                                                                 poff, ptab32_8, ov);
            if (tid == 0) total = (long long)smem_top<RF64<true>, double, N>(dm, last, n, ov);
        } else if (md == 1) {
            const long long* last = smem_dp<RI64<false>, long long, N>(mat, buf0, buf1, n, ptab, poff,
                                                                       ptab32_8, ov);
            if (tid == 0) total = smem_top<RI64<false>, long long, N>(mat, last, n, ov);
        } else {
            const long long* last = smem_dp<RI64<true>, long long, N>(mat, buf0, buf1, n, ptab, poff,
                                                                      ptab32_8, ov);
            if (ov) atomicOr(&flag, 1);
            __syncthreads();
            if (tid == 0 && !(flag & 1)) total = smem_top<RI64<true>, long long, N>(mat, last, n, ov);
        }
        if (tid == 0) {
            if ((flag & 1) || ov) {
                atomicOr(status, 1);
                total = 0;
            }
            out[b0 + h] = total;
        }
        __syncthreads();
    }
}

// The layer DP of a jointly FP32-exact four-matrix pack whose entries all fit a
// signed byte (C3's 0/1 matrices and most small-integer batches): the
// coefficient pack a(k-1, col) is read as ONE 32-bit word of four biased bytes
// (mat8) instead of a gathered 16-byte load, and expanded exactly: the byte
// placed in the mantissa of 2^23 gives the float 2^23 + b, minus 2^23 + 128.
// A 16-byte shared load costs four cycles of the L1TEX data pipe whatever its
// address pattern, a 4-byte one one cycle; the pack kernel is bound by that
// pipe (89 % busy, profiles/r2/full_c3.md), not by issue slots.
__device__ __forceinline__ void f32_coef4(uint32_t w, float (&c)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u + i)) - 8388736.0f;
}

// tab2 / off2: the predecessor entries (rank | column << 12) two terms per
// 32-bit word (batch.cu, Ptab::tab2), so a pair of terms costs one table load.
template <int N, class PT>
__device__ __forceinline__ const PT* smem_dp_f32c(const PT* mat, const uint32_t* __restrict__ mat8, PT* buf0, PT* buf1,
                                                  const uint16_t* __restrict__ ptab,
                                                  const uint32_t* __restrict__ poff,
                                                  const uint32_t* __restrict__ tab2,
                                                  const uint32_t* __restrict__ off2) {
    using PR = PackRing<RF32X, 4>;
    const int tid = (int)threadIdx.x, nt = (int)blockDim.x;
    bool ov = false;
    const uint32_t c2 = poff[3] - poff[2];
    for (uint32_t r = tid; r < c2; r += nt) {
        const uint32_t e = __ldg(ptab + poff[2] + r);
        buf0[r] = base_pair<PR>(mat, N, (int)(e & 0xffu), (int)(e >> 8), ov);
    }
    __syncthreads();
    PT* prev = buf0;
    PT* cur = buf1;
#pragma unroll
    for (int k = 3; k < N; ++k) {
        const uint32_t ck = (uint32_t)binom_u64(N, k);
        const uint32_t* pt = tab2 + off2[k];
        const uint32_t* row8 = mat8 + (k - 1) * N;
        auto term = [&](PT& acc, uint32_t e, bool first) {  // e = rank | column << 12 (16 bits)
            float c[4];
            f32_coef4(row8[(e >> 12) & 0xfu], c);
            const PT x = prev[e & 0xfffu];
#pragma unroll
            for (int i = 0; i < 4; ++i) acc.v[i] = first ? __fmul_rn(c[i], x.v[i]) : __fmaf_rn(c[i], x.v[i], acc.v[i]);
        };
        for (uint32_t r = tid; r < ck; r += nt) {
            PT acc;
            uint32_t w[(N + 1) / 2];
#pragma unroll
            for (int p = 0; p < (k + 1) / 2; ++p) w[p] = __ldg(pt + p * ck + r);
#pragma unroll
            for (int i = 0; i < k; ++i) term(acc, (i & 1) ? w[i / 2] >> 16 : w[i / 2] & 0xffffu, i == 0);
            cur[r] = acc;
        }
        __syncthreads();
        PT* t = prev;
        prev = cur;
        cur = t;
    }
    return prev;
}

// int64 batches, 10 <= n <= 14: four matrices per CTA in lockstep on the FP32
// pipe when all four are FP32-exact (warp_i64_mode_f32 == 3): a pack is 16
// bytes (the same byte offsets as a pair of doubles), so a term is one table
// load, two 16-byte shared loads and four FFMAs, and twice the matrices of the
// double pack share an SM. Other packs run their members one at a time on the
// double / int64 exact paths (as sz_batch_smem_pack_kernel's fallback).
#ifndef PL_F32_THREADS
#define PL_F32_THREADS 256
#endif
constexpr int kF32Threads = PL_F32_THREADS;  // threads per four-matrix pack CTA
#ifndef PL_F32_BYTE_COEF
#define PL_F32_BYTE_COEF 1
#endif
constexpr bool kF32ByteCoef = PL_F32_BYTE_COEF;  // byte-packed coefficients when every entry fits (smem_dp_f32c)

template <int N, int P>
__global__ void __launch_bounds__(kF32Threads) sz_batch_f32_pack_kernel(
    const long long* __restrict__ a, long long* __restrict__ out, int64_t count, int maxc,
    const uint16_t* __restrict__ ptab, const uint32_t* __restrict__ poff, const uint32_t* __restrict__ ptab32_8,
    const uint32_t* __restrict__ ptab32_16, const uint32_t* __restrict__ tab2, const uint32_t* __restrict__ off2,
    int32_t* __restrict__ status, int early_loads) {
    constexpr int n = N, E = N * N;
    using PR = PackRing<RF32X, P>;
    using PT = typename PR::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int mode[P], flag;
    const int tid = threadIdx.x;
    const int64_t npacks = (count + P - 1) / P;
    // programmatic dependent launch (see sz_batch_tma_kernel): the next grid may be scheduled as
    // CTAs of this one exit; nothing is read before the previous grid is done unless the caller
    // marked the input ready (PL_FLAG_INPUT_READY) -- then only the stores wait
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (!early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int64_t pb = blockIdx.x; pb < npacks; pb += gridDim.x) {
        const int64_t b0 = P * pb;
        const int have = count - b0 < P ? (int)(count - b0) : P;
        const long long* g = a + b0 * E;
        for (int w = tid >> 5; w < have; w += (int)(blockDim.x >> 5)) {  // one warp per member's guard
            const int md = warp_i64_mode_f32<N>(g + (size_t)w * E);
            if ((tid & 31) == 0) mode[w] = md;
        }
        __syncthreads();
        bool joint = have == P;
#pragma unroll
        for (int i = 0; i < P; ++i) joint &= i >= have || mode[i] == 3;
        if (joint) {
            PT* mat = reinterpret_cast<PT*>(smem_raw);
            PT* buf0 = mat + E;
            PT* buf1 = buf0 + maxc;
            uint32_t* mat8 = reinterpret_cast<uint32_t*>(buf1 + maxc);  // P = 4: biased-byte coefficient packs
            bool bytes_ok = true;
            for (int e = tid; e < E; e += blockDim.x) {
                PT x;
                uint32_t w = 0;
#pragma unroll
                for (int i = 0; i < P; ++i) {
                    const long long v = g[(size_t)i * E + e];
                    x.v[i] = (float)v;
                    bytes_ok &= v >= -128 && v <= 127;
                    if (i < 4) w |= (uint32_t)((v + 128) & 0xff) << (8 * i);
                }
                mat[e] = x;
                if (P == 4 && kF32ByteCoef) mat8[e] = w;
            }
            bytes_ok = __syncthreads_and(bytes_ok) != 0;
            bool ov = false;
            const PT* last;
            if constexpr (P == 4 && kF32ByteCoef) {
                last = bytes_ok ? smem_dp_f32c<N, PT>(mat, mat8, buf0, buf1, ptab, poff, tab2, off2)
                                : smem_dp<PR, PT, N>(mat, buf0, buf1, n, ptab, poff, ptab32_16, ov);
            } else {
                last = smem_dp<PR, PT, N>(mat, buf0, buf1, n, ptab, poff, ptab32_16, ov);  // 4P-byte offsets
            }
            if (tid == 0) {
                const PT t = smem_top<PR, PT, N>(mat, last, n, ov);
                if (early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // before this grid's stores
#pragma unroll
                for (int i = 0; i < P; ++i) out[b0 + i] = (long long)t.v[i];
            }
        } else {
            if (early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");
            f32_pack_members<N>(g, have, mode, flag, smem_raw, maxc, ptab, poff, ptab32_8, out, b0, status);
        }
        __syncthreads();
    }
}

// Warp-per-matrix variant for 8-byte rings, 6 <= n <= 9 (the matrix and two
// layers of one matrix fit a few KB, so many warps share an SM): no CTA barrier in
// the layer loop, and the int64 exactness guard is computed by the warp (lane
// i sums row i) instead of one thread.
#ifndef PL_WARP_KERNEL_WARPS
#define PL_WARP_KERNEL_WARPS 2
#endif
constexpr int kWarpKernelWarps = PL_WARP_KERNEL_WARPS;  // warps (matrices in flight) per CTA

template <int N>
__host__ __device__ constexpr int warp_kernel_stride() {
    return ((N * N + 1) & ~1) + 2 * (((int)binom_u64(N, N / 2) + 1) & ~1);  // elements per warp
}

template <class R, int N>
__global__ void __launch_bounds__(32 * kWarpKernelWarps) sz_batch_warp_kernel(
    const typename R::T* __restrict__ a, typename R::T* __restrict__ out, int64_t count,
    const uint16_t* __restrict__ ptab, const uint32_t* __restrict__ poff, const uint32_t* __restrict__ ptab32,
    int32_t* __restrict__ status, int early_loads) {
    using T = typename R::T;
    static_assert(sizeof(T) == 8, "8-byte rings only");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // see sz_batch_f32_pack_kernel
    if (!early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    constexpr int E = N * N;
    constexpr int MAXC = (int)binom_u64(N, N / 2);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* mat = reinterpret_cast<T*>(smem_raw) + (size_t)warp * warp_kernel_stride<N>();
    T* buf0 = mat + ((E + 1) & ~1);
    T* buf1 = buf0 + ((MAXC + 1) & ~1);
    bool ov_any = false;
    for (int64_t b = (int64_t)blockIdx.x * kWarpKernelWarps + warp; b < count;
         b += (int64_t)gridDim.x * kWarpKernelWarps) {
        const T* g = a + b * E;
        for (int e = lane; e < E; e += 32) mat[e] = g[e];
        __syncwarp();
        bool ov = false;
        T total = R::zero();
        if constexpr (R::kChecked) {
            const int md = warp_i64_mode<N>(reinterpret_cast<const long long*>(mat));
            if (md == 0) {
                // exact in doubles: convert in place, FMA path
                double* dm = reinterpret_cast<double*>(mat);
                for (int e = lane; e < E; e += 32) dm[e] = (double)reinterpret_cast<const long long*>(mat)[e];
                __syncwarp();
                const double* last = smem_dp<RF64<true>, double, N, true>(dm, reinterpret_cast<double*>(buf0),
                                                                          reinterpret_cast<double*>(buf1), N, ptab,
                                                                          poff, ptab32, ov);
                if (lane == 0) total = (T)smem_top<RF64<true>, double, N>(dm, last, N, ov);
            } else if (md == 1) {
                const T* last = smem_dp<RI64<false>, T, N, true>(mat, buf0, buf1, N, ptab, poff, ptab32, ov);
                if (lane == 0) total = smem_top<RI64<false>, T, N>(mat, last, N, ov);
            } else {
                const T* last = smem_dp<R, T, N, true>(mat, buf0, buf1, N, ptab, poff, ptab32, ov);
                ov = __any_sync(0xffffffffu, ov);
                if (lane == 0 && !ov) total = smem_top<R, T, N>(mat, last, N, ov);
            }
        } else {
            const T* last = smem_dp<R, T, N, true>(mat, buf0, buf1, N, ptab, poff, ptab32, ov);
            if (lane == 0) total = smem_top<R, T, N>(mat, last, N, ov);
        }
        ov = __any_sync(0xffffffffu, ov);
        if (lane == 0) {
            if (early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // before this grid's stores
            if (ov) total = R::zero();
            out[b] = total;
        }
        ov_any |= ov;
        __syncwarp();
    }
    if (ov_any && lane == 0) {
        if (early_loads) asm volatile("griddepcontrol.wait;\n" ::: "memory");
        atomicOr(status, 1);
    }
}

// ---------------------------------------------------------------- layer 2

// Layer 2 (order-2 base case) for ranks [r0, r1): rank({j1 < j2}) = j1 + C(j2, 2).
template <class R>
__global__ void sz_base_layer_kernel(const typename R::T* __restrict__ a, int n, typename R::T* __restrict__ cur,
                                     uint64_t r0, uint64_t r1, int32_t* __restrict__ status) {
    bool ov = false;
    for (uint64_t r = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
         r += (uint64_t)gridDim.x * blockDim.x) {
        int j2 = 1;
        while (binom_u64(j2 + 1, 2) <= r) ++j2;
        const int j1 = (int)(r - binom_u64(j2, 2));
        cur[r] = base_pair<R>(a, n, j1, j2, ov);
    }
    if (ov) atomicOr(status, 1);
}

template <class R>
__global__ void sz_top_kernel(const typename R::T* __restrict__ a, int n, const typename R::T* __restrict__ last,
                              typename R::T* __restrict__ out, const int32_t* __restrict__ guard,
                              int32_t* __restrict__ status) {
    using T = typename R::T;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    bool ov = false;
    const T* row = a + (size_t)(n - 1) * n;
    T total = R::mul(row[0], last[n - 1], ov);
    for (int j = 1; j < n; ++j) total = R::mac(total, row[j], last[n - 1 - j], ov);
    if (ov) {
        atomicOr(status, 1);
        total = R::zero();
    }
    out[0] = total;
}

// Batched forms for a batch of large orders (matrices n x n contiguous, layer
// buffers `stride` elements apart): layer 2, the top level and the int64 guard
// of every matrix in one launch each.
template <class R>
__global__ void sz_base_layer_batch_kernel(const typename R::T* __restrict__ a, int n, typename R::T* __restrict__ cur,
                                           uint64_t stride, uint32_t nmat, int32_t* __restrict__ status) {
    bool ov = false;
    const uint64_t np = binom_u64(n, 2), total = np * nmat;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = t / np, r = t - b * np;
        int j2 = 1;
        while (binom_u64(j2 + 1, 2) <= r) ++j2;
        const int j1 = (int)(r - binom_u64(j2, 2));
        cur[b * stride + r] = base_pair<R>(a + b * (uint64_t)n * n, n, j1, j2, ov);
    }
    if (ov) atomicOr(status, 1);
}

template <class R>
__global__ void sz_top_batch_kernel(const typename R::T* __restrict__ a, int n, const typename R::T* __restrict__ last,
                                    uint64_t stride, typename R::T* __restrict__ out, uint32_t nmat,
                                    int32_t* __restrict__ status) {
    using T = typename R::T;
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nmat) return;
    bool ov = false;
    const T* row = a + ((uint64_t)b * n + (uint64_t)(n - 1)) * n;
    const T* lb = last + (uint64_t)b * stride;
    T total = R::mul(row[0], lb[n - 1], ov);
    for (int j = 1; j < n; ++j) total = R::mac(total, row[j], lb[n - 1 - j], ov);
    if (ov) {
        atomicOr(status, 1);
        total = R::zero();
    }
    out[b] = total;
}

static __global__ void sz_guard_i64_batch_kernel(const long long* __restrict__ a, int n, uint32_t nmat,
                                                 int32_t* __restrict__ guard) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nmat) guard[b] = i64_guard_ok(a + (uint64_t)b * n * n, n) ? 0 : 1;
}

// Top-column terms of one block of layer k (multi-GPU block plan, after a
// partial layer without them): the block's outputs S (pattern P on the top
// columns) get, in ascending column order c in P, the terms
// a(k-1, c) * per(S \ {c}), whose predecessors sit at the same offset i in
// the block of pattern P \ {c} of layer k-1 (received from its owner). The top
// columns are the highest, so these terms come last in the reference's
// ascending order (permanent.cpp:164-174): partial + these is rounding-exact.
// init_first: the block's outputs have no other term (S = P).
struct TopSrc {
    int col[8];
    uint64_t base[8];
};

template <class R>
__global__ void sz_top_terms_kernel(const typename R::T* __restrict__ a, int n, int k,
                                    const typename R::T* __restrict__ prev, typename R::T* __restrict__ cur,
                                    uint64_t base, uint64_t len, int nsrc, TopSrc src, int init_first,
                                    int32_t* __restrict__ status) {
    using T = typename R::T;
    bool ov = false;
    const T* row = a + (size_t)(k - 1) * n;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
        T acc = init_first ? R::zero() : cur[base + i];
        for (int s = 0; s < nsrc; ++s) {
            const T c = row[src.col[s]];
            const T x = prev[src.base[s] + i];
            acc = (init_first && s == 0) ? R::mul(c, x, ov) : R::mac(acc, c, x, ov);
        }
        cur[base + i] = acc;
    }
    if (ov) atomicOr(status, 1);
}

static __global__ void sz_guard_i64_kernel(const long long* __restrict__ a, int n, int32_t* __restrict__ guard) {
    if (threadIdx.x == 0 && blockIdx.x == 0) guard[0] = i64_guard_ok(a, n) ? 0 : 1;
}

// n == 1 and n == 2 single-matrix cases (and any order <= 6 single matrix).
}  // namespace pl
