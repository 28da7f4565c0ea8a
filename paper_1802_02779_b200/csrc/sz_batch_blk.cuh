// Register-blocked FP32-exact pack kernel for int64 batches, 10 <= n <= 12 (C3).
//
// Same recurrence and exactness argument as sz_batch_f32_pack_kernel
// (reference proj/src/permanent.cpp:164-175; every operand, product and partial
// sum of an FP32-exact matrix is an integer below 2^24, so the order of the
// additions does not matter and each FFMA is exact). That kernel gives a thread
// one subset S at a time and pays, per term, a predecessor-table load, a
// gathered coefficient load and a gathered operand load for four FFMAs: it is
// L1TEX-bound (89 % busy, profiles/r2/full_c3.md). Here a thread owns a BLOCK
// (sz_blk.cuh): the 2^LC subsets W u L, L within the LC = n - 9 lowest columns,
// of one subset W of the other nine columns, with the block's 2^LC packs in
// registers. Per predecessor W \ {w} the thread decodes one table entry and
// reads 2^LC operand packs at immediate offsets; the coefficients a(row, w) are
// read once per level |L| (LC + 1 loads per predecessor); the terms of the LC
// lowest columns read registers and warp-uniform coefficients. Per pack-term:
// ~1.4 shared loads instead of 3 L1TEX operations.
//
// A CTA of 128 threads runs one four-matrix pack: super-layer j = |W| = 0 .. 9
// has C(9, j) <= 126 blocks, one per thread, __syncthreads between super-layers;
// a super-layer is stored as 2^LC planes [L][block] of 126 packs (conflict-free
// stores, gathers by block index), two buffers. per(empty set) = 1 starts the
// recurrence (a * 1 is exact).
#pragma once

#include "sz_blk.cuh"
#include "sz_kernels.cuh"

namespace pl {

constexpr int kF32BlkThreads = 128;
constexpr int kF32BlkPlane = 126;  // packs per plane: C(9, 4)

template <int N>
__host__ __device__ constexpr size_t f32_blk_smem_bytes() {
    // matrix packs + two super-layer buffers of 2^LC planes (16-byte packs); the
    // one-matrix fallback layout (8-byte elements) fits inside
    constexpr size_t blk = ((size_t)N * N + 2 * (size_t)(1 << (N - 9)) * kF32BlkPlane) * 16;
    constexpr size_t single = ((size_t)N * N + 2 + 2 * (binom_u64(N, N / 2) + 1)) * 8;
    return (blk > single ? blk : single) + 64;
}

// The block DP of one jointly FP32-exact pack; returns the pack of permanents
// (valid in thread 0).
template <int N, class PT>
__device__ __forceinline__ PT smem_dp_blk_f32(const PT* __restrict__ mat, PT* buf0, PT* buf1,
                                              const uint4* __restrict__ wtab) {
    using PR = PackRing<RF32X, 4>;
    constexpr int LC = N - 9, NL = 1 << LC;
    constexpr uint32_t PSB = kF32BlkPlane * sizeof(PT);  // plane stride in bytes
    const int tid = threadIdx.x;
    bool ov = false;
    PT* prev = buf0;
    PT* cur = buf1;
    PT top = PR::zero();
#pragma unroll 1
    for (int j = 0; j <= 9; ++j) {
        const int nb = (int)blk_c9(j);
        if (tid < nb) {
            // predecessor t: byte offset of block rank9(W \ {w_t}) in a plane | column byte offset << 16
            uint32_t pr[9];
            {
                const uint4 e = __ldg(wtab + blk_moff9(j) + tid);
                const uint64_t lo = e.x | (uint64_t)e.y << 32, hi = e.z | (uint64_t)e.w << 32;
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    const uint32_t fld = (uint32_t)((t < 5 ? lo >> (12 * t) : hi >> (12 * (t - 5))) & 0xfffu);
                    pr[t] = (fld & 127u) * (uint32_t)sizeof(PT) | ((LC + (fld >> 7)) * (uint32_t)sizeof(PT)) << 16;
                }
            }
            const char* pv = reinterpret_cast<const char*>(prev);
            PT val[NL];
#pragma unroll
            for (int p = 0; p <= LC; ++p) {
                const int row = j + p - 1;
                if (row < 0) {  // the empty set
#pragma unroll
                    for (int i = 0; i < 4; ++i) val[0].v[i] = 1.0f;
                    continue;
                }
                const char* rowp = reinterpret_cast<const char*>(mat + row * N);
                // register terms
                if (p >= 1) {
                    PT cl[LC > 0 ? LC : 1];
#pragma unroll
                    for (int v = 0; v < LC; ++v) cl[v] = *reinterpret_cast<const PT*>(rowp + v * sizeof(PT));
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        if (__builtin_popcount(L) != p) continue;
                        bool first = true;
#pragma unroll
                        for (int v = 0; v < LC; ++v) {
                            if (!((L >> v) & 1)) continue;
                            val[L] = first ? PR::mul(cl[v], val[L ^ (1 << v)], ov)
                                           : PR::mac(val[L], cl[v], val[L ^ (1 << v)], ov);
                            first = false;
                        }
                    }
                }
                // terms of the nine upper columns
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    if (t >= j) break;
                    const PT c = *reinterpret_cast<const PT*>(rowp + (pr[t] >> 16));
                    const char* xp = pv + (pr[t] & 0xffffu);
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        if (__builtin_popcount(L) != p) continue;
                        const PT x = *reinterpret_cast<const PT*>(xp + L * PSB);
                        val[L] = (p == 0 && t == 0) ? PR::mul(c, x, ov) : PR::mac(val[L], c, x, ov);
                    }
                }
            }
#pragma unroll
            for (int L = 0; L < NL; ++L) cur[L * kF32BlkPlane + tid] = val[L];
            top = val[NL - 1];
        }
        __syncthreads();
        PT* t = prev;
        prev = cur;
        cur = t;
    }
    return top;  // thread 0 ran the single block of super-layer 9
}

template <int N>
__global__ void __launch_bounds__(kF32BlkThreads) sz_batch_f32_blk_kernel(
    const long long* __restrict__ a, long long* __restrict__ out, int64_t count, int maxc,
    const uint16_t* __restrict__ ptab, const uint32_t* __restrict__ poff, const uint32_t* __restrict__ ptab32_8,
    const uint4* __restrict__ wtab, int32_t* __restrict__ status) {
    constexpr int E = N * N, P = 4;
    using PR = PackRing<RF32X, P>;
    using PT = typename PR::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int mode[P], flag;
    const int tid = threadIdx.x;
    const int64_t npacks = (count + P - 1) / P;
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
            PT* buf1 = buf0 + (1 << (N - 9)) * kF32BlkPlane;
            for (int e = tid; e < E; e += blockDim.x) {
                PT x;
#pragma unroll
                for (int i = 0; i < P; ++i) x.v[i] = (float)g[(size_t)i * E + e];
                mat[e] = x;
            }
            __syncthreads();
            const PT t = smem_dp_blk_f32<N, PT>(mat, buf0, buf1, wtab);
            if (tid == 0) {
#pragma unroll
                for (int i = 0; i < P; ++i) out[b0 + i] = (long long)t.v[i];
            }
        } else {
            f32_pack_members<N>(g, have, mode, flag, smem_raw, maxc, ptab, poff, ptab32_8, out, b0, status);
        }
        __syncthreads();
    }
}

}  // namespace pl
