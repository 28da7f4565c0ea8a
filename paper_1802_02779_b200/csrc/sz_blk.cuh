// Register-blocked layer kernel for one large matrix (float rings).
//
// Recurrence (reference proj/src/permanent.cpp:164-175):
//     per(S) = sum_{j in S, ascending} a(|S|-1, j) * per(S \ {j}).
//
// The per-layer kernels (sz_ws.cuh, sz_lean.cuh) give every thread one or two
// outputs and pay the subset arithmetic (low-term table decode, addresses,
// stage hand-offs) once per TERM: ~24 issued instructions per term, of which 2
// (f64) or 8 (c128) are arithmetic. Here a thread owns a BLOCK: the 2^LC
// subsets W u L, L within the LC lowest columns (LC = 5 for 8-byte rings, 4 for
// complex), of one subset W of the other columns. The block's 2^LC values stay
// in registers, so
//   * the terms of the LC lowest columns (`register terms`) read registers,
//     with compile-time indices and warp-uniform coefficients;
//   * every other predecessor of the block's outputs is one predecessor BLOCK
//     (W \ {w}, same L): its address is computed once per 2^LC terms and the
//     values are read at immediate offsets.
// Columns: [0, LC) register columns; [LC, LC + 9) the gather window; the rest
// high columns. A tile is the set of blocks sharing the high part F of W:
// C(9, m) blocks indexed by the colex rank q of the window part V (|V| = m).
//
// A launch computes one SUPER-LAYER j = |W| (0 <= j <= n - LC): every block
// with |W| = j, i.e. entries of the layers j .. j + LC of the reference DP
// (row |S| - 1 = j + |L| - 1 differs per level |L| inside a block). Inside a
// block the levels run in order |L| = 0 .. LC, because the register terms of
// level p read the level p - 1 values of the same block (final, all terms in).
// Per output the terms run: register columns ascending, window columns
// ascending, high columns ascending = the reference's ascending-j fold, first
// term initialising the accumulator; the non-FMA rings are bitwise equal to it.
//
// Storage of a super-layer: tile after tile (increasing F); a tile is padded
// to whole ROWS of 32 blocks; a row stores its 2^LC x 32 values as [L][lane]
// (8 KB), so a warp's load of one L of 32 neighbouring blocks is one coalesced
// 256/512-byte access. tb[j][F] = the tile's first row (blk_tables_kernel).
//   window terms: the tile's window source = tile (F, j - 1), at most 4 rows
//                 (32 KB), staged whole in shared memory by one bulk copy,
//                 double buffered across tiles; gathered by block index from
//                 the window table (wtab: 9 x 12-bit entries per block);
//   high terms:   block q of tile (F \ {h}, j - 1): same row and lane, read
//                 straight from global memory (L2) into registers, a group of
//                 predecessors ahead of the arithmetic.
// One CTA = 4 warps = the (at most) 4 rows of a tile; CTAs claim tiles from a
// ticket counter in increasing F; warp 3 (the lightest row) also prepares the
// next tile's header and source copy.
#pragma once

#include <cstdint>

#include "ring.cuh"
#include "sz_ws.cuh"  // mbarrier / bulk-copy PTX helpers

namespace pl {

constexpr int kBlkDW = 9;        // gather-window columns
constexpr int kBlkWarps = 4;     // rows per tile: ceil(C(9, 4) / 32)
constexpr int kBlkMaxHigh = 24;  // high columns: n - LC - 9 <= 21
constexpr uint32_t kBlkRowBytes = 8192;
constexpr uint32_t kBlkInvalid = 0xffffffffu;

__host__ __device__ constexpr int blk_reg_cols(int elem_bytes) { return elem_bytes == 16 ? 4 : 5; }
__host__ __device__ constexpr uint32_t blk_c9(int m) { return m < 0 || m > 9 ? 0u : (uint32_t)binom_u64(9, m); }
__host__ __device__ constexpr uint32_t blk_rows9(int m) { return (blk_c9(m) + 31u) / 32u; }
// first wtab entry of the m-subsets of the window
__host__ __device__ constexpr uint32_t blk_moff9(int m) {
    uint32_t s = 0;
    for (int i = 0; i < m; ++i) s += blk_c9(i);
    return s;
}

struct BlkHdr {
    int32_t m, f;  // m < 0: no more tiles
    uint32_t nb, nrows, cur_row, src_row, src_bytes;
    uint32_t sb[kBlkMaxHigh];   // first row of the stream tile (F \ {F_l}, j - 1)
    uint8_t hcol[kBlkMaxHigh];  // column of F_l
};

// ---------------------------------------------------------------- tables

// For every super-layer j (blockIdx.x): tb[j * 2^H + F] = first row of tile
// (F, j) (kBlkInvalid when j - popc(F) is outside [0, 9]) and the list of
// valid F in increasing order at flist + fl_off[j]. One CTA scans all F.
static __global__ void blk_tables_kernel(int H, uint32_t* __restrict__ tb, uint32_t* __restrict__ flist,
                                         const uint64_t* __restrict__ fl_off) {
    const int j = blockIdx.x;
    const uint32_t nF = 1u << H;
    uint32_t* tbj = tb + (size_t)j * nF;
    uint32_t* fl = flist + fl_off[j];
    __shared__ uint32_t wsum_r[32], wsum_v[32];
    __shared__ uint32_t carry_r, carry_v;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry_r = carry_v = 0;
    __syncthreads();
    for (uint32_t F0 = 0; F0 < nF; F0 += blockDim.x) {
        const uint32_t F = F0 + threadIdx.x;
        const int m = j - __popc(F);
        const bool valid = F < nF && m >= 0 && m <= kBlkDW;
        const uint32_t rows = valid ? blk_rows9(m) : 0u;
        uint32_t ir = rows, iv = valid ? 1u : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, ir, d), b = __shfl_up_sync(0xffffffffu, iv, d);
            if (lane >= d) {
                ir += a;
                iv += b;
            }
        }
        if (lane == 31) {
            wsum_r[warp] = ir;
            wsum_v[warp] = iv;
        }
        __syncthreads();
        uint32_t br = carry_r, bv = carry_v;
        for (int w = 0; w < warp; ++w) {
            br += wsum_r[w];
            bv += wsum_v[w];
        }
        if (valid) {
            tbj[F] = br + ir - rows;
            fl[bv + iv - 1] = F;
        } else if (F < nF) {
            tbj[F] = kBlkInvalid;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) {
            uint32_t tr = 0, tv = 0;
            for (int w = 0; w < nw; ++w) {
                tr += wsum_r[w];
                tv += wsum_v[w];
            }
            carry_r += tr;
            carry_v += tv;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- kernel

template <class T>
__device__ __forceinline__ T blk_ld_global(const T* p) {
    if constexpr (sizeof(T) == 16) {
        double2 v;
        asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
        return v;
    } else {
        unsigned long long v;
        asm volatile("ld.global.L1::no_allocate.b64 %0, [%1];\n" : "=l"(v) : "l"(p));
        return *reinterpret_cast<T*>(&v);
    }
}

// One level (|L| = P) of a block: val[L] for every L of popcount P.
//   ar      a(j + P - 1, .) in shared memory
//   row0    the level's row is 0: a single-column subset, per = a(0, c)
//   pr[t]   window predecessor t: byte offset of its block in the source | column << 20
//   srcb    the tile's window source in shared memory
//   sp      prev + lane (+ row r): stream tile l's block is at sp + sb[l] * ROW
template <class R, int LC, int P, class T>
__device__ __forceinline__ void blk_level(T (&val)[1 << LC], const T* __restrict__ ar, bool row0, int m,
                                          const uint32_t (&pr)[kBlkDW], const unsigned char* __restrict__ srcb, int f,
                                          const BlkHdr& h, const T* __restrict__ sp, bool& ov) {
    constexpr int NL = 1 << LC;
    constexpr uint32_t LSTRIDE = 32 * sizeof(T);  // bytes between consecutive L of one block
    constexpr int CNT = (int)binom_u64(LC, P);
    // predecessors per group of stream loads (issued one group ahead)
    // (at most 10 8-byte or 6 16-byte values per group: two groups live in registers)
    constexpr int GV = sizeof(T) == 16 ? 6 : 10;
    constexpr int UL = GV / CNT >= 4 ? 4 : (GV / CNT >= 1 ? GV / CNT : 1);
    // register terms
    if constexpr (P >= 1) {
        T cl[LC];
#pragma unroll
        for (int v = 0; v < LC; ++v) cl[v] = ar[v];
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            if (__builtin_popcount(L) != P) continue;
            bool first = true;
#pragma unroll
            for (int v = 0; v < LC; ++v) {
                if (!((L >> v) & 1)) continue;
                const T x = val[L ^ (1 << v)];
                if (first) {
                    if constexpr (P == 1)
                        val[L] = row0 ? cl[v] : R::mul(cl[v], x, ov);
                    else
                        val[L] = R::mul(cl[v], x, ov);
                } else {
                    val[L] = R::mac(val[L], cl[v], x, ov);
                }
                first = false;
            }
        }
    }
    // window terms (m is uniform over the tile)
#pragma unroll
    for (int t = 0; t < kBlkDW; ++t) {
        if (t >= m) break;
        const T c = ar[pr[t] >> 20];
        const unsigned char* p = srcb + (pr[t] & 0xfffffu);
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            if (__builtin_popcount(L) != P) continue;
            const T x = *reinterpret_cast<const T*>(p + L * LSTRIDE);
            if (P == 0 && t == 0)
                val[L] = row0 ? c : R::mul(c, x, ov);
            else
                val[L] = R::mac(val[L], c, x, ov);
        }
    }
    // high terms: groups of UL predecessors, the next group's loads in flight
    if (f > 0) {
        T nx[UL][CNT];
        auto issue = [&](int l0) {
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                if (l0 + u < f) {
                    const T* p = sp + (size_t)h.sb[l0 + u] * (NL * 32);
                    int o = 0;
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        if (__builtin_popcount(L) != P) continue;
                        nx[u][o++] = blk_ld_global(p + L * 32);
                    }
                }
            }
        };
        issue(0);
        for (int l0 = 0; l0 < f; l0 += UL) {
            T cx[UL][CNT];
            T cc[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) {
#pragma unroll
                for (int o = 0; o < CNT; ++o) cx[u][o] = nx[u][o];
                cc[u] = ar[h.hcol[min(l0 + u, f - 1)]];
            }
            issue(l0 + UL);
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                if (l0 + u < f) {
                    int o = 0;
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        if (__builtin_popcount(L) != P) continue;
                        if (P == 0 && m == 0 && l0 + u == 0)
                            val[L] = row0 ? cc[u] : R::mul(cc[u], cx[u][o], ov);
                        else
                            val[L] = R::mac(val[L], cc[u], cx[u][o], ov);
                        ++o;
                    }
                }
            }
        }
    }
}

template <class R, int LC>
__global__ void __launch_bounds__(32 * kBlkWarps, 3)
    sz_blk_kernel(const typename R::T* __restrict__ a, int n, int j, const typename R::T* __restrict__ prev,
                  typename R::T* __restrict__ cur, typename R::T* __restrict__ out, uint32_t* __restrict__ ticket,
                  const uint32_t* __restrict__ flist, uint32_t ntiles, const uint32_t* __restrict__ tb_cur,
                  const uint32_t* __restrict__ tb_prev, const uint4* __restrict__ wtab, int32_t* __restrict__ status,
                  uint32_t hints) {
    using T = typename R::T;
    constexpr int NL = 1 << LC;
    constexpr int RE = NL * 32;  // elements per row
    static_assert(RE * sizeof(T) == kBlkRowBytes, "row size");
    extern __shared__ __align__(128) unsigned char blk_smem[];  // two window sources, 4 rows each
    __shared__ BlkHdr hdr[2];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ T arow[LC + 1][kMaxOrder];  // a(j + p - 1, .), p = 0 .. LC
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int e = threadIdx.x; e < (LC + 1) * n; e += blockDim.x) {
        const int p = e / n, c = e - p * n, row = j + p - 1;
        if (row >= 0 && row < n) arow[p][c] = a[(size_t)row * n + c];
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the previous super-layer is complete and visible
    asm volatile("fence.proxy.async.global;\n" ::: "memory");

    // producer state (warp 3): the next tile to publish
    uint32_t t_next = 0, F_next = 0;
    auto publish = [&](int b) {  // whole warp 3
        const uint32_t t = __shfl_sync(0xffffffffu, t_next, 0);
        BlkHdr& h = hdr[b];
        if (t >= ntiles) {
            if (lane == 0) h.m = -1;
            return;
        }
        const uint32_t F = __shfl_sync(0xffffffffu, F_next, 0);
        const int f = __popc(F), m = j - f;
        if (lane < f) {
            const int bit = __fns(F, 0, lane + 1);
            h.sb[lane] = __ldg(tb_prev + (F & ~(1u << bit)));
            h.hcol[lane] = (uint8_t)(LC + kBlkDW + bit);
        }
        if (lane == 0) {
            h.m = m;
            h.f = f;
            h.nb = blk_c9(m);
            h.nrows = blk_rows9(m);
            h.cur_row = __ldg(tb_cur + F);
            const uint32_t sbytes = m >= 1 ? blk_rows9(m - 1) * kBlkRowBytes : 0u;
            h.src_bytes = sbytes;
            if (sbytes) {
                const uint32_t srow = __ldg(tb_prev + F);
                h.src_row = srow;
                mbar_arrive_expect_tx(&full[b], sbytes);
                bulk_g2s(blk_smem + (size_t)b * kBlkWarps * kBlkRowBytes, prev + (size_t)srow * RE, sbytes, &full[b]);
            }
            // claim the tile after
            t_next = atomicAdd(ticket, 1u);
            F_next = t_next < ntiles ? __ldg(flist + t_next) : 0u;
        }
    };
    if (warp == 3) {
        if (lane == 0) {
            t_next = atomicAdd(ticket, 1u);
            F_next = t_next < ntiles ? __ldg(flist + t_next) : 0u;
        }
        publish(0);
    }

    bool ov = false;
    uint32_t phbits = 0;
    for (uint32_t i = 0;; ++i) {
        const int b = (int)(i & 1u);
        __syncthreads();  // tile i - 1 done everywhere (its source buffer is free); hdr[b] visible
        const BlkHdr& h = hdr[b];
        if (h.m < 0) break;
        const int m = (hints & 2u) ? 0 : h.m;  // hints bit 1: timing probe without the window terms
        if (warp == 3) publish(b ^ 1);
        const bool has_src = h.src_bytes != 0;
        if ((uint32_t)warp < h.nrows) {
            const int f = (hints & 1u) ? 0 : h.f;  // hints bit 0: timing probe without the high terms
            const uint32_t nb = h.nb;
            const uint32_t q = (uint32_t)warp * 32u + (uint32_t)lane;
            const bool valid = q < nb;
            const uint32_t qc = valid ? q : nb - 1u;
            uint32_t pr[kBlkDW];
            if (m >= 1) {
                const uint4 e = __ldg(wtab + blk_moff9(m) + qc);
                const uint64_t lo = e.x | (uint64_t)e.y << 32, hi = e.z | (uint64_t)e.w << 32;
#pragma unroll
                for (int t = 0; t < kBlkDW; ++t) {
                    const uint32_t fld = (uint32_t)((t < 5 ? lo >> (12 * t) : hi >> (12 * (t - 5))) & 0xfffu);
                    const uint32_t bi = fld & 127u, w = fld >> 7;
                    pr[t] = ((bi >> 5) * kBlkRowBytes + (bi & 31u) * (uint32_t)sizeof(T)) | (uint32_t)(LC + w) << 20;
                }
            } else {
#pragma unroll
                for (int t = 0; t < kBlkDW; ++t) pr[t] = 0;
            }
            const unsigned char* srcb = blk_smem + (size_t)b * kBlkWarps * kBlkRowBytes;
            const T* sp = prev + (size_t)warp * RE + lane;
            T* dst = cur + ((size_t)h.cur_row + warp) * RE + lane;
            if (has_src) mbar_wait(&full[b], (phbits >> b) & 1u);
            T val[NL];
            auto store_level = [&](int P) {
                if (valid) {
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        if (__builtin_popcount(L) == P) dst[L * 32] = val[L];
                }
            };
            // level 0 (j = 0: the empty set, never used as a factor: row0 below)
            if (j == 0) {
                val[0] = R::zero();
            } else {
                blk_level<R, LC, 0>(val, arow[0], j == 1, m, pr, srcb, f, h, sp, ov);
            }
            store_level(0);
            blk_level<R, LC, 1>(val, arow[1], j == 0, m, pr, srcb, f, h, sp, ov);
            store_level(1);
            blk_level<R, LC, 2>(val, arow[2], false, m, pr, srcb, f, h, sp, ov);
            store_level(2);
            blk_level<R, LC, 3>(val, arow[3], false, m, pr, srcb, f, h, sp, ov);
            store_level(3);
            blk_level<R, LC, 4>(val, arow[4], false, m, pr, srcb, f, h, sp, ov);
            store_level(4);
            if constexpr (LC >= 5) {
                blk_level<R, LC, 5>(val, arow[LC >= 5 ? 5 : 0], false, m, pr, srcb, f, h, sp, ov);
                store_level(5);
            }
            // the last super-layer is the single block of every column: its top value is the permanent
            if (j == n - LC && q == 0) out[0] = val[NL - 1];
        }
        if (has_src) phbits ^= 1u << b;
    }
    if (ov) atomicOr(status, 1);
}

}  // namespace pl
