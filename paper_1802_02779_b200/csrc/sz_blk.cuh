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
// to whole ROWS of 32 blocks; a row stores its 2^LC x 32 values as
// [position of L][lane] (8 KB), L ordered by level |L| (BlkOrder), so the values
// one level needs from 32 neighbouring blocks are one contiguous run.
// tb[j][F] = the tile's first row (blk_tables_kernel).
//   window terms: the tile's window source = tile (F, j - 1), at most 4 rows
//                 (32 KB), staged whole in shared memory by one bulk copy;
//                 gathered by block index from the window table (wtab: 9 x
//                 12-bit entries per block);
//   high terms:   block q of tile (F \ {h}, j - 1): same row and lane. Each warp
//                 stages them through its own ring of kBlkSlots shared-memory
//                 slots: lane 0 issues one bulk copy per (piece of a level,
//                 stream), three chunks ahead of the reads (version 1 read them
//                 straight into registers, one group ahead: every group exposed
//                 an L2 round trip, profiles/r2c/NOTES.md).
// One CTA = 4 warps = the (at most) 4 rows of a tile, four CTAs per SM; CTAs
// claim tiles from a ticket counter in increasing F; warp 3 (the lightest row)
// also prepares the next tile's header.
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
// C(9, m), rows of 32 blocks per tile, first wtab entry of the m-subsets of the window:
// 4-, 4- and 10-bit fields of packed constants (a run-time binomial loop was 7 % of the
// kernel's instructions, profiles/r2c)
__host__ __device__ constexpr uint32_t blk_c9(int m) {  // 1 9 36 84 126 126 84 36 9 1
    return m < 0 || m > 9 ? 0u : (uint32_t)((0x7e54240901ull >> (8 * (m > 4 ? 9 - m : m))) & 0xffu);
}
__host__ __device__ constexpr uint32_t blk_rows9(int m) {  // 1 1 2 3 4 4 3 2 1 1
    return m < 0 || m > 9 ? 0u : (uint32_t)((0x1123443211ull >> (4 * m)) & 0xfu);
}
__host__ __device__ constexpr uint32_t blk_moff9(int m) {  // 0 1 10 46 130 256 | 382 466 502 511 512
    return m < 6 ? (uint32_t)((0x400820b80a00400ull >> (10 * (m < 0 ? 0 : m))) & 0x3ffu)
                 : (uint32_t)((0x2007fdf67497eull >> (10 * ((m > 10 ? 10 : m) - 6))) & 0x3ffu);
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

// In-row order of a block's values: by level |L|, then by L. Level P holds the
// positions [off[P], off[P + 1]), so the values one level needs from a
// predecessor block row are one contiguous run (one bulk copy).
template <int LC>
struct BlkOrder {
    int pos[1 << LC];
    int off[LC + 2];
};
template <int LC>
__host__ __device__ constexpr BlkOrder<LC> blk_order() {
    BlkOrder<LC> t{};
    int n = 0;
    for (int P = 0; P <= LC; ++P) {
        t.off[P] = n;
        for (int L = 0; L < (1 << LC); ++L) {
            int c = 0;
            for (int b = 0; b < LC; ++b) c += (L >> b) & 1;
            if (c == P) t.pos[L] = n++;
        }
    }
    t.off[LC + 1] = n;
    return t;
}

// A level is processed in pieces of at most SUB outputs (5 for 8-byte rings, 3
// for complex): eight pieces per block for both. Piece ip covers the in-row
// positions [first, first + count): packed 8 bits per piece for the issue side.
template <int LC>
struct BlkPieces;
template <>
struct BlkPieces<5> {  // counts 1 | 5 | 5 5 | 5 5 | 5 | 1
    static constexpr uint64_t kFirst = 0x1f1a15100b060100ull;
    static constexpr uint64_t kCount = 0x0105050505050501ull;
    static constexpr int kSub = 5;
};
template <>
struct BlkPieces<4> {  // counts 1 | 2 2 | 3 3 | 2 2 | 1
    static constexpr uint64_t kFirst = 0x0f0d0b0805030100ull;
    static constexpr uint64_t kCount = 0x0102020303020201ull;
    static constexpr int kSub = 3;
};
constexpr int kBlkPieces = 8;
#ifndef PL_BLK_SLOTS
#define PL_BLK_SLOTS 3
#endif
constexpr int kBlkSlots = PL_BLK_SLOTS;  // stream-ring slots per warp

// The warp's stream ring: slot s holds one (piece, stream) chunk, count x 32
// values; lane 0 issues the bulk copies kBlkSlots chunks ahead of the reads.
template <class T, int LC>
struct BlkRing {
    static constexpr uint32_t kSlotBytes = BlkPieces<LC>::kSub * 32 * sizeof(T);
    unsigned char* base;  // this warp's slots
    uint64_t* full;       // [kBlkSlots]
    uint32_t slot, par;   // read cursor: slot, phase parity bits per slot
    int ip, il;           // issue cursor: piece, stream
    uint32_t left;        // chunks not yet issued
    uint32_t islot;       // next slot to fill
};

template <class T, int LC>
__device__ __forceinline__ void blk_issue(BlkRing<T, LC>& rg, const BlkHdr& h, const T* __restrict__ rowp, int f,
                                          uint32_t dep) {
    // lane 0 only. rowp = prev + row r of the tile: stream l's block row is rowp + sb[l] * RE
    constexpr int RE = (1 << LC) * 32;
    const uint32_t first = (uint32_t)(BlkPieces<LC>::kFirst >> (8 * rg.ip)) & 0xffu;
    const uint32_t cnt = (uint32_t)(BlkPieces<LC>::kCount >> (8 * rg.ip)) & 0xffu;
    const uint32_t bytes = cnt * 32u * (uint32_t)sizeof(T);
    const T* src = rowp + (size_t)h.sb[rg.il] * RE + first * 32u;
    uint64_t* bar = rg.full + rg.islot;
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(rg.base + rg.islot * BlkRing<T, LC>::kSlotBytes + dep, src, bytes, bar);
    rg.islot = rg.islot + 1 == kBlkSlots ? 0 : rg.islot + 1;
    if (++rg.il == f) {
        rg.il = 0;
        ++rg.ip;
    }
    --rg.left;
}

// One piece of a block: the outputs of level P at in-level ordinals
// [O0, O0 + CN): register terms, window terms, then the high terms from the
// stream ring, in this order per output (ascending columns).
//   ar      a(j + P - 1, .) in shared memory
//   row0    the level's row is 0: a single-column subset, per = a(0, c)
//   pr[t]   window predecessor t: byte offset of its block in the source | column << 20
template <class R, int LC, int P, int O0, int CN, class T>
__device__ __forceinline__ void blk_piece(T (&val)[1 << LC], const T* __restrict__ ar, bool row0, int m,
                                          const uint32_t (&pr)[kBlkDW], const unsigned char* __restrict__ srcb, int f,
                                          const BlkHdr& h, BlkRing<T, LC>& rg, const T* __restrict__ rowp, int lane,
                                          uint32_t rt_zero, bool& ov) {
    constexpr int NL = 1 << LC;
    constexpr uint32_t LSTRIDE = 32 * sizeof(T);  // bytes between consecutive in-row positions
    constexpr BlkOrder<LC> ord = blk_order<LC>();
    constexpr int P0 = ord.off[P] + O0;  // first in-row position of the piece
    // register terms
    if constexpr (P >= 1) {
        T cl[LC];
#pragma unroll
        for (int v = 0; v < LC; ++v) cl[v] = ar[v];
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            if (ord.pos[L] < P0 || ord.pos[L] >= P0 + CN) continue;
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
            if (ord.pos[L] < P0 || ord.pos[L] >= P0 + CN) continue;
            const T x = *reinterpret_cast<const T*>(p + ord.pos[L] * LSTRIDE);
            if (P == 0 && t == 0)
                val[L] = row0 ? c : R::mul(c, x, ov);
            else
                val[L] = R::mac(val[L], c, x, ov);
        }
    }
    // high terms: chunk (piece, l) from the ring
    for (int l = 0; l < f; ++l) {
        const T c = ar[h.hcol[l]];
        mbar_wait(rg.full + rg.slot, (rg.par >> rg.slot) & 1u);
        const unsigned char* sp = rg.base + rg.slot * BlkRing<T, LC>::kSlotBytes + lane * sizeof(T);
        T xs[CN];
#pragma unroll
        for (int o = 0; o < CN; ++o) xs[o] = *reinterpret_cast<const T*>(sp + o * LSTRIDE);
        // the slot is refilled only after this warp's loads have returned (loaded_dep, sz_ws.cuh)
        const uint32_t dep = loaded_dep(xs, CN, rt_zero);
        rg.par ^= 1u << rg.slot;
        rg.slot = rg.slot + 1 == kBlkSlots ? 0 : rg.slot + 1;
        if (lane == 0 && rg.left) blk_issue<T, LC>(rg, h, rowp, f, dep);
        int o = 0;
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            if (ord.pos[L] < P0 || ord.pos[L] >= P0 + CN) continue;
            if (P == 0 && m == 0 && l == 0)
                val[L] = row0 ? c : R::mul(c, xs[o], ov);
            else
                val[L] = R::mac(val[L], c, xs[o], ov);
            ++o;
        }
    }
}

#ifndef PL_BLK_MINCTAS
#define PL_BLK_MINCTAS 4
#endif
template <class R, int LC>
__global__ void __launch_bounds__(32 * kBlkWarps, PL_BLK_MINCTAS)
    sz_blk_kernel(const typename R::T* __restrict__ a, int n, int j, const typename R::T* __restrict__ prev,
                  typename R::T* __restrict__ cur, typename R::T* __restrict__ out, uint32_t* __restrict__ ticket,
                  const uint32_t* __restrict__ flist, uint32_t ntiles, const uint32_t* __restrict__ tb_cur,
                  const uint32_t* __restrict__ tb_prev, const uint4* __restrict__ wtab, int32_t* __restrict__ status,
                  uint32_t hints) {
    using T = typename R::T;
    using Ring = BlkRing<T, LC>;
    constexpr int NL = 1 << LC;
    constexpr int RE = NL * 32;  // elements per row
    constexpr BlkOrder<LC> ord = blk_order<LC>();
    static_assert(RE * sizeof(T) == kBlkRowBytes, "row size");
    // dynamic shared memory: the tile's window source (4 rows), then the warps' stream rings
    extern __shared__ __align__(128) unsigned char blk_smem[];
    __shared__ BlkHdr hdr[2];
    __shared__ __align__(8) uint64_t src_full;
    __shared__ __align__(8) uint64_t ring_full[kBlkWarps][kBlkSlots];
    __shared__ T arow[LC + 1][kMaxOrder];  // a(j + p - 1, .), p = 0 .. LC
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* srcb = blk_smem;

    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&src_full, 1);
        for (int w = 0; w < kBlkWarps; ++w)
            for (int s = 0; s < kBlkSlots; ++s) mbar_init(&ring_full[w][s], 1);
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
    auto publish = [&](int b) {  // whole warp 3: header of the next tile
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
            h.src_bytes = m >= 1 ? blk_rows9(m - 1) * kBlkRowBytes : 0u;
            h.src_row = m >= 1 ? __ldg(tb_prev + F) : 0u;
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

    Ring rg;
    rg.base = blk_smem + kBlkWarps * kBlkRowBytes + (size_t)warp * kBlkSlots * Ring::kSlotBytes;
    rg.full = &ring_full[warp][0];
    rg.slot = 0;
    rg.par = 0;
    rg.islot = 0;
    const uint32_t rt_zero = hints >> 31;  // bit 31 is never set
    bool ov = false;
    uint32_t src_phase = 0;
    for (uint32_t i = 0;; ++i) {
        const int b = (int)(i & 1u);
        __syncthreads();  // tile i - 1 done everywhere (the source buffer is free); hdr[b] visible
        const BlkHdr& h = hdr[b];
        if (h.m < 0) break;
        const int m = (hints & 2u) ? 0 : h.m;  // hints bit 1: timing probe without the window terms
        const bool has_src = h.src_bytes != 0;
        if (threadIdx.x == 96 && has_src) {
            mbar_arrive_expect_tx(&src_full, h.src_bytes);
            bulk_g2s(srcb, prev + (size_t)h.src_row * RE, h.src_bytes, &src_full);
        }
        if (warp == 3) publish(b ^ 1);
        if ((uint32_t)warp < h.nrows) {
            const int f = (hints & 1u) ? 0 : h.f;  // hints bit 0: timing probe without the high terms
            const uint32_t nb = h.nb;
            const uint32_t q = (uint32_t)warp * 32u + (uint32_t)lane;
            const bool valid = q < nb;
            const uint32_t qc = valid ? q : nb - 1u;
            const T* rowp = prev + (size_t)warp * RE + lane;
            // start the stream ring: the first chunks of this row
            rg.ip = 0;
            rg.il = 0;
            rg.left = (uint32_t)(kBlkPieces * f);
            if (lane == 0) {
#pragma unroll
                for (int s = 0; s < kBlkSlots; ++s)
                    if (rg.left) blk_issue<T, LC>(rg, h, rowp - lane, f, 0u);
            }
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
            T* dst = cur + ((size_t)h.cur_row + warp) * RE + lane;
            if (has_src) mbar_wait(&src_full, src_phase);
            T val[NL];
            auto store_level = [&](int P) {
                if (valid) {
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        if (__builtin_popcount(L) == P) dst[ord.pos[L] * 32] = val[L];
                }
            };
#define PL_BLK_PIECE(P, O0, CN, R0) \
    blk_piece<R, LC, P, O0, CN>(val, arow[P], R0, m, pr, srcb, f, h, rg, rowp - lane, lane, rt_zero, ov)
            // level 0 (j = 0: the empty set, never used as a factor: row0 below)
            if (j == 0) {
                val[0] = R::zero();
            } else {
                PL_BLK_PIECE(0, 0, 1, j == 1);
            }
            store_level(0);
            if constexpr (LC == 5) {
                PL_BLK_PIECE(1, 0, 5, j == 0);
                store_level(1);
                PL_BLK_PIECE(2, 0, 5, false);
                PL_BLK_PIECE(2, 5, 5, false);
                store_level(2);
                PL_BLK_PIECE(3, 0, 5, false);
                PL_BLK_PIECE(3, 5, 5, false);
                store_level(3);
                PL_BLK_PIECE(4, 0, 5, false);
                store_level(4);
                PL_BLK_PIECE(5, 0, 1, false);
                store_level(5);
            } else {
                PL_BLK_PIECE(1, 0, 2, j == 0);
                PL_BLK_PIECE(1, 2, 2, j == 0);
                store_level(1);
                PL_BLK_PIECE(2, 0, 3, false);
                PL_BLK_PIECE(2, 3, 3, false);
                store_level(2);
                PL_BLK_PIECE(3, 0, 2, false);
                PL_BLK_PIECE(3, 2, 2, false);
                store_level(3);
                PL_BLK_PIECE(4, 0, 1, false);
                store_level(4);
            }
#undef PL_BLK_PIECE
            // the last super-layer is the single block of every column: its top value is the permanent
            if (j == n - LC && q == 0) out[0] = val[NL - 1];
        }
        if (has_src) src_phase ^= 1u;
    }
    if (ov) atomicOr(status, 1);
}

}  // namespace pl
