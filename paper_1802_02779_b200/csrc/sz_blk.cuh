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
#include <cstdio>

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
    int32_t m, f;  // window / high terms used (m < 0: no more tiles)
    uint32_t nb, nrows, nsrc_rows, cur_row, src_row;
    uint32_t g0, nch;           // the tile's chunks in the CTA's chunk sequence: [g0, g0 + nch)
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
#define PL_BLK_SLOTS 4
#endif
constexpr int kBlkSlots = PL_BLK_SLOTS;  // chunk-ring slots per CTA
constexpr int kBlkHdrs = 4;              // tile headers in flight per CTA

// A chunk: the values of one piece (<= kSub in-row positions) of every row of
// one predecessor tile -- contiguous in the tile-major layout [position][row][lane]
// -- staged by one bulk copy. The chunks of a tile, in the order they are read:
// per piece, the window source (tile (F, j - 1), if the tile has window terms),
// then the stream tiles l = 0 .. f - 1.
template <class T, int LC>
struct BlkChunks {
    static constexpr uint32_t kSlotBytes = BlkPieces<LC>::kSub * kBlkWarps * 32 * sizeof(T);
};

// Shared state of the CTA's chunk ring.
struct BlkRingSh {
    uint64_t full[kBlkSlots];  // chunk landed (transaction bytes)
    uint32_t readers[kBlkSlots];  // warps that have finished reading the slot's chunk
    uint64_t hdr_full[kBlkHdrs];   // header published (publisher arrives)
    uint64_t hdr_empty[kBlkHdrs];  // every warp has left the tile (kBlkWarps arrivals)
};

// mbarrier wait of the block kernel; -DPL_BLK_DEBUG: a watchdog that reports a wait that never ends.
__device__ __forceinline__ void blk_wait(uint64_t* bar, unsigned parity, int tag, uint32_t a, uint32_t b) {
#ifdef PL_BLK_DEBUG
    for (unsigned long long spins = 0;; ++spins) {
        if (mbar_test(bar, parity)) return;
        if (spins == 50000000ull && (threadIdx.x & 31) == 0)
            printf("blk stuck: cta %d warp %d tag %d a %u b %u parity %u\n", (int)blockIdx.x, (int)(threadIdx.x >> 5), tag,
                   a, b, parity);
        if (spins == 200000000ull) __trap();
    }
#else
    (void)tag;
    (void)a;
    (void)b;
    mbar_wait(bar, parity);
#endif
}

// Issue chunk gi of the CTA's sequence into its slot (one thread). `ti` is a
// tile whose header is known to be published and whose chunks start at or
// before gi; the chunk lies in tile ti or ti + 1 (a tile has 0 or >= 8 chunks).
template <class T, int LC>
__device__ __forceinline__ void blk_issue_chunk(uint32_t gi, uint32_t ti, const BlkHdr* hdr, BlkRingSh& rs,
                                                unsigned char* ring, const T* __restrict__ prev, uint32_t hints) {
    constexpr int RE = (1 << LC) * 32;
    const BlkHdr* h = &hdr[ti % kBlkHdrs];
    if (h->m < 0) return;  // the CTA has no (more) tiles
    if (gi >= h->g0 + h->nch) {
        ++ti;
        blk_wait(&rs.hdr_full[ti % kBlkHdrs], (ti / kBlkHdrs) & 1u, 1, ti, gi);
        h = &hdr[ti % kBlkHdrs];
        if (h->m < 0 || gi >= h->g0 + h->nch) return;  // past the last tile (or an empty one)
    }
    const uint32_t local = gi - h->g0;
    const uint32_t s = h->m >= 1 ? 1u : 0u, per = (uint32_t)h->f + s;
    const uint32_t ip = local / per, idx = local - ip * per;
    const uint32_t first = (uint32_t)(BlkPieces<LC>::kFirst >> (8 * ip)) & 0xffu;
    const uint32_t cnt = (uint32_t)(BlkPieces<LC>::kCount >> (8 * ip)) & 0xffu;
    uint32_t rows, base;
    bool skip;  // timing probes (hints bit 0: no high terms, bit 1: no window terms): the chunk stays empty
    if (s && idx == 0) {
        rows = h->nsrc_rows;
        base = h->src_row;
        skip = hints & 2u;
    } else {
        rows = h->nrows;
        base = h->sb[idx - s];
        skip = hints & 1u;
    }
    const uint32_t slot = gi % kBlkSlots;
    if (skip) {
        mbar_arrive(&rs.full[slot]);
        return;
    }
    const uint32_t bytes = cnt * rows * 32u * (uint32_t)sizeof(T);
    const T* src = prev + (size_t)base * RE + (size_t)first * rows * 32u;
    mbar_arrive_expect_tx(&rs.full[slot], bytes);
    bulk_g2s(ring + slot * BlkChunks<T, LC>::kSlotBytes, src, bytes, &rs.full[slot]);
}

// A warp has finished reading chunk g (its loads have returned: `dep` is
// computed from them, see loaded_dep): the last of the CTA's warps refills the
// slot with chunk g + kBlkSlots. Every warp passes every chunk, also the warps
// without a row in the tile (they wait for the chunk and release it unread):
// a warp that skipped ahead would wait two phases ahead of a slot's barrier,
// which a one-bit phase parity cannot tell from the phase already completed.
template <class T, int LC>
__device__ __forceinline__ void blk_release(uint32_t g, uint32_t ti, uint32_t nrows, const BlkHdr* hdr, BlkRingSh& rs,
                                            unsigned char* ring, const T* __restrict__ prev, int lane, uint32_t dep,
                                            uint32_t hints) {
    if (lane == 0) {
        const uint32_t slot = g % kBlkSlots;
        const uint32_t old = atomicAdd(&rs.readers[slot + dep], 1u);
        if (old + 1u == (uint32_t)kBlkWarps) {
            rs.readers[slot] = 0;
            blk_issue_chunk<T, LC>(g + kBlkSlots, ti, hdr, rs, ring, prev, hints);
        }
    }
}

// One piece of a block row: the outputs of level P at in-level ordinals
// [O0, O0 + CN): register terms, window terms, then the high terms, in this
// order per output (ascending columns). `g` is the CTA's chunk counter.
//   ar      a(j + P - 1, .) in shared memory
//   row0    the level's row is 0: a single-column subset, per = a(0, c)
//   pr[t]   window predecessor t: byte offset of its block inside one position of the source chunk | column << 20
template <class R, int LC, int P, int O0, int CN, class T>
__device__ __forceinline__ void blk_piece(T (&val)[1 << LC], const T* __restrict__ ar, bool row0, int m,
                                          const uint32_t (&pr)[kBlkDW], int f, const BlkHdr& h, uint32_t ti,
                                          const BlkHdr* hdr, BlkRingSh& rs, unsigned char* ring,
                                          const T* __restrict__ prev, uint32_t& g, int warp, int lane,
                                          uint32_t hints, bool& ov) {
    constexpr int NL = 1 << LC;
    constexpr BlkOrder<LC> ord = blk_order<LC>();
    constexpr int P0 = ord.off[P] + O0;  // first in-row position of the piece
    const uint32_t nrows = h.nrows;
    const uint32_t rt_zero = hints >> 31;  // bit 31 is never set: a run-time zero (loaded_dep)
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
    // window terms: the piece's positions of the source tile, one chunk
    if (m >= 1) {
        const uint32_t slot = g % kBlkSlots;
        blk_wait(&rs.full[slot], (g / kBlkSlots) & 1u, 2, ti, g);
        const unsigned char* sb = ring + slot * BlkChunks<T, LC>::kSlotBytes;
        const uint32_t pstride = h.nsrc_rows * 32u * (uint32_t)sizeof(T);  // bytes between positions
#pragma unroll
        for (int t = 0; t < kBlkDW; ++t) {
            if (t >= m || (hints & 2u)) break;
            const T c = ar[pr[t] >> 20];
            const unsigned char* p = sb + (pr[t] & 0xfffffu);
            int o = 0;
#pragma unroll
            for (int L = 0; L < NL; ++L) {
                if (ord.pos[L] < P0 || ord.pos[L] >= P0 + CN) continue;
                const T x = *reinterpret_cast<const T*>(p + o * pstride);
                if (P == 0 && t == 0)
                    val[L] = row0 ? c : R::mul(c, x, ov);
                else
                    val[L] = R::mac(val[L], c, x, ov);
                ++o;
            }
        }
        // every load of the chunk feeds these accumulators
        uint32_t d = 0;
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            if (ord.pos[L] < P0 || ord.pos[L] >= P0 + CN) continue;
            d ^= *reinterpret_cast<const uint32_t*>(&val[L]);
        }
        blk_release<T, LC>(g, ti, nrows, hdr, rs, ring, prev, lane, (uint32_t)(d == 0x9e3779b9u) & rt_zero, hints);
        ++g;
    }
    // high terms: chunk (piece, l)
    const uint32_t rstride = 32u * (uint32_t)sizeof(T);
    for (int l = 0; l < f; ++l) {
        const T c = ar[h.hcol[l]];
        const uint32_t slot = g % kBlkSlots;
        blk_wait(&rs.full[slot], (g / kBlkSlots) & 1u, 3, ti, g);
        const unsigned char* sp =
            ring + slot * BlkChunks<T, LC>::kSlotBytes + (uint32_t)warp * rstride + (uint32_t)lane * (uint32_t)sizeof(T);
        T xs[CN];
#pragma unroll
        for (int o = 0; o < CN; ++o) xs[o] = *reinterpret_cast<const T*>(sp + o * nrows * rstride);
        blk_release<T, LC>(g, ti, nrows, hdr, rs, ring, prev, lane, loaded_dep(xs, CN, rt_zero), hints);
        ++g;
        if (hints & 1u) continue;
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
    constexpr int NL = 1 << LC;
    constexpr int RE = NL * 32;  // elements per row
    constexpr BlkOrder<LC> ord = blk_order<LC>();
    static_assert(RE * sizeof(T) == kBlkRowBytes, "row size");
    extern __shared__ __align__(128) unsigned char ring[];  // kBlkSlots chunk slots
    __shared__ BlkHdr hdr[kBlkHdrs];
    __shared__ __align__(8) BlkRingSh rs;
    __shared__ T arow[LC + 1][kMaxOrder];  // a(j + p - 1, .), p = 0 .. LC
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < kBlkSlots; ++s) {
            mbar_init(&rs.full[s], 1);
            rs.readers[s] = 0;
        }
        for (int s = 0; s < kBlkHdrs; ++s) {
            mbar_init(&rs.hdr_full[s], 1);
            mbar_init(&rs.hdr_empty[s], kBlkWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int e = threadIdx.x; e < (LC + 1) * n; e += blockDim.x) {
        const int p = e / n, c = e - p * n, row = j + p - 1;
        if (row >= 0 && row < n) arow[p][c] = a[(size_t)row * n + c];
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the previous super-layer is complete and visible
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncthreads();

    // publisher state (warp 3): the next tile to publish, its place in the chunk sequence
    uint32_t t_next = 0, F_next = 0, g_next = 0, pub = 0;
    bool pub_end = false;
    auto publish = [&]() {  // whole warp 3: header of tile `pub`
        if (pub_end) return;
        const uint32_t hs = pub % kBlkHdrs;
        if (pub >= (uint32_t)kBlkHdrs) blk_wait(&rs.hdr_empty[hs], ((pub / kBlkHdrs) - 1u) & 1u, 4, pub, 0u);
        const uint32_t t = __shfl_sync(0xffffffffu, t_next, 0);
        BlkHdr& h = hdr[hs];
        if (t >= ntiles) {
            if (lane == 0) {
                h.m = -1;
                h.g0 = g_next;
                h.nch = 0;
                __threadfence_block();
                mbar_arrive(&rs.hdr_full[hs]);
            }
            pub_end = true;
            ++pub;
            return;
        }
        const uint32_t F = __shfl_sync(0xffffffffu, F_next, 0);
        const int fr = __popc(F), mr = j - fr;
        const int f = fr, m = mr;
        if (lane < fr) {
            const int bit = __fns(F, 0, lane + 1);
            h.sb[lane] = __ldg(tb_prev + (F & ~(1u << bit)));
            h.hcol[lane] = (uint8_t)(LC + kBlkDW + bit);
        }
        const uint32_t nch = (uint32_t)kBlkPieces * (uint32_t)(f + (m >= 1 ? 1 : 0));
        if (lane == 0) {
            h.m = m;
            h.f = f;
            h.nb = blk_c9(mr);
            h.nrows = blk_rows9(mr);
            h.nsrc_rows = mr >= 1 ? blk_rows9(mr - 1) : 0u;
            h.cur_row = __ldg(tb_cur + F);
            h.src_row = mr >= 1 ? __ldg(tb_prev + F) : 0u;
            h.g0 = g_next;
            h.nch = nch;
            // claim the tile after
            t_next = atomicAdd(ticket, 1u);
            F_next = t_next < ntiles ? __ldg(flist + t_next) : 0u;
        }
        g_next += nch;
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            mbar_arrive(&rs.hdr_full[hs]);
        }
        ++pub;
    };
    if (warp == 3) {
        if (lane == 0) {
            t_next = atomicAdd(ticket, 1u);
            F_next = t_next < ntiles ? __ldg(flist + t_next) : 0u;
        }
        publish();
        publish();
        if (lane == 0) {  // start the ring
            for (uint32_t gi = 0; gi < (uint32_t)kBlkSlots; ++gi)
                blk_issue_chunk<T, LC>(gi, 0u, hdr, rs, ring, prev, hints);
        }
        __syncwarp();
    }

    bool ov = false;
    for (uint32_t ti = 0;; ++ti) {
        const uint32_t hs = ti % kBlkHdrs;
        blk_wait(&rs.hdr_full[hs], (ti / kBlkHdrs) & 1u, 5, ti, 0u);
        const BlkHdr& h = hdr[hs];
#ifdef PL_BLK_DEBUG
        if (lane == 0 && blockIdx.x == 0)
            printf("cta0 warp %d tile %u: m %d f %d nrows %u g0 %u nch %u\n", warp, ti, h.m, h.f, h.nrows, h.g0, h.nch);
#endif
        if (h.m < 0) break;
        if (warp == 3) publish();  // tile ti + 2
        if ((uint32_t)warp < h.nrows) {
            const int m = h.m, f = h.f;
            const uint32_t nb = h.nb, nrows = h.nrows;
            const uint32_t q = (uint32_t)warp * 32u + (uint32_t)lane;
            const bool valid = q < nb;
            const uint32_t qc = valid ? q : nb - 1u;
            uint32_t g = h.g0;
            uint32_t pr[kBlkDW];
            if (m >= 1) {
                const uint4 e = __ldg(wtab + blk_moff9(m) + qc);
                const uint64_t lo = e.x | (uint64_t)e.y << 32, hi = e.z | (uint64_t)e.w << 32;
#pragma unroll
                for (int t = 0; t < kBlkDW; ++t) {
                    const uint32_t fld = (uint32_t)((t < 5 ? lo >> (12 * t) : hi >> (12 * (t - 5))) & 0xfffu);
                    const uint32_t bi = fld & 127u, w = fld >> 7;  // block bi of the source tile: row bi / 32, lane bi % 32
                    pr[t] = (bi * (uint32_t)sizeof(T)) | (uint32_t)(LC + w) << 20;
                }
            } else {
#pragma unroll
                for (int t = 0; t < kBlkDW; ++t) pr[t] = 0;
            }
            T* dst = cur + (size_t)h.cur_row * RE + (size_t)warp * 32 + lane;
            T val[NL];
            auto store_level = [&](int P) {
                if (valid) {
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        if (__builtin_popcount(L) == P) dst[(size_t)ord.pos[L] * nrows * 32] = val[L];
                }
            };
#define PL_BLK_PIECE(P, O0, CN, R0)                                                                              \
    blk_piece<R, LC, P, O0, CN>(val, arow[P], R0, m, pr, f, h, ti, hdr, rs, ring, prev, g, warp, lane, hints, \
                                ov)
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
        } else {
            // no row in this tile: pass its chunks
            for (uint32_t g = h.g0; g != h.g0 + h.nch; ++g) {
                blk_wait(&rs.full[g % kBlkSlots], (g / kBlkSlots) & 1u, 6, ti, g);
                blk_release<T, LC>(g, ti, h.nrows, hdr, rs, ring, prev, lane, 0u, hints);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rs.hdr_empty[hs]);
    }
    if (ov) atomicOr(status, 1);
}

}  // namespace pl
