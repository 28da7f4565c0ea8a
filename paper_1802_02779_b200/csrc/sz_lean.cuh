// Lean per-layer kernel (round 2): the same tiling as sz_ws.cuh, with the
// high-term streams read straight from global memory instead of being staged
// through shared-memory rings.
//
// Recurrence (reference proj/src/permanent.cpp:164-175):
//     per(S) = sum_{j in S, ascending} a(k-1, j) * per(S \ {j}),   |S| = k.
// Tiling (see sz_ws.cuh): columns [0, D) low, [D, n) high; the k-subsets
// S = F u V sharing their high part F form the contiguous tile (F, k) of
// C(D, m) entries (m = |V|). Output q of the tile needs
//   * m low terms from the tile's low source X(F, k-1) (C(D, m-1) entries,
//     staged whole in shared memory by one bulk copy, gathered through the
//     low-term table ltab: rank_D(V \ {v_i}) | v_i << 12);
//   * f = |F| high terms: entry q of the stream tile X(F \ {F_l}, k-1), times
//     the tile-uniform coefficient a(k-1, F_l) -- aligned with the output, so
//     a warp's 32 consecutive outputs read 32 consecutive entries (one
//     coalesced load per term).
// Low columns come before high columns, so "low ascending, then high
// ascending" is the reference's ascending-j order; the non-FMA rings keep its
// rounding sequence bit for bit.
//
// Why a second kernel. The warp-specialised kernel stages every stream
// segment by TMA into a shared-memory ring and hands it to the consumers
// through mbarriers; per term that is a bulk copy share, a wait/arrive share,
// a shared load and the hand-back dependency -- ~20 issued instructions per
// term for 8-byte rings (profiles/r1l_full_c4.md: DMUL+DADD 8 % of the
// instructions). Here a high term is one global load (L2 for layers that fit
// it, HBM otherwise), one broadcast shared load of the coefficient and the
// arithmetic; loads of a whole batch of terms are issued before the first
// product, so a thread keeps 8 (16 with two outputs) loads in flight.
//
// Schedule. Persistent CTAs (several per SM); CTA b takes tiles b, b + G,
// b + 2G, ... of the layer's tile list (increasing F: the GPU sweeps the
// layer as one front, so stream tiles of nearby high columns are re-read from
// L2). One producer warp per CTA builds the next tile's header (two warp
// scans) and stages its low source while the consumer warps compute the
// current tile; one CTA barrier per tile swaps the two slots. Programmatic
// dependent launch overlaps the prologue with the previous layer.
#pragma once

#include <cstdint>

#include "ring.cuh"
#include "sz_ws.cuh"

namespace pl {

#ifndef PL_LN_D
#define PL_LN_D 10
#endif
#ifndef PL_LN_WPB16
#define PL_LN_WPB16 10
#endif
#ifndef PL_LN_WPB8
#define PL_LN_WPB8 16
#endif
#ifndef PL_LN_MINB16
#define PL_LN_MINB16 2
#endif
#ifndef PL_LN_MINB8
#define PL_LN_MINB8 2
#endif
#ifndef PL_LN_PER16
#define PL_LN_PER16 1
#endif
#ifndef PL_LN_PER8
#define PL_LN_PER8 2
#endif
#ifndef PL_LN_BATCH16
#define PL_LN_BATCH16 4
#endif
#ifndef PL_LN_BATCH8
#define PL_LN_BATCH8 4
#endif

constexpr int kLnMaxD = PL_LN_D;  // low window of the lean kernel (compact ltab, source slot)

template <int ELEM>
struct LnGeom {
    static constexpr int WPB = ELEM == 16 ? PL_LN_WPB16 : PL_LN_WPB8;     // warps per CTA (each its own tiles)
    static constexpr int kThreads = 32 * WPB;
    static constexpr int kMinBlocks = ELEM == 16 ? PL_LN_MINB16 : PL_LN_MINB8;
    static constexpr int PER = ELEM == 16 ? PL_LN_PER16 : PL_LN_PER8;     // outputs per lane per pass
    static constexpr int B = ELEM == 16 ? PL_LN_BATCH16 : PL_LN_BATCH8;   // high-term loads per batch
    // source slot: C(D, D/2) entries + 8-byte alignment pad, rounded to 16 bytes
    static constexpr int kSrcSlot =
        (int)((binom_u64(kLnMaxD, kLnMaxD / 2) + 2 + 16 / ELEM - 1) / (16 / ELEM) * (16 / ELEM));
};

template <class T>
struct LnHdr {
    int32_t m, f;               // m < 0: no more tiles for this warp
    uint32_t q0, q1;            // this range's outputs of the tile: [q0, q1)
    T* out;                     // cur + rank of the tile's first output
    const uint4* lt;            // compact ltab rows of the m-subsets
    uint32_t pad_src;           // 8-byte rings: element offset of the source in its slot
    int32_t checked;            // int64: this matrix needs checked arithmetic (its guard flag)
    T rowlow[kLnMaxD];          // a(k-1, v), v < D, of the tile's matrix
    T coef[kWsMaxHigh];         // a(k-1, F_l)
    const T* sptr[kWsMaxHigh];  // prev + base rank of stream tile (F \ {F_l}, k-1)
};

// Per-warp state: two source slots, two headers, two transaction barriers.
template <class T>
struct alignas(16) LnWarp {
    static constexpr int kSlot = LnGeom<(int)sizeof(T)>::kSrcSlot;
    alignas(16) T src[2][kSlot];  // bulk-copy destinations: 16-byte aligned
    LnHdr<T> hdr[2];
    uint64_t full[2];
};

template <class T>
struct LnSmem {
    uint2 B2[kBinomDim * kBinomDim];  // (C(s, i), C(s, i - 1)) at [i * 35 + s]
    LnWarp<T> w[LnGeom<(int)sizeof(T)>::WPB];
};

// Compact low-term table: for the m-subset V of [0, D) of colex rank q, its m
// entries rank_D(V \ {v_i}) | v_i << 12 (ascending v_i) as u16, in one uint4
// (m <= 8) or two (m > 8) at ltab[off[m] + q * (m <= 8 ? 1 : 2)].
template <int M>
__device__ __forceinline__ void ln_ltab(const uint4* __restrict__ lt, uint32_t q, uint4& ea, uint4& eb) {
    if constexpr (M == 0) {
        ea = eb = make_uint4(0, 0, 0, 0);
    } else if constexpr (M <= 8) {
        ea = __ldg(lt + q);
        eb = make_uint4(0, 0, 0, 0);
    } else {
        ea = __ldg(lt + 2 * q);
        eb = __ldg(lt + 2 * q + 1);
    }
}

template <class T>
__device__ __forceinline__ T ln_load_stream(const T* p) {
    // stream tiles are read once per output tile: keep them out of L1
    if constexpr (sizeof(T) == 16) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
        return *reinterpret_cast<const T*>(&v);
    } else {
        const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(p));
        return *reinterpret_cast<const T*>(&v);
    }
}

// Low terms of PER outputs (m = M compile-time: the term loop unrolls).
template <class RR, int M, int PER, class T>
__device__ __forceinline__ void ln_low(const T* __restrict__ row, const uint4* __restrict__ lt,
                                       const T* __restrict__ src, const uint32_t (&q)[PER], T (&acc)[PER],
                                       bool (&lov)[PER]) {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        uint4 ea, eb;
        ln_ltab<M>(lt, q[p], ea, eb);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const uint32_t e = ltab_entry(ea, eb, i);
            const T x = src[e & ((1u << kWsLtabRankBits) - 1)];
            const T c = row[e >> kWsLtabRankBits];
            acc[p] = i == 0 ? RR::mul(c, x, lov[p]) : RR::mac(acc[p], c, x, lov[p]);
        }
    }
}

template <class RR, int PER, class T>
__device__ __forceinline__ void ln_low_dispatch(int m, const T* row, const uint4* lt, const T* src,
                                                const uint32_t (&q)[PER], T (&acc)[PER], bool (&lov)[PER]) {
    switch (m) {
#define PL_LN_LOW(M)                                          \
    case M:                                                   \
        ln_low<RR, M, PER>(row, lt, src, q, acc, lov);        \
        break;
        PL_LN_LOW(1) PL_LN_LOW(2) PL_LN_LOW(3) PL_LN_LOW(4) PL_LN_LOW(5) PL_LN_LOW(6)
#if PL_LN_D >= 7
        PL_LN_LOW(7)
#endif
#if PL_LN_D >= 8
        PL_LN_LOW(8)
#endif
#if PL_LN_D >= 9
        PL_LN_LOW(9)
#endif
#if PL_LN_D >= 10
        PL_LN_LOW(10)
#endif
#if PL_LN_D >= 11
        PL_LN_LOW(11)
#endif
#if PL_LN_D >= 12
        PL_LN_LOW(12)
#endif
#undef PL_LN_LOW
        default:
            break;
    }
}

// The outputs of one tile, by one warp: lane handles q = q0 + lane + 32 p + 32 PER i.
// Only the low-term loop is specialised per m (a small switch per pass): the
// kernel stays a few KB of code, so warps on tiles of different m do not
// evict each other from the instruction cache.
template <class RR, class T>
__device__ __forceinline__ void ln_tile(const T* __restrict__ row, const LnHdr<T>& h, const T* __restrict__ src,
                                        int lane, bool& ov) {
    constexpr int PER = LnGeom<(int)sizeof(T)>::PER;
    constexpr int B = LnGeom<(int)sizeof(T)>::B;
    const int f = h.f, m = h.m;
    const uint32_t q0 = h.q0, q1 = h.q1;
    const uint4* lt = h.lt;
    T* out = h.out;
    for (uint32_t qb = q0; qb < q1; qb += 32 * PER) {
        uint32_t q[PER];
        bool live[PER];
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const uint32_t qq = qb + lane + 32 * p;
            live[p] = qq < q1;
            q[p] = live[p] ? qq : q1 - 1;  // dead lanes recompute the last output, store nothing
        }
        T acc[PER];
        bool lov[PER];
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            lov[p] = false;
            acc[p] = RR::zero();
        }
        // the first batch of high-term loads is in flight during the low terms
        const int nb0 = f < B ? f : B;
        T y[PER][B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
            if (i < nb0) {
                const T* sp = h.sptr[i];
#pragma unroll
                for (int p = 0; p < PER; ++p) y[p][i] = ln_load_stream(sp + q[p]);
            }
        }
        ln_low_dispatch<RR, PER>(m, row, lt, src, q, acc, lov);
        int l = 0;
        for (;;) {
            const int nb = f - l < B ? f - l : B;
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (i < nb) {
                    const T c = h.coef[l + i];
#pragma unroll
                    for (int p = 0; p < PER; ++p)
                        acc[p] = (m == 0 && l + i == 0) ? RR::mul(c, y[p][i], lov[p])
                                                         : RR::mac(acc[p], c, y[p][i], lov[p]);
                }
            }
            l += B;
            if (l >= f) break;
            const int nn = f - l < B ? f - l : B;
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (i < nn) {
                    const T* sp = h.sptr[l + i];
#pragma unroll
                    for (int p = 0; p < PER; ++p) y[p][i] = ln_load_stream(sp + q[p]);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            if (live[p]) {
                out[q[p]] = acc[p];
                ov |= lov[p];
            }
        }
    }
}

// Header of tile t (or the end marker) into the warp's slot s; the tile's low
// source staged by one bulk copy completing on the slot's barrier. Returns
// false when the tile has no outputs in [r0, r1) (nothing armed).
// Batched form: tile t of the launch is tile t % ntiles of matrix t / ntiles
// (matrices n x n contiguous from `a`, their layer buffers `lstride`
// elements apart); a single matrix is nmat = 1.
template <class T>
__device__ __forceinline__ bool ln_prepare(LnSmem<T>& sm, LnWarp<T>& w, int s, uint64_t t, uint32_t ntiles,
                                           uint64_t total, const uint32_t* __restrict__ flist, const T* __restrict__ a,
                                           int n, int k, int D, int H, const T* __restrict__ prev_all,
                                           T* __restrict__ cur_all, uint64_t lstride, uint64_t r0, uint64_t r1,
                                           const uint4* __restrict__ ltab, const uint32_t* __restrict__ ltab_off,
                                           const int32_t* __restrict__ guard, int tcut, int lane) {
    LnHdr<T>& h = w.hdr[s];
    if (t >= total) {
        if (lane == 0) {
            h.m = -1;
            mbar_arrive(&w.full[s]);
        }
        __syncwarp();
        return true;
    }
    const uint64_t b = t / ntiles;
    const T* prev = prev_all + b * lstride;
    T* cur = cur_all + b * lstride;
    const T* arow = a + (b * (uint64_t)n + (uint64_t)(k - 1)) * (uint64_t)n;
    const uint32_t F = __ldg(flist + (t - b * ntiles));
    const int f = __popc(F), m = k - f;
    const bool set = lane < H && ((F >> lane) & 1u);
    const int idx = __popc(F & ((1u << lane) - 1u));
    uint64_t x = 0, y = 0;
    if (set) {
        const uint2 b = sm.B2[(m + idx + 1) * kBinomDim + D + lane];  // (C(D+h, m+l), C(D+h, m+l-1))
        x = b.x;
        y = b.y;
    }
    const uint64_t ixy = warp_scan_u64(x | y << 32);  // both prefix sums (ranks < 2^32)
    const uint64_t ix = ixy & 0xffffffffull, iy = ixy >> 32;
    const uint64_t last = __shfl_sync(0xffffffffu, ixy, 31);
    const uint64_t cur_base = last & 0xffffffffull;
    const uint64_t src_base = last >> 32;
    const uint32_t len = sm.B2[m * kBinomDim + D].x;
    const uint32_t q0 = r0 > cur_base ? (uint32_t)(r0 - cur_base) : 0u;
    const uint32_t q1 = (r1 - cur_base) < len ? (uint32_t)(r1 - cur_base) : len;
    if (q1 <= q0) return false;
    if (set) {
        h.coef[idx] = arow[D + lane];
        h.sptr[idx] = prev + ((ix - x) + (src_base - iy));
    }
    if (lane < D) h.rowlow[lane] = arow[lane];
    if (lane == 0) {
        h.checked = guard != nullptr ? guard[b] : 0;
        h.m = m;
        // tcut > 0: a partial layer without the top `tcut` columns' terms (see sz_ws.cuh)
        h.f = tcut ? __popc(F & ((1u << (H - tcut)) - 1u)) : f;
        h.q0 = q0;
        h.q1 = q1;
        h.out = cur + cur_base;
        h.lt = ltab + __ldg(ltab_off + m);
        h.pad_src = sizeof(T) == 16 ? 0u : (uint32_t)(src_base & 1u);
    }
    __syncwarp();
    if (lane == 0) {
        const uint32_t slen = m >= 1 ? sm.B2[(m - 1) * kBinomDim + D].x : 0u;
        const BulkSpan<T> sp = slen ? bulk_span(prev, src_base, slen) : BulkSpan<T>{prev, 0u, 0};
        mbar_arrive_expect_tx(&w.full[s], sp.bytes);
        if (sp.bytes) bulk_g2s(w.src[s], sp.src, sp.bytes, &w.full[s]);
    }
    __syncwarp();
    return true;
}

template <class R, class RU>
__global__ void __launch_bounds__(LnGeom<(int)sizeof(typename R::T)>::kThreads,
                                  LnGeom<(int)sizeof(typename R::T)>::kMinBlocks)
    sz_lean_kernel(const typename R::T* __restrict__ a, int n, int k, int D, const typename R::T* __restrict__ prev,
                   typename R::T* __restrict__ cur, uint64_t r0, uint64_t r1, const uint32_t* __restrict__ flist,
                   uint32_t ntiles, uint32_t nmat, uint64_t lstride, const uint4* __restrict__ ltab,
                   const uint32_t* __restrict__ ltab_off, const uint2* __restrict__ binom_pairs,
                   const int32_t* __restrict__ guard, int32_t* __restrict__ status, int top_cut) {
    using T = typename R::T;
    constexpr int WPB = LnGeom<(int)sizeof(T)>::WPB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LnSmem<T>& sm = *reinterpret_cast<LnSmem<T>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    LnWarp<T>& w = sm.w[warp];

    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (int e = threadIdx.x; e < kBinomDim * kBinomDim; e += blockDim.x) sm.B2[e] = __ldg(&binom_pairs[e]);
    if (lane == 0) {
        mbar_init(&w.full[0], 1);
        mbar_init(&w.full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the previous layer is complete and visible
    // generic-proxy stores of the previous layer, read below by bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncthreads();

    bool ov = false;
    const int H = n - D;
    const uint64_t total = (uint64_t)ntiles * nmat;
    // warp gw takes tiles gw, gw + W, gw + 2W, ... (increasing F: one sweep front)
    const uint64_t W = (uint64_t)gridDim.x * WPB;
    uint64_t t = (uint64_t)blockIdx.x * WPB + warp;
    auto prep = [&](int slot) {
        return ln_prepare(sm, w, slot, t, ntiles, total, flist, a, n, k, D, H, prev, cur, lstride, r0, r1, ltab,
                          ltab_off, guard, top_cut, lane);
    };
    while (!prep(0)) t += W;
    for (uint32_t it = 0;; ++it) {
        const int s = (int)(it & 1u);
        if (t < total) {
            // next tile into the other slot (last read by this warp's previous tile)
            do {
                t += W;
            } while (!prep(s ^ 1));
        }
        mbar_wait(&w.full[s], (it >> 1) & 1u);
        const LnHdr<T>& h = w.hdr[s];
        if (h.m < 0) break;
        const T* src = w.src[s] + h.pad_src;
        if constexpr (R::kChecked) {
            if (h.checked)
                ln_tile<R>(h.rowlow, h, src, lane, ov);
            else
                ln_tile<RU>(h.rowlow, h, src, lane, ov);
        } else {
            ln_tile<R>(h.rowlow, h, src, lane, ov);
        }
        __syncwarp();
    }
    if (ov) atomicOr(status, 1);
}

}  // namespace pl
