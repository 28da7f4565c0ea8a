// Warp-specialised per-layer kernel (the large-order hot path).
//
// Recurrence (reference proj/src/permanent.cpp:268-279):
//     per(S) = sum_{j in S, ascending} a(k-1, j) * per(S \ {j}),   |S| = k,
// evaluated one layer at a time, every layer dense in colex order.
//
// Tiling. Columns split into a low window [0, D) and high columns [D, n). For
// S = F u V (F = S n [D, n), |F| = f; V = S n [0, D), |V| = m)
//     rank(S) = rank_D(V) + sum_{l=1..f} C(F_l, m + l),
// so the k-subsets sharing F form one contiguous colex range, the tile (F, k),
// of C(D, m) entries indexed by q = rank_D(V). Output q needs
//   * low terms  S \ {v_i}: inside the tile (F, k-1), a small contiguous
//     region (<= C(D, D/2) entries) gathered through L1 (__ldg);
//     rank_D(V \ {v_i}) = P_i + Q_i (P_i = sum_{l<i} C(v_l, l),
//     Q_i = sum_{l>i} C(v_l, l-1)), one paired-binomial lookup per term;
//   * high terms S \ {F_l}: entry q of the tile (F \ {F_l}, k-1) -> aligned
//     contiguous streams with a tile-uniform coefficient, staged by TMA.
// Low columns are all below high columns, so "low ascending, then high
// ascending" is the reference's ascending-j order; the non-FMA rings keep its
// rounding sequence bit for bit.
//
// Schedule. One CTA per SM, persistent. CTA b takes the b-th, (b+G)-th, ...
// valid tile in increasing F (increasing colex order), so the GPU sweeps each
// layer front to back and stream tiles of nearby high columns are re-read
// from L2. Every warp walks the same tile sequence and derives each tile's
// descriptor itself: there is no per-tile synchronisation at all.
//
// Roles.
//   last warp, producer  streams the high-term segments of every chunk of CH
//                        outputs into the owning consumer group's NSG-stage
//                        shared-memory ring, FS segments per stage, one
//                        cp.async.bulk per segment, completion by mbarrier
//                        transaction counts (~160 KB in flight per SM). It is
//                        the highest warp id: the issue arbiter favours high
//                        ids over the consumers.
//   warps 0..15          two consumer groups of 8 warps taking alternate
//                        chunks, one output per thread: low terms (L1
//                        gathers), high terms from the group's ring, coalesced
//                        store. Each group owns its ring, so every waiter is
//                        at most one mbarrier phase ahead of the producer.
#pragma once

#include <cstdint>

#include "ring.cuh"

namespace pl {

constexpr int kWsGroupWarps = 8;
constexpr int kWsMaxGroups = 3;
constexpr int kWsLanes = 32 * kWsGroupWarps;   // consumer threads per group
constexpr int kWsPer = 2;                      // outputs per consumer thread per chunk (independent chains)
constexpr int kWsChunk = kWsLanes * kWsPer;    // CH: outputs per chunk
constexpr int kWsFS = 4;                      // stream segments per ring stage
constexpr int kQtabShift = 17;                // qtab entry: mask(V) | rank(V \ {min V}) << 17
constexpr int kWsEnd = -1;

// Window width D and ring depth per element size (shared memory <= 227 KB;
// what the ring leaves is L1 for the low-source gathers).
__host__ __device__ constexpr int ws_window(int elem_bytes) { return elem_bytes == 16 ? 17 : 17; }
// Consumer groups per CTA: three for 8-byte elements (more warps to hide the
// low-source gather latency); two for complex, whose arithmetic needs the
// registers.
template <int ELEM>
struct WsGeom {
    static constexpr int G = ELEM == 16 ? 2 : 3;             // consumer groups
    static constexpr int NSG = ELEM == 16 ? 2 : 4;           // stages per group ring (power of two)
    static constexpr int kConsumerWarps = kWsGroupWarps * G;
    static constexpr int kThreads = 32 * (1 + kConsumerWarps);
};

__host__ __device__ constexpr size_t round16(size_t b) { return (b + 15) & ~size_t(15); }

template <class T>
struct WsSmem {
    static constexpr int NSG = WsGeom<(int)sizeof(T)>::NSG;
    static constexpr int G = WsGeom<(int)sizeof(T)>::G;
    static constexpr int CW = WsGeom<(int)sizeof(T)>::kConsumerWarps;
    static constexpr size_t kSlot = round16(sizeof(T) * kWsChunk + 16) / sizeof(T);  // elements per segment slot
    uint2* B2;        // B2[i * kBinomDim + s] = (C(s, i), C(s, i - 1))
    T* row_low;       // [32]   a(k-1, v), v < D
    T* coef;          // [warps][kMaxOrder]  per-warp a(k-1, F_l) of the warp's current tile
    uint64_t* full;   // [G][NSG]
    uint64_t* empty;  // [G][NSG]
    T* stage;         // [G][NSG][FS][kSlot]

    __host__ __device__ static size_t bytes() {
        return round16(sizeof(uint2) * kBinomDim * kBinomDim) + round16(sizeof(T) * 32) +
               round16(sizeof(T) * kMaxOrder * (CW + 1)) + round16(8 * 2 * G * NSG) +
               round16((size_t)G * NSG * kWsFS * kSlot * sizeof(T));
    }
    __device__ explicit WsSmem(unsigned char* base) {
        size_t off = 0;
        auto take = [&](size_t b) {
            unsigned char* p = base + off;
            off += round16(b);
            return p;
        };
        B2 = reinterpret_cast<uint2*>(take(sizeof(uint2) * kBinomDim * kBinomDim));
        row_low = reinterpret_cast<T*>(take(sizeof(T) * 32));
        coef = reinterpret_cast<T*>(take(sizeof(T) * kMaxOrder * (CW + 1)));
        uint64_t* bars = reinterpret_cast<uint64_t*>(take(8 * 2 * G * NSG));
        full = bars;
        empty = bars + G * NSG;
        stage = reinterpret_cast<T*>(take((size_t)G * NSG * kWsFS * kSlot * sizeof(T)));
    }
    __device__ T* slot(int g, int s, int li) const { return stage + (((size_t)g * NSG + s) * kWsFS + li) * kSlot; }
    __device__ uint64_t* full_bar(int g, int s) const { return full + g * NSG + s; }
    __device__ uint64_t* empty_bar(int g, int s) const { return empty + g * NSG + s; }
    __device__ T* warp_coef(int w) const { return coef + (size_t)w * kMaxOrder; }
};

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA 1D bulk copy global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Same, with an L2 eviction-priority hint for the source lines.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// A run [start, start + len) of T staged by a 16-byte aligned bulk copy. For
// 8-byte T the copy starts at the aligned element below (pad = 1 when start
// is odd) and is rounded up to whole 16-byte units: it may read one element
// on either side of the run (layer buffers carry 16 bytes of slack).
template <class T>
struct BulkSpan {
    const T* src;
    unsigned bytes;
    int pad;
};

template <class T>
__device__ __forceinline__ BulkSpan<T> bulk_span(const T* base, uint64_t start, uint32_t len) {
    if constexpr (sizeof(T) == 16) {
        return {base + start, len * 16u, 0};
    } else {
        const uint64_t s0 = start & ~uint64_t(1);
        const int pad = (int)(start - s0);
        return {base + s0, ((len + pad + 1) & ~1u) * 8u, pad};
    }
}

// ---------------------------------------------------------------- tiles

struct WsTile {
    int32_t F, m, f;
    uint32_t q0, q1, nchunks;
    uint64_t cur_base, src_base;
};

// Next tile of this CTA's list, or kWsEnd. The host deals the layer's tiles,
// in increasing F, to the least-loaded CTA (load = chunks), so all CTAs sweep
// the layer as one tight front and the stream tiles of near high columns are
// still in L2 when they are re-read. Every warp walks the same list.
struct WsCursor {
    const uint32_t* list;
    uint32_t pos, end;
};

__device__ __forceinline__ WsCursor ws_cursor(const uint32_t* __restrict__ sched) {
    const uint32_t* off = sched;
    return {sched + gridDim.x + 1, __ldg(off + blockIdx.x), __ldg(off + blockIdx.x + 1)};
}

__device__ __forceinline__ int32_t ws_next(WsCursor& c) {
    if (c.pos >= c.end) return kWsEnd;
    return (int32_t)__ldg(c.list + c.pos++);
}

__device__ __forceinline__ WsTile ws_tile(int32_t F, int k, int D, uint64_t r0, uint64_t r1,
                                          const uint2* __restrict__ B2) {
    WsTile t;
    t.F = F;
    t.f = __popc((uint32_t)F);
    t.m = k - t.f;
    t.cur_base = 0;
    t.src_base = 0;
    int l = 1;
    for (uint32_t ff = (uint32_t)F; ff; ff &= ff - 1, ++l) {
        const int col = D + __ffs(ff) - 1;
        const uint2 b = B2[(t.m + l) * kBinomDim + col];
        t.cur_base += b.x;
        t.src_base += b.y;
    }
    const uint32_t len = B2[t.m * kBinomDim + D].x;
    t.q0 = r0 > t.cur_base ? (uint32_t)(r0 - t.cur_base) : 0u;
    t.q1 = (r1 - t.cur_base) < len ? (uint32_t)(r1 - t.cur_base) : len;
    t.nchunks = t.q1 > t.q0 ? (t.q1 - t.q0 + kWsChunk - 1) / kWsChunk : 0u;
    return t;
}

// Column of the l-th (0-based) high element of F.
__device__ __forceinline__ int ws_high_col(uint32_t F, int l, int D) {
    for (int i = 0; i < l; ++i) F &= F - 1;
    return D + __ffs(F) - 1;
}

// Base rank, in the previous layer, of the stream tile (F \ {F_l}, k-1): the
// remaining high elements keep the low count m and shift down one position.
__device__ __forceinline__ uint64_t ws_stream_base(uint32_t F, int l, int m, int D, const uint2* __restrict__ B2) {
    uint64_t b = 0;
    int i = 0, p = 1;
    for (uint32_t ff = F; ff; ff &= ff - 1, ++i) {
        if (i == l) continue;
        b += B2[(m + p) * kBinomDim + D + __ffs(ff) - 1].x;
        ++p;
    }
    return b;
}

// ---------------------------------------------------------------- consumer math

// Low-source gathers: the tile's source region is re-read for the whole life of
// the tile, so its lines are kept in L2 with an evict-last policy.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

template <class T>
__device__ __forceinline__ T ldg_keep(const T* p, uint64_t pol) {
    if constexpr (sizeof(T) == 16) {
        double2 v;
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n"
                     : "=d"(v.x), "=d"(v.y)
                     : "l"(p), "l"(pol));
        return *reinterpret_cast<T*>(&v);
    } else {
        unsigned long long v;
        asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;\n" : "=l"(v) : "l"(p), "l"(pol));
        return *reinterpret_cast<T*>(&v);
    }
}

template <class T>
__device__ __forceinline__ void stg_hint(T* p, const T& v, uint64_t pol) {
    if constexpr (sizeof(T) == 16) {
        const double2 d = *reinterpret_cast<const double2*>(&v);
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(d.x), "d"(d.y), "l"(pol)
                     : "memory");
    } else {
        const unsigned long long d = *reinterpret_cast<const unsigned long long*>(&v);
        asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;\n" ::"l"(p), "l"(d), "l"(pol) : "memory");
    }
}

template <class RR, int M, class T>
__device__ __forceinline__ T ws_low(uint32_t e, const T* __restrict__ src, const T* __restrict__ row_low,
                                    const uint2* __restrict__ B2, uint64_t pol, bool& ov) {
    uint32_t V = e & ((1u << kQtabShift) - 1);
    uint32_t Q = e >> kQtabShift, P = 0;
    int sv[M];
    uint32_t pr[M];
#pragma unroll
    for (int i = 1; i <= M; ++i) {
        const int s = __ffs(V) - 1;
        V &= V - 1;
        const uint2 b = B2[i * kBinomDim + s];  // (C(s, i), C(s, i-1))
        if (i >= 2) Q -= b.y;
        sv[i - 1] = s;
        pr[i - 1] = P + Q;
        P += b.x;
    }
    T x[M];
#pragma unroll
    for (int i = 0; i < M; ++i) x[i] = ldg_keep(src + pr[i], pol);
    T acc = RR::mul(row_low[sv[0]], x[0], ov);
#pragma unroll
    for (int i = 1; i < M; ++i) acc = RR::mac(acc, row_low[sv[i]], x[i], ov);
    return acc;
}

template <class RR, class T>
__device__ __forceinline__ T ws_low_dispatch(int m, uint32_t e, const T* src, const T* row_low, const uint2* B2,
                                             uint64_t pol, bool& ov) {
    switch (m) {
#define PL_WS_CASE(M) \
    case M:           \
        return ws_low<RR, M>(e, src, row_low, B2, pol, ov);
        PL_WS_CASE(1) PL_WS_CASE(2) PL_WS_CASE(3) PL_WS_CASE(4) PL_WS_CASE(5) PL_WS_CASE(6) PL_WS_CASE(7)
        PL_WS_CASE(8) PL_WS_CASE(9) PL_WS_CASE(10) PL_WS_CASE(11) PL_WS_CASE(12) PL_WS_CASE(13) PL_WS_CASE(14)
        PL_WS_CASE(15) PL_WS_CASE(16) PL_WS_CASE(17)
#undef PL_WS_CASE
    }
    return RR::zero();
}

// One ring stage's high terms for output j (a full stage needs no predicates).
template <class RR, class T>
__device__ __forceinline__ T ws_stage_terms(T acc, const WsSmem<T>& sm, const T* __restrict__ coef, int g, int s,
                                            int l0, int nl, const int* __restrict__ pads, int j, bool init_first,
                                            bool& ov) {
    const T* st = sm.slot(g, s, 0) + j;
    if (nl == kWsFS && !init_first) {
#pragma unroll
        for (int li = 0; li < kWsFS; ++li) acc = RR::mac(acc, coef[l0 + li], st[li * WsSmem<T>::kSlot + pads[li]], ov);
        return acc;
    }
#pragma unroll
    for (int li = 0; li < kWsFS; ++li) {
        if (li < nl) {
            const T x = st[li * WsSmem<T>::kSlot + pads[li]];
            acc = (init_first && li == 0) ? RR::mul(coef[l0 + li], x, ov) : RR::mac(acc, coef[l0 + li], x, ov);
        }
    }
    return acc;
}

// Consumer group g's share of one tile: chunks c0g, c0g + G, ... (chunks are
// dealt to groups round-robin over the CTA's whole tile sequence, so tiles of
// a single chunk alternate between groups). Each of
// its chunks takes ceil(f / FS) consecutive stages of the group's own ring;
// `seq` is the group's running stage counter (stage seq % NSG, use seq / NSG).
template <class RR, class T>
__device__ __forceinline__ void ws_consume_tile(const WsSmem<T>& sm, const WsTile& t, const T* __restrict__ src,
                                                const T* __restrict__ coef, const uint64_t* __restrict__ sbase_pad,
                                                const uint32_t* __restrict__ qt, T* __restrict__ cur, int g, int j,
                                                uint32_t c_first, uint32_t& seq, bool& ov, bool store_first) {
    constexpr int NSG = WsSmem<T>::NSG;
    const int m = t.m, f = t.f;
    const uint64_t keep = l2_evict_last_policy();
    const uint64_t pol_store = l2_evict_first_policy();
    uint32_t c = c_first;
    // each thread owns outputs j and j + kWsLanes of every chunk: two independent
    // accumulation chains; qtab entries are prefetched one chunk ahead
    uint32_t e_next[kWsPer] = {};
    if (m >= 1 && c < t.nchunks) {
#pragma unroll
        for (int p = 0; p < kWsPer; ++p) e_next[p] = __ldg(qt + min(t.q0 + c * kWsChunk + j + p * kWsLanes, t.q1 - 1));
    }
    constexpr int G = WsSmem<T>::G;
    for (; c < t.nchunks; c += G) {
        const uint32_t c0 = t.q0 + c * kWsChunk;
        const uint32_t len = min((uint32_t)kWsChunk, t.q1 - c0);
        // Lanes past the tile end compute a duplicate of its last output
        // (no divergence); only their store and overflow flag are dropped.
        uint32_t e[kWsPer];
#pragma unroll
        for (int p = 0; p < kWsPer; ++p) e[p] = e_next[p];
        if (m >= 1 && c + G < t.nchunks) {
#pragma unroll
            for (int p = 0; p < kWsPer; ++p)
                e_next[p] = __ldg(qt + min(c0 + G * kWsChunk + j + p * kWsLanes, t.q1 - 1));
        }
        bool lov[kWsPer];
        T acc[kWsPer];
#pragma unroll
        for (int p = 0; p < kWsPer; ++p) {
            lov[p] = false;
            acc[p] = RR::zero();
            if (m >= 1) acc[p] = ws_low_dispatch<RR>(m, e[p], src, sm.row_low, sm.B2, keep, lov[p]);
        }
        for (int l0 = 0; l0 < f; l0 += kWsFS, ++seq) {
            const int nl = min(kWsFS, f - l0);
            int pads[kWsFS];
#pragma unroll
            for (int li = 0; li < kWsFS; ++li) {
                pads[li] = sizeof(T) == 16 || li >= nl ? 0 : (int)((sbase_pad[l0 + li] + c0) & 1u);
            }
            const int s = (int)(seq % NSG);
            mbar_wait(sm.full_bar(g, s), (seq / NSG) & 1u);
#pragma unroll
            for (int p = 0; p < kWsPer; ++p)
                acc[p] = ws_stage_terms<RR>(acc[p], sm, coef, g, s, l0, nl, pads, j + p * kWsLanes, m == 0 && l0 == 0,
                                            lov[p]);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(sm.empty_bar(g, s));
        }
#pragma unroll
        for (int p = 0; p < kWsPer; ++p) {
            if ((uint32_t)(j + p * kWsLanes) < len) {
                if (store_first)
                    stg_hint(cur + t.cur_base + c0 + j + p * kWsLanes, acc[p], pol_store);
                else
                    cur[t.cur_base + c0 + j + p * kWsLanes] = acc[p];
                ov |= lov[p];  // duplicates past the tile end never report
            }
        }
    }
}

// ---------------------------------------------------------------- kernel

template <class R, class RU>
__global__ void __launch_bounds__(WsGeom<(int)sizeof(typename R::T)>::kThreads, 1)
    sz_ws_kernel(const typename R::T* __restrict__ a, int n, int k, int D, const typename R::T* __restrict__ prev,
                 typename R::T* __restrict__ cur, uint64_t r0, uint64_t r1, const uint32_t* __restrict__ sched,
                 const uint32_t* __restrict__ qtab, const uint32_t* __restrict__ qtab_off,
                 const uint2* __restrict__ binom_pairs, const int32_t* __restrict__ guard,
                 int32_t* __restrict__ status, uint32_t hints) {
    using T = typename R::T;
    constexpr int NSG = WsSmem<T>::NSG;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t sbase_sh[kWsGroupWarps * kWsMaxGroups + 1][kMaxOrder];  // per-warp stream bases (8-byte pads)
    constexpr int G = WsSmem<T>::G;
    constexpr int CW = WsSmem<T>::CW;
    const WsSmem<T> sm(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* row = a + (size_t)(k - 1) * n;

    for (int e = threadIdx.x; e < kBinomDim * kBinomDim; e += blockDim.x) sm.B2[e] = __ldg(&binom_pairs[e]);
    for (int v = threadIdx.x; v < D; v += blockDim.x) sm.row_low[v] = row[v];
    if (threadIdx.x == 0) {
        for (int s = 0; s < G * NSG; ++s) {
            mbar_init(&sm.full[s], 1);               // producer's arrive.expect_tx
            mbar_init(&sm.empty[s], kWsGroupWarps);  // the owning group's warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    WsCursor cursor = ws_cursor(sched);
    if (warp == CW) {
        // ------------------------------------------------------------ producer
        uint32_t seqg[G] = {};
        uint32_t gchunk = 0;  // running chunk counter over the tile sequence
        const uint64_t pol_first = l2_evict_first_policy(), pol_last = l2_evict_last_policy();
        for (int32_t F = ws_next(cursor); F != kWsEnd; F = ws_next(cursor)) {
            const WsTile t = ws_tile(F, k, D, r0, r1, sm.B2);
            // lane l holds the base of stream tile F \ {F_l}
            const uint64_t my_base = lane < t.f ? ws_stream_base((uint32_t)F, lane, t.m, D, sm.B2) : 0;
            // and its L2 policy: the next read of tile F' = F \ {F_l} in this layer comes from
            // F' + 2^h2 (h2 = lowest free high column above F_l); beyond the reuse horizon the
            // lines are marked evict-first so they do not displace tiles with near reuse.
            int my_mode = 0;  // 0 plain, 1 evict_first, 2 evict_last
            if ((hints & 3u) != 0 && lane < t.f) {
                const int H = n - D;
                const int h = ws_high_col((uint32_t)F, lane, D) - D;
                const uint32_t Fp = (uint32_t)F & ~(1u << h);
                const uint32_t z = ~Fp & ((1u << H) - 1u) & ~((2u << h) - 1u);
                bool far = true;
                if (z != 0) {
                    const int h2 = __ffs(z) - 1;
                    far = ((1u << h2) - (1u << h)) > (1u << ((hints >> 8) & 31u));
                }
                my_mode = far ? 1 : ((hints & 3u) == 2 ? 2 : 0);
            }
            int g = (int)(gchunk % G);
            for (uint32_t c = 0; c < t.nchunks; ++c, g = (g + 1 == G) ? 0 : g + 1) {
                const uint32_t c0 = t.q0 + c * kWsChunk;
                const uint32_t len = min((uint32_t)kWsChunk, t.q1 - c0);
                for (int l0 = 0; l0 < t.f; l0 += kWsFS) {
                    const int nl = min(kWsFS, t.f - l0);
                    const uint64_t base = __shfl_sync(0xffffffffu, my_base, (l0 + lane) & 31);
                    const int mode = __shfl_sync(0xffffffffu, my_mode, (l0 + lane) & 31);
                    const uint32_t sq = seqg[g]++;
                    const int s = (int)(sq % NSG);
                    mbar_wait(sm.empty_bar(g, s), ((sq / NSG) & 1u) ^ 1u);
                    BulkSpan<T> seg{prev, 0u, 0};
                    if (lane < nl) seg = bulk_span(prev, base + c0, len);
                    const unsigned total = __reduce_add_sync(0xffffffffu, seg.bytes);
                    if (lane == 0) mbar_arrive_expect_tx(sm.full_bar(g, s), total);
                    __syncwarp();
                    if (lane < nl) {
                        if (mode == 0)
                            bulk_g2s(sm.slot(g, s, lane), seg.src, seg.bytes, sm.full_bar(g, s));
                        else
                            bulk_g2s_hint(sm.slot(g, s, lane), seg.src, seg.bytes, sm.full_bar(g, s),
                                          mode == 1 ? pol_first : pol_last);
                    }
                }
            }
            gchunk += t.nchunks;
        }
    } else {
        // ------------------------------------------------------------ consumers
        const int g = warp / kWsGroupWarps;
        const int j = (warp % kWsGroupWarps) * 32 + lane;
        T* coef = sm.warp_coef(warp);
        uint64_t* sb = sbase_sh[warp];
        bool use_checked = false;
        if constexpr (R::kChecked) use_checked = guard != nullptr && guard[0] != 0;
        bool ov = false;
        const bool store_first = (hints & 4u) != 0;
        uint32_t seq = 0, gchunk = 0;
        for (int32_t F = ws_next(cursor); F != kWsEnd; F = ws_next(cursor)) {
            const WsTile t = ws_tile(F, k, D, r0, r1, sm.B2);
            // this group's first chunk of the tile; skip tiles with none (no stages either)
            const uint32_t c_first = (uint32_t)((g - (int)(gchunk % G) + G) % G);
            gchunk += t.nchunks;
            if (c_first >= t.nchunks) continue;
            __syncwarp();
            if (lane < t.f) {
                coef[lane] = row[ws_high_col((uint32_t)F, lane, D)];
                if constexpr (sizeof(T) != 16) sb[lane] = ws_stream_base((uint32_t)F, lane, t.m, D, sm.B2);
            }
            __syncwarp();
            const uint32_t* qt = qtab + qtab_off[t.m];
            const T* src = prev + t.src_base;
            if constexpr (R::kChecked) {
                if (use_checked) {
                    ws_consume_tile<R>(sm, t, src, coef, sb, qt, cur, g, j, c_first, seq, ov, store_first);
                } else {
                    ws_consume_tile<RU>(sm, t, src, coef, sb, qt, cur, g, j, c_first, seq, ov, store_first);
                }
            } else {
                ws_consume_tile<R>(sm, t, src, coef, sb, qt, cur, g, j, c_first, seq, ov, store_first);
            }
        }
        if (ov) atomicOr(status, 1);
    }
}

}  // namespace pl
