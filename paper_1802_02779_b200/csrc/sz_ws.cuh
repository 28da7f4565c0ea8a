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
//   * low terms  S \ {v_i}: inside the tile (F, k-1) -> staged in shared memory,
//     rank_D(V \ {v_i}) = P_i + Q_i (P_i = sum_{l<i} C(v_l, l),
//     Q_i = sum_{l>i} C(v_l, l-1)), one paired-binomial lookup per term;
//   * high terms S \ {F_l}: entry q of the tile (F \ {F_l}, k-1) -> aligned
//     contiguous streams with a tile-uniform coefficient.
// Low columns are all below high columns, so "low ascending, then high
// ascending" is the reference's ascending-j order; the non-FMA rings keep its
// rounding sequence bit for bit.
//
// Roles (one CTA per SM, persistent):
//   warp 0, producer    claims tiles in increasing F (atomic counter: the GPU
//                       sweeps each layer front to back, so stream tiles of
//                       nearby high columns are re-read from L2), writes tile
//                       descriptors, stages each tile's low source with one
//                       TMA bulk copy into a double buffer (the next tile's
//                       source is issued as soon as its buffer frees, while
//                       the current tile still streams), and streams the
//                       high-term segments of every chunk of CH outputs into
//                       the owning group's NSG-stage ring, FS segments per stage, one
//                       cp.async.bulk per segment, completion by mbarrier
//                       transaction counts (~100 KB per SM in flight);
//   warps 1..16         two consumer groups of 8 warps taking alternate chunks
//                       (one output per thread): low terms from the staged
//                       source, high terms from the group's ring, coalesced
//                       store. Each group owns its ring, so every waiter is at
//                       most one mbarrier phase ahead of the producer (a ring
//                       shared by groups that run ahead of each other would
//                       let parity waits pass a phase early).
#pragma once

#include <cstdint>

#include "ring.cuh"

namespace pl {

constexpr int kWsGroupWarps = 8;
constexpr int kWsGroups = 2;
constexpr int kWsConsumerWarps = kWsGroupWarps * kWsGroups;
constexpr int kWsThreads = 32 * (1 + kWsConsumerWarps);
constexpr int kWsChunk = 32 * kWsGroupWarps;  // CH: outputs per chunk (one per thread of a group)
constexpr int kWsFS = 4;                      // stream segments per ring stage
constexpr int kQtabShift = 17;                // qtab entry: mask(V) | rank(V \ {min V}) << 17
constexpr int kWsEnd = -1;

// Window width D and ring depth NS per element size (shared memory <= 227 KB).
__host__ __device__ constexpr int ws_window(int elem_bytes) { return elem_bytes == 16 ? 14 : 15; }
template <int ELEM>
struct WsGeom {
    static constexpr int NSG = ELEM == 16 ? 3 : 6;  // stages per group ring
    static constexpr int NS = NSG * kWsGroups;
};

template <class T>
struct WsDesc {
    int32_t F, m, f, src_pad;
    uint32_t q0, q1, rounds, pad;
    uint64_t cur_base;
    uint64_t sbase[kMaxOrder];  // bases of the stream tiles (F \ {F_l}, k-1) in the previous layer
    T coef[kMaxOrder];          // a(k-1, F_l)
};

__host__ __device__ constexpr size_t round16(size_t b) { return (b + 15) & ~size_t(15); }

template <class T>
struct WsSmem {
    static constexpr int NS = WsGeom<(int)sizeof(T)>::NS;
    static constexpr int NSG = WsGeom<(int)sizeof(T)>::NSG;
    static constexpr size_t kSlot = round16(sizeof(T) * kWsChunk + 16) / sizeof(T);  // elements per segment slot
    uint2* B2;         // B2[i * kBinomDim + s] = (C(s, i), C(s, i - 1))
    WsDesc<T>* desc;   // [2]
    uint64_t* full;    // [G][NSG]
    uint64_t* empty;   // [G][NSG]
    uint64_t* sfull;   // [2]
    uint64_t* sempty;  // [2]
    T* row_low;        // [32]
    T* src;            // [2][src_stride]
    T* stage;          // [G][NSG][FS][kSlot]
    size_t src_stride;

    __host__ __device__ static size_t bytes(int D) {
        const size_t cap = (size_t)binom_u64(D, D / 2);
        return round16(sizeof(uint2) * kBinomDim * kBinomDim) + 2 * round16(sizeof(WsDesc<T>)) +
               round16(8 * (2 * NS + 4)) + round16(sizeof(T) * 32) + 2 * round16(sizeof(T) * cap + 16) +
               round16((size_t)NS * kWsFS * kSlot * sizeof(T));
    }
    __device__ WsSmem(unsigned char* base, int D) {
        size_t off = 0;
        auto take = [&](size_t b) {
            unsigned char* p = base + off;
            off += round16(b);
            return p;
        };
        const size_t cap = (size_t)binom_u64(D, D / 2);
        B2 = reinterpret_cast<uint2*>(take(sizeof(uint2) * kBinomDim * kBinomDim));
        desc = reinterpret_cast<WsDesc<T>*>(take(2 * round16(sizeof(WsDesc<T>))));
        uint64_t* bars = reinterpret_cast<uint64_t*>(take(8 * (2 * NS + 4)));
        full = bars;
        empty = bars + NS;
        sfull = bars + 2 * NS;
        sempty = bars + 2 * NS + 2;
        row_low = reinterpret_cast<T*>(take(sizeof(T) * 32));
        src_stride = round16(sizeof(T) * cap + 16) / sizeof(T);
        src = reinterpret_cast<T*>(take(2 * round16(sizeof(T) * cap + 16)));
        stage = reinterpret_cast<T*>(take((size_t)NS * kWsFS * kSlot * sizeof(T)));
    }
    __device__ T* src_buf(int b) const { return src + (size_t)b * src_stride; }
    // ring slot of group g, stage s, segment li
    __device__ T* slot(int g, int s, int li) const { return stage + (((size_t)g * NSG + s) * kWsFS + li) * kSlot; }
    __device__ uint64_t* full_bar(int g, int s) const { return full + g * NSG + s; }
    __device__ uint64_t* empty_bar(int g, int s) const { return empty + g * NSG + s; }
    __device__ WsDesc<T>* desc_buf(int b) const {
        return reinterpret_cast<WsDesc<T>*>(reinterpret_cast<unsigned char*>(desc) + b * round16(sizeof(WsDesc<T>)));
    }
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

__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// TMA 1D bulk copy global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
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

// ---------------------------------------------------------------- consumer math

template <class RR, int M, class T>
__device__ __forceinline__ T ws_low(uint32_t e, const T* __restrict__ src, const T* __restrict__ row_low,
                                    const uint2* __restrict__ B2, bool& ov) {
    uint32_t V = e & ((1u << kQtabShift) - 1);
    uint32_t Q = e >> kQtabShift, P = 0;
    T acc;
#pragma unroll
    for (int i = 1; i <= M; ++i) {
        const int s = __ffs(V) - 1;
        V &= V - 1;
        const uint2 b = B2[i * kBinomDim + s];  // (C(s, i), C(s, i-1))
        if (i >= 2) Q -= b.y;
        const T c = row_low[s];
        const T x = src[P + Q];
        acc = i == 1 ? RR::mul(c, x, ov) : RR::mac(acc, c, x, ov);
        P += b.x;
    }
    return acc;
}

template <class RR, class T>
__device__ __forceinline__ T ws_low_dispatch(int m, uint32_t e, const T* src, const T* row_low, const uint2* B2,
                                             bool& ov) {
    switch (m) {
#define PL_WS_CASE(M) \
    case M:           \
        return ws_low<RR, M>(e, src, row_low, B2, ov);
        PL_WS_CASE(1) PL_WS_CASE(2) PL_WS_CASE(3) PL_WS_CASE(4) PL_WS_CASE(5) PL_WS_CASE(6) PL_WS_CASE(7)
        PL_WS_CASE(8) PL_WS_CASE(9) PL_WS_CASE(10) PL_WS_CASE(11) PL_WS_CASE(12) PL_WS_CASE(13) PL_WS_CASE(14)
        PL_WS_CASE(15)
#undef PL_WS_CASE
    }
    return RR::zero();
}

// One ring stage's high terms for output j.
template <class RR, class T>
__device__ __forceinline__ T ws_stage_terms(T acc, const WsSmem<T>& sm, const WsDesc<T>& d, int g, int s, int l0,
                                            int nl, uint32_t c0, int j, bool init_first, bool& ov) {
#pragma unroll
    for (int li = 0; li < kWsFS; ++li) {
        if (li < nl) {
            const int pad = sizeof(T) == 16 ? 0 : (int)((d.sbase[l0 + li] + c0) & 1u);
            const T x = sm.slot(g, s, li)[pad + j];
            acc = (init_first && li == 0) ? RR::mul(d.coef[l0 + li], x, ov) : RR::mac(acc, d.coef[l0 + li], x, ov);
        }
    }
    return acc;
}

// Consumer group g's share of one tile: chunks g, g + G, g + 2G, ... Each of
// its chunks takes `rounds` consecutive stages of the group's own ring; `seq`
// is the group's running stage counter (stage seq % NSG, use seq / NSG).
template <class RR, class T>
__device__ __forceinline__ void ws_consume_tile(const WsSmem<T>& sm, const WsDesc<T>& d, const T* src,
                                                const uint32_t* __restrict__ qt, T* __restrict__ cur, int g, int j,
                                                uint32_t& seq, bool& ov) {
    constexpr int NSG = WsSmem<T>::NSG;
    const int m = d.m, f = d.f;
    const uint32_t nchunks = (d.q1 - d.q0 + kWsChunk - 1) / kWsChunk;
    // qtab prefetch one chunk ahead (its latency is a global load)
    uint32_t c = (uint32_t)g;
    uint32_t e_next = 0;
    if (m >= 1 && c < nchunks) {
        const uint32_t q = d.q0 + c * kWsChunk + j;
        if (q < d.q1) e_next = __ldg(qt + q);
    }
    for (; c < nchunks; c += kWsGroups) {
        const uint32_t c0 = d.q0 + c * kWsChunk;
        const uint32_t len = min((uint32_t)kWsChunk, d.q1 - c0);
        const bool valid = (uint32_t)j < len;
        const uint32_t e = e_next;
        if (m >= 1 && c + kWsGroups < nchunks) {
            const uint32_t qn = c0 + kWsGroups * kWsChunk + j;
            if (qn < d.q1) e_next = __ldg(qt + qn);
        }
        T acc = RR::zero();
        if (valid && m >= 1) acc = ws_low_dispatch<RR>(m, e, src, sm.row_low, sm.B2, ov);
        for (int l0 = 0; l0 < f; l0 += kWsFS, ++seq) {
            const int nl = min(kWsFS, f - l0);
            const int s = (int)(seq % NSG);
            mbar_wait(sm.full_bar(g, s), (seq / NSG) & 1u);
            if (valid) acc = ws_stage_terms<RR>(acc, sm, d, g, s, l0, nl, c0, j, m == 0 && l0 == 0, ov);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(sm.empty_bar(g, s));
        }
        if (valid) cur[d.cur_base + c0 + j] = acc;
    }
}

// ---------------------------------------------------------------- producer helpers

// Claims the next valid tile (F with 0 <= k - |F| <= D) or kWsEnd; lane 0 only.
__device__ __forceinline__ int32_t ws_claim(unsigned int* counter, uint32_t F0, uint32_t F1, int k, int D) {
    for (;;) {
        const uint32_t t = F0 + atomicAdd(counter, 1u);
        if (t > F1) return kWsEnd;
        const int mm = k - __popc(t);
        if (mm >= 0 && mm <= D) return (int32_t)t;
    }
}

// Writes the descriptor of tile F into buffer tb and issues its low-source
// bulk copy (whole warp; the arrive on sfull[tb] releases the descriptor).
template <class T>
__device__ __forceinline__ void ws_open_tile(const WsSmem<T>& sm, int tb, int32_t F, int k, int D, uint64_t r0,
                                             uint64_t r1, const T* __restrict__ prev, const T* __restrict__ row,
                                             int lane) {
    WsDesc<T>* d = sm.desc_buf(tb);
    if (F == kWsEnd) {
        if (lane == 0) {
            d->F = kWsEnd;
            mbar_arrive(&sm.sfull[tb]);
        }
        return;
    }
    const int f = __popc((uint32_t)F), m = k - f;
    uint64_t cur_base = 0, src_base = 0;
    {
        int l = 1;
        for (uint32_t ff = (uint32_t)F; ff; ff &= ff - 1, ++l) {
            const int col = D + __ffs(ff) - 1;
            const uint2 b = sm.B2[(m + l) * kBinomDim + col];
            cur_base += b.x;
            src_base += b.y;
        }
    }
    if (lane < f) {
        uint64_t b = 0;
        int l = 0, p = 1;
        for (uint32_t ff = (uint32_t)F; ff; ff &= ff - 1, ++l) {
            const int col = D + __ffs(ff) - 1;
            if (l == lane) {
                d->coef[lane] = row[col];
                continue;
            }
            b += sm.B2[(m + p) * kBinomDim + col].x;
            ++p;
        }
        d->sbase[lane] = b;
    }
    const uint32_t tile_len = sm.B2[m * kBinomDim + D].x;
    const uint32_t q0 = r0 > cur_base ? (uint32_t)(r0 - cur_base) : 0u;
    const uint32_t q1 = (r1 - cur_base) < tile_len ? (uint32_t)(r1 - cur_base) : tile_len;
    BulkSpan<T> sp{prev, 0u, 0};
    if (m >= 1) sp = bulk_span(prev, src_base, sm.B2[(m - 1) * kBinomDim + D].x);
    if (lane == 0) {
        d->F = F;
        d->m = m;
        d->f = f;
        d->q0 = q0;
        d->q1 = q1;
        d->rounds = (uint32_t)((f + kWsFS - 1) / kWsFS);
        d->cur_base = cur_base;
        d->src_pad = sp.pad;
    }
    __syncwarp();
    if (lane == 0) {
        mbar_arrive_expect_tx(&sm.sfull[tb], sp.bytes);
        if (sp.bytes) bulk_g2s(sm.src_buf(tb), sp.src, sp.bytes, &sm.sfull[tb]);
    }
}

// ---------------------------------------------------------------- kernel

template <class R, class RU>
__global__ void __launch_bounds__(kWsThreads, 1)
    sz_ws_kernel(const typename R::T* __restrict__ a, int n, int k, int D, const typename R::T* __restrict__ prev,
                 typename R::T* __restrict__ cur, uint64_t r0, uint64_t r1, uint32_t F0, uint32_t F1,
                 unsigned int* __restrict__ counter, const uint32_t* __restrict__ qtab,
                 const uint32_t* __restrict__ qtab_off, const int32_t* __restrict__ guard,
                 int32_t* __restrict__ status) {
    using T = typename R::T;
    constexpr int NSG = WsSmem<T>::NSG;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const WsSmem<T> sm(smem_raw, D);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* row = a + (size_t)(k - 1) * n;

    for (int e = threadIdx.x; e < kBinomDim * kBinomDim; e += blockDim.x) {
        const int i = e / kBinomDim, s = e % kBinomDim;
        sm.B2[e] = make_uint2((uint32_t)binom_u64(s, i), i >= 1 ? (uint32_t)binom_u64(s, i - 1) : 0u);
    }
    for (int v = threadIdx.x; v < D; v += blockDim.x) sm.row_low[v] = row[v];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWsGroups * NSG; ++s) {
            mbar_init(&sm.full[s], 1);               // producer's arrive.expect_tx
            mbar_init(&sm.empty[s], kWsGroupWarps);  // the owning group's warps
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.sfull[b], 1);
            mbar_init(&sm.sempty[b], kWsConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        uint32_t seqg[kWsGroups] = {};
        uint32_t tile_u = 0;
        int32_t F = 0;
        if (lane == 0) F = ws_claim(counter, F0, F1, k, D);
        F = __shfl_sync(0xffffffffu, F, 0);
        ws_open_tile(sm, 0, F, k, D, r0, r1, prev, row, lane);  // buffer 0 starts free
        while (F != kWsEnd) {
            const WsDesc<T>* d = sm.desc_buf((int)(tile_u & 1u));
            int32_t Fn = 0;
            if (lane == 0) Fn = ws_claim(counter, F0, F1, k, D);
            Fn = __shfl_sync(0xffffffffu, Fn, 0);
            const int nb = (int)((tile_u + 1) & 1u);
            const unsigned npar = (((tile_u + 1) >> 1) & 1u) ^ 1u;
            bool opened = false;
            const int f = d->f;
            int g = 0;
            for (uint32_t c0 = d->q0; c0 < d->q1; c0 += kWsChunk, g = (g + 1) % kWsGroups) {
                const uint32_t len = min((uint32_t)kWsChunk, d->q1 - c0);
                for (int l0 = 0; l0 < f; l0 += kWsFS) {
                    // one lane decides (per-lane test_wait results may differ) and broadcasts
                    bool ready = false;
                    if (!opened) ready = __shfl_sync(0xffffffffu, lane == 0 ? mbar_test(&sm.sempty[nb], npar) : false, 0);
                    if (ready) {
                        ws_open_tile(sm, nb, Fn, k, D, r0, r1, prev, row, lane);
                        opened = true;
                    }
                    const int nl = min(kWsFS, f - l0);
                    const uint32_t sq = seqg[g]++;
                    const int s = (int)(sq % NSG);
                    mbar_wait(sm.empty_bar(g, s), ((sq / NSG) & 1u) ^ 1u);
                    BulkSpan<T> seg{prev, 0u, 0};
                    if (lane < nl) seg = bulk_span(prev, d->sbase[l0 + lane] + c0, len);
                    unsigned total = seg.bytes;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
                    if (lane == 0) mbar_arrive_expect_tx(sm.full_bar(g, s), total);
                    __syncwarp();
                    if (lane < nl) bulk_g2s(sm.slot(g, s, lane), seg.src, seg.bytes, sm.full_bar(g, s));
                }
            }
            if (!opened) {
                mbar_wait(&sm.sempty[nb], npar);
                ws_open_tile(sm, nb, Fn, k, D, r0, r1, prev, row, lane);
            }
            F = Fn;
            ++tile_u;
        }
    } else {
        // ------------------------------------------------------------ consumers
        const int cw = warp - 1;
        const int g = cw / kWsGroupWarps;
        const int j = (cw % kWsGroupWarps) * 32 + lane;
        bool use_checked = false;
        if constexpr (R::kChecked) use_checked = guard != nullptr && guard[0] != 0;
        bool ov = false;
        uint32_t seq = 0, tile_u = 0;
        for (;;) {
            const int tb = (int)(tile_u & 1u);
            mbar_wait(&sm.sfull[tb], (tile_u >> 1) & 1u);
            const WsDesc<T>& d = *sm.desc_buf(tb);
            if (d.F == kWsEnd) break;
            const uint32_t* qt = qtab + qtab_off[d.m];
            const T* src = sm.src_buf(tb) + d.src_pad;
            if constexpr (R::kChecked) {
                if (use_checked) {
                    ws_consume_tile<R>(sm, d, src, qt, cur, g, j, seq, ov);
                } else {
                    ws_consume_tile<RU>(sm, d, src, qt, cur, g, j, seq, ov);
                }
            } else {
                ws_consume_tile<R>(sm, d, src, qt, cur, g, j, seq, ov);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.sempty[tb]);
            ++tile_u;
        }
        if (ov) atomicOr(status, 1);
    }
}

}  // namespace pl
