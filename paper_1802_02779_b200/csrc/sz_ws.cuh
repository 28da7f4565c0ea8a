// Warp-specialised per-layer kernel (the large-order hot path).
//
// Recurrence (reference proj/src/permanent.cpp:164-175):
//     per(S) = sum_{j in S, ascending} a(k-1, j) * per(S \ {j}),   |S| = k,
// evaluated one layer at a time, every layer dense in colex order.
//
// Tiling. Columns split into a low window [0, D) and high columns [D, n). For
// S = F u V (F = S n [D, n), |F| = f; V = S n [0, D), |V| = m)
//     rank(S) = rank_D(V) + sum_{l=1..f} C(F_l, m + l),
// so the k-subsets sharing F form one contiguous colex range, the tile (F, k),
// of C(D, m) entries indexed by q = rank_D(V). Output q needs
//   * low terms  S \ {v_i}: inside the tile's low source (F, k-1), C(D, m-1)
//     contiguous entries staged whole in shared memory by one bulk copy; the
//     ranks rank_D(V \ {v_i}) and columns v_i come from the host-built low-term
//     table (ltab: one 16-byte load per output for m <= 8);
//   * high terms S \ {F_l}: entry q of the tile (F \ {F_l}, k-1) -> aligned
//     contiguous streams with a tile-uniform coefficient, staged by TMA.
// Low columns are all below high columns, so "low ascending, then high
// ascending" is the reference's ascending-j order; the non-FMA rings keep its
// rounding sequence bit for bit.
//
// Schedule. One CTA per SM, persistent. Tiles are claimed on the device, in
// increasing F (increasing colex order), from one ticket counter per launch:
// ticket t is the t-th valid high set F (popcount in [k - D, k]) from the
// range's first one on, read from the layer's tile list (generated once per
// (device, n) by sz_tile_list_kernel and cached). So the GPU sweeps each
// layer as one tight front, every SM takes the next tile when it has room
// (no per-CTA schedule to build on the host), and stream tiles of nearby
// high columns are re-read from L2 (far ones are loaded evict-first). Launched with programmatic dependent launch:
// the prologue overlaps the previous layer.
//
// Roles (warp-specialised, mbarrier hand-offs, no CTA-wide sync after setup).
//   publisher (last warp)  walks the CTA's tile list; per tile builds the
//                          header (bases and clip range by two warp scans,
//                          coefficients, stream bases, pad mask), places the
//                          tile's low source in a variable-size shared-memory
//                          ring (FIFO, up to NHDR = 8 tiles in flight) and
//                          stages it with one cp.async.bulk.
//   streamers (NST warps)  for the chunks (CH outputs) of their consumer
//                          groups, stream the high-term segments into the
//                          group's NSG-stage ring, FS segments per stage, one
//                          cp.async.bulk per segment, mbarrier tx counts.
//   consumers (G groups    take alternate chunks, PER outputs per thread: low
//   of GW warps)           terms from the source ring, high terms from the
//                          group's ring (read to registers; every thread hands
//                          the slot back once its own loads have returned,
//                          loaded_dep; then the math), coalesced stores. The
//                          chunk loop is specialised per low count m.
// Geometry per element size (WsGeom): complex 3 groups x 4 warps, D = 14,
// FS = 2 segments per stage, 4 stages per group ring (C5 114 -> 108.5 ms against
// FS = 4 x 2 stages in the same shared memory); 8-byte 3 groups x 8 warps, D = 14,
// FS = 4, 2 stages.
#pragma once

#include <cstdint>

#include "ring.cuh"

namespace pl {

constexpr int kWsMaxHigh = 32;                 // high columns per tile (n - D <= 31)
constexpr int kWsLtabRankBits = 12;           // ltab entry: rank_D(V \ {v}) | v << 12 (D <= 14)
constexpr int kWsEnd = -1;
#ifndef PL_WS_LOW_INTERLEAVE
#define PL_WS_LOW_INTERLEAVE 0
#endif
constexpr bool kWsLowInterleave = PL_WS_LOW_INTERLEAVE;  // large m: low terms of both outputs term by term
constexpr int kWaitHintNs = 20000;             // mbarrier try_wait suspend-time hint
#ifndef PL_WS_PSLEEP
#define PL_WS_PSLEEP 0
#endif
#ifndef PL_WS_PUBSLEEP
#define PL_WS_PUBSLEEP 0
#endif
constexpr unsigned kProdSleepNs = PL_WS_PSLEEP;     // max poll sleep of streamer waits (0: try_wait)
constexpr unsigned kPubSleepNs = PL_WS_PUBSLEEP;    // max poll sleep of publisher waits (0: try_wait)

// Low window D per element size: the largest tile source C(D, D/2) must fit a
// shared-memory slot next to the stage rings (<= 227 KB in all).
// (PL_WS_* macros: build-time tuning overrides.)
#ifndef PL_WS_D16
#define PL_WS_D16 14
#endif
#ifndef PL_WS_D8
#define PL_WS_D8 14
#endif
#ifndef PL_WS_NSG16
#define PL_WS_NSG16 4
#endif
#ifndef PL_WS_NSG8
#define PL_WS_NSG8 2
#endif
#ifndef PL_WS_FS16
#define PL_WS_FS16 2
#endif
#ifndef PL_WS_FS8
#define PL_WS_FS8 4
#endif
#ifndef PL_WS_NSRC16
#define PL_WS_NSRC16 2
#endif
#ifndef PL_WS_NSRC8
#define PL_WS_NSRC8 3
#endif
#ifndef PL_WS_G16
#define PL_WS_G16 3
#endif
#ifndef PL_WS_G8
#define PL_WS_G8 3
#endif
#ifndef PL_WS_GW16
#define PL_WS_GW16 4
#endif
#ifndef PL_WS_GW8
#define PL_WS_GW8 8
#endif
#ifndef PL_WS_NST16
#define PL_WS_NST16 3
#endif
#ifndef PL_WS_NST8
#define PL_WS_NST8 3
#endif
#ifndef PL_WS_PER16
#define PL_WS_PER16 2
#endif
#ifndef PL_WS_PER8
#define PL_WS_PER8 2
#endif
__host__ __device__ constexpr int ws_window(int elem_bytes) { return elem_bytes == 16 ? PL_WS_D16 : PL_WS_D8; }

// Consumer groups per CTA: three for 8-byte elements, two for complex, whose
// arithmetic needs the registers.
template <int ELEM>
struct WsGeom {
    static constexpr int G = ELEM == 16 ? PL_WS_G16 : PL_WS_G8;       // consumer groups
    static constexpr int GW = ELEM == 16 ? PL_WS_GW16 : PL_WS_GW8;    // warps per group
    static constexpr int PER = ELEM == 16 ? PL_WS_PER16 : PL_WS_PER8; // outputs per thread per chunk
    static constexpr int LANES = 32 * GW;                             // consumer threads per group
    static constexpr int CHUNK = LANES * PER;                         // CH: outputs per chunk
    static constexpr int NSG = ELEM == 16 ? PL_WS_NSG16 : PL_WS_NSG8;     // stages per group ring
    static constexpr int FS = ELEM == 16 ? PL_WS_FS16 : PL_WS_FS8;        // stream segments per ring stage
    static constexpr int NSRC = ELEM == 16 ? PL_WS_NSRC16 : PL_WS_NSRC8;  // low-source ring, in largest tiles
    static constexpr int NHDR = 8;                                        // tile headers in flight
    // elements per low-source slot: the largest tile source C(D, D/2), plus the
    // 8-byte alignment pad and round-up of bulk_span
    static constexpr int kSrcSlot =
        (int)((binom_u64(ws_window(ELEM), ws_window(ELEM) / 2) + 2 + 16 / ELEM - 1) / (16 / ELEM) * (16 / ELEM));
    static constexpr int kConsumerWarps = GW * G;
    static constexpr int NST = ELEM == 16 ? PL_WS_NST16 : PL_WS_NST8;  // streamer warps (streamer s feeds groups g = s mod NST)
    static constexpr int kThreads = 32 * (kConsumerWarps + NST + 1);    // consumers, streamers, publisher
    // registers per thread that still fit one CTA per SM (64K registers, 8-register units)
    static constexpr int kMaxReg = (65536 / kThreads) / 8 * 8 > 255 ? 255 : (65536 / kThreads) / 8 * 8;
};

__host__ __device__ constexpr size_t round16(size_t b) { return (b + 15) & ~size_t(15); }

// Tile header, written by the producer into a tile slot before the slot's
// full barrier completes.
template <class T>
struct WsHdr {
    int32_t m, f;                    // m < 0: end of the CTA's tile list
    uint32_t q1, nchunks, cb, cs;    // clip end; this CTA's chunks start at cb + i * cs
    uint64_t cur_base;               // rank of the tile's first output
    uint32_t qoff, pad_src;          // ltab offset for m; 8-byte alignment pad of the source
    uint32_t padmask;                // bit l: 8-byte alignment pad of stream l's chunks (cb, cs even)
    uint32_t src_off, src_len;       // the low source's place in the source ring (elements)
    T coef[kWsMaxHigh];              // a(k-1, F_l)
    uint64_t sbase[kWsMaxHigh];      // base rank of stream tile (F \ {F_l}, k-1)
    int8_t mode[kWsMaxHigh];         // L2 policy of stream l (0 plain, 1 evict-first, 2 evict-last)
};

template <class T>
struct WsSmem {
    static constexpr int NSG = WsGeom<(int)sizeof(T)>::NSG;
    static constexpr int G = WsGeom<(int)sizeof(T)>::G;
    static constexpr int CW = WsGeom<(int)sizeof(T)>::kConsumerWarps;
    static constexpr int NSRC = WsGeom<(int)sizeof(T)>::NSRC;
    static constexpr int NHDR = WsGeom<(int)sizeof(T)>::NHDR;
    static constexpr int kSrcSlot = WsGeom<(int)sizeof(T)>::kSrcSlot;
#ifdef PL_WS_SRCRING_PCT  // ring size in percent of NSRC largest sources (tuning)
    static constexpr uint32_t kSrcRing = ((uint32_t)NSRC * kSrcSlot * PL_WS_SRCRING_PCT / 100) & ~1u;
#else
    static constexpr uint32_t kSrcRing = (uint32_t)NSRC * kSrcSlot;  // ring elements (even)
#endif
    static constexpr int FS = WsGeom<(int)sizeof(T)>::FS;
    static constexpr int GW = WsGeom<(int)sizeof(T)>::GW;
    static constexpr int NST = WsGeom<(int)sizeof(T)>::NST;
    static constexpr int PER = WsGeom<(int)sizeof(T)>::PER;
    static constexpr int LANES = WsGeom<(int)sizeof(T)>::LANES;
    static constexpr int CHUNK = WsGeom<(int)sizeof(T)>::CHUNK;
    static constexpr size_t kSlot = round16(sizeof(T) * CHUNK + 16) / sizeof(T);  // elements per segment slot
    uint2* B2;            // B2[i * kBinomDim + s] = (C(s, i), C(s, i - 1))
    T* row_low;           // [32]   a(k-1, v), v < D
    uint64_t* full;       // [G][NSG]
    uint64_t* empty;      // [G][NSG]
    T* stage;             // [G][NSG][FS][kSlot]
    uint64_t* src_full;   // [NHDR]  header written and low source landed (consumers)
    uint64_t* src_empty;  // [NHDR]  tile released by every consumer and streamer warp
    uint64_t* hdr_full;   // [NHDR]  header written (streamers: they need no source)
    WsHdr<T>* hdr;        // [NHDR]
    T* src;               // [kSrcRing]  ring of tile low sources X(F, k-1), variable size

    __host__ __device__ static size_t bytes() {
        return round16(sizeof(uint2) * kBinomDim * kBinomDim) + round16(sizeof(T) * 32) + round16(8 * 2 * G * NSG) +
               round16((size_t)G * NSG * FS * kSlot * sizeof(T)) + round16(8 * 3 * NHDR) +
               round16(sizeof(WsHdr<T>) * NHDR) + round16((size_t)kSrcRing * sizeof(T));
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
        uint64_t* bars = reinterpret_cast<uint64_t*>(take(8 * 2 * G * NSG));
        full = bars;
        empty = bars + G * NSG;
        stage = reinterpret_cast<T*>(take((size_t)G * NSG * FS * kSlot * sizeof(T)));
        src_full = reinterpret_cast<uint64_t*>(take(8 * 3 * NHDR));
        src_empty = src_full + NHDR;
        hdr_full = src_full + 2 * NHDR;
        hdr = reinterpret_cast<WsHdr<T>*>(take(sizeof(WsHdr<T>) * NHDR));
        src = reinterpret_cast<T*>(take((size_t)kSrcRing * sizeof(T)));
    }
    __device__ T* slot(int g, int s, int li) const { return stage + (((size_t)g * NSG + s) * FS + li) * kSlot; }
    __device__ uint64_t* full_bar(int g, int s) const { return full + g * NSG + s; }
    __device__ uint64_t* empty_bar(int g, int s) const { return empty + g * NSG + s; }
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
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(kWaitHintNs)
        : "memory");
}

// Same wait, separate code location (profiles attribute tile-slot waits here).
__device__ __forceinline__ void mbar_wait_slot(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(kWaitHintNs)
        : "memory");
}

// Same wait, separate code location (producer's ring-slot waits).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    uint32_t ok;
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

// Wait of a warp that is normally ahead (streamer on a full ring, publisher
// on busy slots): poll with a growing sleep so that it leaves the issue
// slots to the consumer warps.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, unsigned parity, unsigned max_ns) {
    unsigned ns = 32;
    while (!mbar_test(bar, parity)) {
        __nanosleep(ns);
        ns = ns * 2 < max_ns ? ns * 2 : max_ns;
    }
}

// Same wait, separate code location (producer's ring-slot waits).
__device__ __forceinline__ void mbar_wait_prod(uint64_t* bar, unsigned parity) {
    if constexpr (kProdSleepNs == 0)
        mbar_wait_slot(bar, parity);
    else
        mbar_wait_backoff(bar, parity, kProdSleepNs);
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

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
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

// L2 prefetch of a 16-byte aligned run (no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
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

// Inclusive warp prefix sum (lane order).
__device__ __forceinline__ uint64_t warp_scan_u64(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

// Zero, computed from `n` loaded values (one 32-bit word of each: a load
// instruction's scoreboard covers its whole result): an mbarrier arrive whose
// address adds it cannot issue before those loads have returned. An
// mbarrier.arrive does not wait for the thread's outstanding shared-memory
// loads (ptxas emits no scoreboard wait before SYNCS.ARRIVE), so a slot handed
// back right after ld.shared can be refilled by the next TMA copy before a
// queued load has read it (seen as wrong second outputs per thread in
// profiles/archive_probe.py). `rt_zero` must be 0 at run time but unknown to
// the compiler (a kernel argument), so the dependency survives ptxas.
template <class T>
__device__ __forceinline__ uint32_t loaded_dep(const T* v, int n, uint32_t rt_zero) {
    uint32_t d = 0;
    for (int i = 0; i < n; ++i) d ^= *reinterpret_cast<const uint32_t*>(&v[i]);
    return (uint32_t)(d == 0x9e3779b9u) & rt_zero;
}

// ---------------------------------------------------------------- debug trace
// Event trace of CTA 0 for pipeline analysis (PL_WS_TRACE, see capi.cu):
// region r holds (clock64, event | arg << 8) pairs; r = 0/1 first warp of
// consumer group 0/1, 2 streamer of group 0, 3 publisher.
static __device__ unsigned long long* g_ws_trace = nullptr;
constexpr int kWsTraceCap = 65536;

#ifndef PL_WS_TRACE_ENABLE
struct WsTrace {  // compiled out unless built with -DPL_WS_TRACE_ENABLE
    __device__ __forceinline__ void init(int) {}
    __device__ __forceinline__ void ev(uint32_t, uint32_t = 0) {}
};
#else
struct WsTrace {
    unsigned long long* p = nullptr;
    uint32_t i = 0;
    __device__ __forceinline__ void init(int region) {
        p = (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && g_ws_trace) ? g_ws_trace + (size_t)region * kWsTraceCap * 2
                                                                          : nullptr;
    }
    __device__ __forceinline__ void ev(uint32_t e, uint32_t arg = 0) {
        if (p && i < kWsTraceCap) {
            p[2 * i] = clock64();
            p[2 * i + 1] = e | (unsigned long long)arg << 8;
            ++i;
        }
    }
};
#endif

// ---------------------------------------------------------------- tile lists

// Valid high sets of layer k: F in [0, 2^H) with fmin <= popc(F) <= fmax
// (fmin = max(0, k - D), fmax = min(k, H)), in increasing integer order (=
// increasing colex rank of their tiles). Thread g writes the g-th one: bit b
// is 0 iff g < the number of valid completions of the prefix with bit b = 0,
// sum_{j in [fmin - p, fmax - p]} C(b, j) (p = ones so far).
static __global__ void sz_tile_list_kernel(int H, int fmin, int fmax, uint32_t count, uint32_t* __restrict__ out) {
    const uint32_t g0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t g = g0; g < count; g += gridDim.x * blockDim.x) {
        uint32_t r = g, F = 0;
        int p = 0;
        for (int b = H - 1; b >= 0; --b) {
            uint64_t c0 = 0;
            const int jlo = fmin - p > 0 ? fmin - p : 0, jhi = fmax - p < b ? fmax - p : b;
            uint64_t c = binom_u64(b, jlo);
            for (int j = jlo; j <= jhi; ++j) {  // C(b, j) by the multiplicative step
                c0 += c;
                c = c * (uint64_t)(b - j) / (uint64_t)(j + 1);
            }
            if (r >= c0) {
                r -= (uint32_t)c0;
                F |= 1u << b;
                ++p;
            }
        }
        out[g] = F;
    }
}

// ---------------------------------------------------------------- consumer math

// Low terms of one output from its ltab list (entries rank | column << 12,
// ascending column): gathers from the shared-memory tile source.
__device__ __forceinline__ uint32_t ltab_entry(const uint4& a, const uint4& b, int i) {
    const uint4& v = i < 8 ? a : b;
    const int w = (i & 7) >> 1;
    const uint32_t word = w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
    return (i & 1) ? word >> 16 : word & 0xffffu;
}

// Low-term coefficient a(k-1, v). PL_WS_COEF_SPLIT=1 (build-time experiment,
// round 2c): complex rows kept as two double arrays (re[32], im[32]) and read
// by two 8-byte loads -- 14 columns x 8 bytes fall in distinct banks, whereas a
// gathered 16-byte load makes columns v and v + 8 collide within a quarter
// warp. Measured equal on C5 (110.6-111.2 ms either way, profiles/r2c/
// coef_split.txt): the saved bank conflicts cost one more issue slot per low term.
#ifndef PL_WS_COEF_SPLIT
#define PL_WS_COEF_SPLIT 0
#endif
template <class T>
__device__ __forceinline__ T ws_coef_low(const T* __restrict__ row_low, uint32_t v) {
    if constexpr (sizeof(T) == 16 && PL_WS_COEF_SPLIT) {
        const double* p = reinterpret_cast<const double*>(row_low);
        T c;
        c.x = p[v];
        c.y = p[32 + v];
        return c;
    } else {
        return row_low[v];
    }
}

template <class RR, int M, class T>
__device__ __forceinline__ T ws_low(const uint4& ea, const uint4& eb, const T* __restrict__ src,
                                    const T* __restrict__ row_low, bool& ov) {
    T x[M];
#pragma unroll
    for (int i = 0; i < M; ++i) x[i] = src[ltab_entry(ea, eb, i) & ((1u << kWsLtabRankBits) - 1)];
    T acc = RR::mul(ws_coef_low(row_low, ltab_entry(ea, eb, 0) >> kWsLtabRankBits), x[0], ov);
#pragma unroll
    for (int i = 1; i < M; ++i)
        acc = RR::mac(acc, ws_coef_low(row_low, ltab_entry(ea, eb, i) >> kWsLtabRankBits), x[i], ov);
    return acc;
}

// Low terms of all PER outputs of a thread, term by term (the register
// footprint stays bounded for large m; the scheduler still runs ahead on the
// independent shared-memory loads).
template <class RR, int M, int PER, class T>
__device__ __forceinline__ void ws_low_interleaved(const uint4 (&ea)[PER], const uint4 (&eb)[PER],
                                                   const T* __restrict__ src, const T* __restrict__ row_low,
                                                   T (&acc)[PER], bool (&ov)[PER]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const uint32_t e = ltab_entry(ea[p], eb[p], i);
            const T x = src[e & ((1u << kWsLtabRankBits) - 1)];
            const T c = ws_coef_low(row_low, e >> kWsLtabRankBits);
            acc[p] = i == 0 ? RR::mul(c, x, ov[p]) : RR::mac(acc[p], c, x, ov[p]);
        }
    }
}

// Consumer group g's share of one tile: its chunks c_first, c_first + G, ...
// (chunks are dealt to groups round-robin over the CTA's whole tile sequence).
// Each chunk takes ceil(f / FS) consecutive stages of the group's own ring;
// `seq` is the group's running stage counter (stage seq % NSG, use seq / NSG).
template <class RR, int M, class T>
__device__ __forceinline__ void ws_consume_tile(const WsSmem<T>& sm, const WsHdr<T>& h, const T* __restrict__ src,
                                                const uint4* __restrict__ qt, T* __restrict__ cur, int g, int j,
                                                uint32_t c_first, uint32_t& seq, bool& ov, uint32_t hints,
                                                WsTrace& tr) {
    constexpr int NSG = WsSmem<T>::NSG;
    constexpr int G = WsSmem<T>::G;
    constexpr int FS = WsSmem<T>::FS;
    constexpr int PER = WsSmem<T>::PER, LANES = WsSmem<T>::LANES, CHUNK = WsSmem<T>::CHUNK;
    const int f = h.f;
    const uint32_t q1 = h.q1, nchunks = h.nchunks, cb = h.cb, cs = h.cs, padmask = h.padmask;
    const uint64_t cur_base = h.cur_base;
    const uint64_t pol_store = l2_evict_first_policy();
    uint32_t c = c_first;
    // each thread owns outputs j + p * LANES of every chunk: independent
    // accumulation chains; ltab lists are prefetched one chunk ahead
    uint4 ea_next[PER], eb_next[PER];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
        const uint32_t q = min(cb + c * cs + j + p * LANES, q1 - 1);
        if constexpr (M >= 1) ea_next[p] = __ldg(qt + 2 * q);
        if constexpr (M > 8) eb_next[p] = __ldg(qt + 2 * q + 1);
    }
    for (; c < nchunks; c += G) {
        const uint32_t c0 = cb + c * cs;
        const uint32_t len = min((uint32_t)CHUNK, q1 - c0);
        // Lanes past the tile end compute a duplicate of its last output
        // (no divergence); only their store and overflow flag are dropped.
        uint4 ea[PER], eb[PER];
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            ea[p] = ea_next[p];
            eb[p] = eb_next[p];
        }
        if (c + G < nchunks) {
#pragma unroll
            for (int p = 0; p < PER; ++p) {
                const uint32_t q = min(c0 + G * cs + j + p * LANES, q1 - 1);
                if constexpr (M >= 1) ea_next[p] = __ldg(qt + 2 * q);
                if constexpr (M > 8) eb_next[p] = __ldg(qt + 2 * q + 1);
            }
        }
        bool lov[PER];
        T acc[PER];
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            lov[p] = false;
            acc[p] = RR::zero();
        }
        if constexpr (M >= 1) {
            if constexpr (kWsLowInterleave && (sizeof(T) == 16 ? M > 6 : M > 10))
                ws_low_interleaved<RR, M, PER>(ea, eb, src, sm.row_low, acc, lov);
            else
#pragma unroll
                for (int p = 0; p < PER; ++p) acc[p] = ws_low<RR, M>(ea[p], eb[p], src, sm.row_low, lov[p]);
        }
        for (int l0 = 0; l0 < f; l0 += FS, ++seq) {
            const int nl = min(FS, f - l0);
            int pads[FS];
#pragma unroll
            for (int li = 0; li < FS; ++li) pads[li] = sizeof(T) == 16 ? 0 : (int)((padmask >> (l0 + li)) & 1u);
            const int s = (int)(seq % NSG);
            tr.ev(3, seq);
            mbar_wait(sm.full_bar(g, s), (seq / NSG) & 1u);
            tr.ev(4, seq);
            // read the stage into registers and hand the slot back before the math,
            // so the producer refills it one compute phase earlier
            T xs[PER][FS];
            const T* st = sm.slot(g, s, 0) + j;
            if (nl == FS) {
#pragma unroll
                for (int p = 0; p < PER; ++p)
#pragma unroll
                    for (int li = 0; li < FS; ++li) xs[p][li] = st[p * LANES + li * WsSmem<T>::kSlot + pads[li]];
            } else {
#pragma unroll
                for (int p = 0; p < PER; ++p)
#pragma unroll
                    for (int li = 0; li < FS; ++li)
                        xs[p][li] = li < nl ? st[p * LANES + li * WsSmem<T>::kSlot + pads[li]] : RR::zero();
            }
            // every consumer thread hands the slot back once its own loads have
            // returned (the empty barrier counts GW * 32 arrivals)
            mbar_arrive(sm.empty_bar(g, s) + loaded_dep(&xs[0][0], PER * FS, hints >> 31));  // hints bit 31 is never set
            const bool init_first = M == 0 && l0 == 0;
#pragma unroll
            for (int p = 0; p < PER; ++p) {
                if (nl == FS && !init_first) {
#pragma unroll
                    for (int li = 0; li < FS; ++li) acc[p] = RR::mac(acc[p], h.coef[l0 + li], xs[p][li], lov[p]);
                } else {
#pragma unroll
                    for (int li = 0; li < FS; ++li) {
                        if (li < nl)
                            acc[p] = (init_first && li == 0) ? RR::mul(h.coef[l0 + li], xs[p][li], lov[p])
                                                             : RR::mac(acc[p], h.coef[l0 + li], xs[p][li], lov[p]);
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            if ((uint32_t)(j + p * LANES) < len) {
                if (hints & 4u)
                    stg_hint(cur + cur_base + c0 + j + p * LANES, acc[p], pol_store);
                else
                    cur[cur_base + c0 + j + p * LANES] = acc[p];
                ov |= lov[p];  // duplicates past the tile end never report
            }
        }
    }
}

// The low count m is uniform over a tile: one specialised chunk loop per m.
template <class RR, class T>
__device__ __forceinline__ void ws_consume_dispatch(const WsSmem<T>& sm, const WsHdr<T>& h, const T* src,
                                                    const uint4* qt, T* cur, int g, int j, uint32_t c_first,
                                                    uint32_t& seq, bool& ov, uint32_t hints, WsTrace& tr) {
    switch (h.m) {
#define PL_WS_CT(M)                                                                        \
    case M:                                                                                \
        ws_consume_tile<RR, M>(sm, h, src, qt, cur, g, j, c_first, seq, ov, hints, tr); \
        break;
        PL_WS_CT(0) PL_WS_CT(1) PL_WS_CT(2) PL_WS_CT(3) PL_WS_CT(4) PL_WS_CT(5) PL_WS_CT(6) PL_WS_CT(7)
        PL_WS_CT(8) PL_WS_CT(9) PL_WS_CT(10) PL_WS_CT(11) PL_WS_CT(12) PL_WS_CT(13) PL_WS_CT(14)
#undef PL_WS_CT
    }
}

// ---------------------------------------------------------------- kernel

template <class R, class RU>
__global__ void __launch_bounds__(WsGeom<(int)sizeof(typename R::T)>::kThreads, 1)
    __maxnreg__(WsGeom<(int)sizeof(typename R::T)>::kMaxReg) sz_ws_kernel(const typename R::T* __restrict__ a, int n, int k, int D, const typename R::T* __restrict__ prev,
                 typename R::T* __restrict__ cur, uint64_t r0, uint64_t r1, uint32_t* __restrict__ tickets,
                 const uint32_t* __restrict__ flist, uint32_t ntiles, const uint4* __restrict__ qtab,
                 const uint32_t* __restrict__ qtab_off, const uint2* __restrict__ binom_pairs,
                 const int32_t* __restrict__ guard, int32_t* __restrict__ status, uint32_t hints) {
    using T = typename R::T;
    constexpr int NSG = WsSmem<T>::NSG;
    constexpr int NHDR = WsSmem<T>::NHDR;
    constexpr uint32_t SR = WsSmem<T>::kSrcRing;
    constexpr int G = WsSmem<T>::G;
    constexpr int CW = WsSmem<T>::CW;
    constexpr int FS = WsSmem<T>::FS;
    constexpr int GW = WsSmem<T>::GW, CHUNK = WsSmem<T>::CHUNK;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ T row_sh[kMaxOrder];
    __shared__ uint32_t qoff_sh[kMaxOrder + 2];
    const WsSmem<T> sm(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* row = a + (size_t)(k - 1) * n;

    // Programmatic dependent launch: the next layer's grid may be scheduled as
    // soon as SMs free up; this grid's prologue (engine tables, barriers)
    // overlaps the previous layer's tail, and nothing it reads or writes in the
    // layer buffers (or the matrix) is touched before griddepcontrol.wait.
#ifndef PL_WS_TRIGGER
#define PL_WS_TRIGGER 1
#endif
    if (PL_WS_TRIGGER == 1) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (int e = threadIdx.x; e < kBinomDim * kBinomDim; e += blockDim.x) sm.B2[e] = __ldg(&binom_pairs[e]);
    for (int v = threadIdx.x; v <= D; v += blockDim.x) qoff_sh[v] = __ldg(qtab_off + v);
    if (threadIdx.x == 0) {
        for (int s = 0; s < G * NSG; ++s) {
            mbar_init(&sm.full[s], 1);               // the group's streamer: arrive.expect_tx
            mbar_init(&sm.empty[s], GW * 32);  // every thread of the group's consumer warps
        }
        for (int s = 0; s < NHDR; ++s) {
            mbar_init(&sm.src_full[s], 1);        // publisher: arrive.expect_tx
            mbar_init(&sm.hdr_full[s], 1);        // publisher: arrive
            mbar_init(&sm.src_empty[s], CW + WsSmem<T>::NST);  // every consumer and streamer warp, once per tile
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the previous layer is complete and visible
#ifndef PL_WS_PROXY_FENCE
#define PL_WS_PROXY_FENCE 1
#endif
    // The previous layer's outputs were written by generic-proxy stores and are
    // read below by TMA bulk copies (async proxy): order the two proxies after
    // the grid-dependency wait.
    if (PL_WS_PROXY_FENCE) asm volatile("fence.proxy.async.global;\n" ::: "memory");
    for (int v = threadIdx.x; v < D; v += blockDim.x) {
        if constexpr (sizeof(T) == 16 && PL_WS_COEF_SPLIT) {
            double* p = reinterpret_cast<double*>(sm.row_low);
            const T c = row[v];
            p[v] = *reinterpret_cast<const double*>(&c);
            p[32 + v] = *(reinterpret_cast<const double*>(&c) + 1);
        } else {
            sm.row_low[v] = row[v];
        }
    }
    for (int v = threadIdx.x; v < n; v += blockDim.x) row_sh[v] = row[v];
    __syncthreads();

    if (warp == CW + WsSmem<T>::NST) {
        // ------------------------------------------------------------ publisher
        // Claims tiles (see the schedule note above); per tile it builds the
        // header (two warp scans, no loops) and stages the low source into the
        // next tile slot; a terminal header ends the sequence. It publishes a
        // new tile only while the chunks already queued here are at most
        // `qcap` (hints bits 20-27; 0 = as far ahead as the slots allow): a CTA
        // must not hoard tiles its consumers cannot reach before the layer's
        // end while other SMs idle.
        const int H = n - D;
        const uint32_t qcap = (hints >> 20) & 0xffu;
        uint32_t queued = 0;         // chunks of published tiles not yet released
        uint32_t pub = 0, rel = 0;   // tiles published / tiles whose release this warp has seen
        uint32_t head = 0, tail = 0; // source ring: end of the newest, start of the oldest in-flight source
        // wait until tile `rel` is released by every consumer and streamer warp
        auto release_one = [&]() {
            // the publisher runs up to NHDR tiles ahead: it may poll lazily
            if constexpr (kPubSleepNs == 0)
                mbar_wait_slot(&sm.src_empty[rel % NHDR], (rel / NHDR) & 1u);
            else
                mbar_wait_backoff(&sm.src_empty[rel % NHDR], (rel / NHDR) & 1u, kPubSleepNs);
            queued -= sm.hdr[rel % NHDR].nchunks;
            ++rel;
            tail = rel < pub ? sm.hdr[rel % NHDR].src_off : head;
        };
        // place a source of L elements in the ring (FIFO; a source never wraps)
        auto alloc = [&](uint32_t L) -> uint32_t {
            for (;;) {
                if (pub - rel >= (uint32_t)NHDR) {  // header slot of tile pub still in use
                    release_one();
                    continue;
                }
                if (pub == rel) {
                    head = tail = 0;
                    return 0;
                }
                if (L == 0) return head;
                if (tail < head) {  // in flight: [tail, head)
                    if (head + L <= SR) return head;
                    if (L <= tail) return 0;
                } else if (head + L <= tail) {  // in flight: [tail, SR) u [0, head)
                    return head;
                }
                release_one();
            }
        };
        WsTrace tr;
        tr.init(3);
        // lane 0 keeps two claims in flight: while tile i is published, the F
        // of tile i + 1 is being loaded (its ticket arrived one tile ago) and
        // the ticket of tile i + 2 is being taken; no round trip is waited for
        // inside a tile. Tickets rise per CTA, so past ntiles nothing is lost.
        uint32_t q_t1 = 0, q_F1 = 0, q_t2 = 0;
        if (lane == 0) {
            q_t1 = atomicAdd(tickets, 1u);
            q_F1 = q_t1 < ntiles ? __ldg(flist + q_t1) : 0u;
            q_t2 = atomicAdd(tickets, 1u);
        }
        for (;;) {
            if (qcap) {
                while (pub != rel && queued > qcap) release_one();
            }
            const uint32_t t_cur = __shfl_sync(0xffffffffu, q_t1, 0);
            if (t_cur >= ntiles) break;
            const uint32_t F = __shfl_sync(0xffffffffu, q_F1, 0);
            if (lane == 0) {
                q_t1 = q_t2;
                q_F1 = q_t1 < ntiles ? __ldg(flist + q_t1) : 0u;
                q_t2 = q_t1 < ntiles ? atomicAdd(tickets, 1u) : q_t1;
            }
            const int f = __popc(F), m = k - f;
            // lane h stands for high column D + h; set lanes are F's elements in
            // increasing order, idx = position among them
            const bool set = (F >> lane) & 1u;
            const int idx = __popc(F & ((1u << lane) - 1u));
            uint64_t x = 0, y = 0;
            if (set) {
                const uint2 b = sm.B2[(m + idx + 1) * kBinomDim + D + lane];  // (C(D+h, m+l), C(D+h, m+l-1))
                x = b.x;
                y = b.y;
            }
            // both prefix sums in one 64-bit scan: every partial sum is a colex rank
            // below C(34, 17) < 2^32, so the low half never carries into the high one
            const uint64_t ixy = warp_scan_u64(x | y << 32);
            const uint64_t ix = ixy & 0xffffffffull, iy = ixy >> 32;
            const uint64_t last = __shfl_sync(0xffffffffu, ixy, 31);
            const uint64_t cur_base = last & 0xffffffffull;
            const uint64_t src_base = last >> 32;
            // stream tile (F \ {F_idx}, k-1): elements below keep their position,
            // elements above shift down one
            const uint64_t sbase = (ix - x) + (src_base - iy);
            const uint32_t len = sm.B2[m * kBinomDim + D].x;
            const uint32_t q0 = r0 > cur_base ? (uint32_t)(r0 - cur_base) : 0u;
            const uint32_t q1 = (r1 - cur_base) < len ? (uint32_t)(r1 - cur_base) : len;
            const uint32_t nchunks = q1 > q0 ? (q1 - q0 + CHUNK - 1) / CHUNK : 0u;
            if (nchunks == 0) continue;

            // the low source X(F, k-1): C(D, m-1) entries (+ alignment pad and round-up)
            const uint32_t slen = m >= 1 ? sm.B2[(m - 1) * kBinomDim + D].x : 0u;
            const uint32_t salloc = slen ? (sizeof(T) == 16 ? slen : (slen + 3u) & ~1u) : 0u;
            const int ss = (int)(pub % NHDR);
            tr.ev(8, pub);
            const uint32_t soff = alloc(salloc);
            head = soff + salloc;
            tr.ev(9, pub);
            ++pub;
            queued += nchunks;
            WsHdr<T>& h = sm.hdr[ss];
            if (set) {
                h.coef[idx] = row_sh[D + lane];
                h.sbase[idx] = sbase;
                int mode = 0;
                if ((hints & 3u) != 0) {
                    // the next read of stream tile F' = F \ {h} in this layer comes from
                    // F' + 2^h2 (h2 = lowest free high column above h); beyond the reuse
                    // horizon its lines are marked evict-first
                    const uint32_t Fp = F & ~(1u << lane);
                    const uint32_t z = ~Fp & ((1u << H) - 1u) & ~((2u << lane) - 1u);
                    bool far = true;
                    if (z != 0) far = ((1u << (__ffs(z) - 1)) - (1u << lane)) > (1u << ((hints >> 8) & 31u));
                    mode = far ? 1 : ((hints & 3u) == 2 ? 2 : 0);
                }
                if ((hints & 0x10000u) && lane >= (int)((hints >> 8) & 31u)) mode = 3;  // probe: drop far streams
                h.mode[idx] = mode;
            }
            if (lane == 0) {
                h.m = m;
                // hints bits 28-30: a partial layer without the terms of the top
                // `tcut` columns (they come last in the reference order; the
                // multi-GPU block plan adds them once the exchange has landed)
                const int tcut = (int)((hints >> 28) & 7u);
                h.f = tcut ? __popc(F & ((1u << (H - tcut)) - 1u)) : f;
                h.q1 = q1;
                h.nchunks = nchunks;
                h.cb = q0;
                h.cs = CHUNK;
                h.cur_base = cur_base;
                h.qoff = qoff_sh[m];
                h.pad_src = sizeof(T) == 16 ? 0u : (uint32_t)(src_base & 1u);
                h.src_off = soff;
                h.src_len = salloc;
            }
            {
                // chunk starts cb + i * cs share cb's parity (cs is even)
                const uint32_t cbv = q0;
                const uint32_t pm = __reduce_or_sync(0xffffffffu, set && ((sbase + cbv) & 1u) ? 1u << idx : 0u);
                if (lane == 0) h.padmask = sizeof(T) == 16 ? 0u : pm;
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                const BulkSpan<T> sp = slen ? bulk_span(prev, src_base, slen) : BulkSpan<T>{prev, 0u, 0};
                mbar_arrive(&sm.hdr_full[ss]);  // the streamers may start on the tile now
                mbar_arrive_expect_tx(&sm.src_full[ss], sp.bytes);
                if (sp.bytes) bulk_g2s(sm.src + soff, sp.src, sp.bytes, &sm.src_full[ss]);
            }
            __syncwarp();
        }
        while (pub - rel >= (uint32_t)NHDR) release_one();
        const int ss = (int)(pub % NHDR);
        if (lane == 0) {
            sm.hdr[ss].m = kWsEnd;
            __threadfence_block();
            mbar_arrive(&sm.hdr_full[ss]);
            mbar_arrive(&sm.src_full[ss]);
        }
    } else if (warp >= CW) {
        // ------------------------------------------------------------ streamers
        // Streamer s streams the high-term segments of the chunks of groups
        // g = s mod NST into their rings.
        constexpr int NST = WsSmem<T>::NST;
        const int sid = warp - CW;
        const uint64_t pol_first = l2_evict_first_policy(), pol_last = l2_evict_last_policy();
        uint32_t sqg[G] = {};
        uint32_t gchunk = 0;
        WsTrace tr;
        if (sid == 0) tr.init(2);
        for (uint32_t ts = 0;; ++ts) {
            const int ss = (int)(ts % NHDR);
            mbar_wait_slot(&sm.hdr_full[ss], (ts / NHDR) & 1u);
            const WsHdr<T>& h = sm.hdr[ss];
            if (h.m < 0) break;
            const int f = h.f;
            const uint32_t nchunks = h.nchunks, cb = h.cb, cs = h.cs, q1 = h.q1;
            uint64_t base = 0;
            int mode = 0;
            const int g0 = (int)(gchunk % G);
            gchunk += nchunks;
            for (uint32_t c = 0; c < nchunks; ++c) {
                const int g = (g0 + (int)(c % G)) % G;
                if (g % NST != sid) continue;
                uint32_t& sq = sqg[g];
                const uint32_t c0 = cb + c * cs;
                const uint32_t clen = min((uint32_t)CHUNK, q1 - c0);
                if ((hints & 0x20000u) && c + G < nchunks && lane < f) {
                    // warm L2 with this group's next chunk of the tile (all its streams)
                    const uint32_t n0 = c0 + G * cs;
                    const BulkSpan<T> sp = bulk_span(prev, h.sbase[lane] + n0, min((uint32_t)CHUNK, q1 - n0));
                    bulk_prefetch_l2(sp.src, sp.bytes);
                }
                for (int l0 = 0; l0 < f; l0 += FS, ++sq) {
                    const int nl = min(FS, f - l0);
                    const int s = (int)(sq % NSG);
                    if (lane < nl) {
                        base = h.sbase[l0 + lane];
                        mode = h.mode[l0 + lane];
                    }
                    tr.ev(6, sq);
                    mbar_wait_prod(sm.empty_bar(g, s), ((sq / NSG) & 1u) ^ 1u);
                    tr.ev(7, sq);
                    BulkSpan<T> seg{prev, 0u, 0};
                    if (lane < nl && !(hints & 32u) && mode != 3) seg = bulk_span(prev, base + c0, clen);  // 32: timing probe
                    unsigned bytes;
                    if constexpr (sizeof(T) == 16)
                        bytes = (hints & 0x10020u) ? __reduce_add_sync(0xffffffffu, seg.bytes) : (unsigned)nl * clen * 16u;
                    else
                        bytes = __reduce_add_sync(0xffffffffu, seg.bytes);
                    if (lane == 0) mbar_arrive_expect_tx(sm.full_bar(g, s), bytes);
                    __syncwarp();
                    if (lane < nl && seg.bytes) {
                        if (mode == 0)
                            bulk_g2s(sm.slot(g, s, lane), seg.src, seg.bytes, sm.full_bar(g, s));
                        else
                            bulk_g2s_hint(sm.slot(g, s, lane), seg.src, seg.bytes, sm.full_bar(g, s),
                                          mode == 1 ? pol_first : pol_last);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.src_empty[ss]);
        }
    } else {
        // ------------------------------------------------------------ consumers
        const int g = warp / GW;
        const int j = (warp % GW) * 32 + lane;
        bool use_checked = false;
        if constexpr (R::kChecked) use_checked = guard != nullptr && guard[0] != 0;
        bool ov = false;
        uint32_t seq = 0, gchunk = 0;
        WsTrace tr;
        if (warp % GW == 0 && warp / GW < 2) tr.init(warp / GW);
        for (uint32_t ts = 0;; ++ts) {
            const int ss = (int)(ts % NHDR);
            tr.ev(1, ts);
            mbar_wait_slot(&sm.src_full[ss], (ts / NHDR) & 1u);
            tr.ev(2, ts);
            const WsHdr<T>& h = sm.hdr[ss];
            if (h.m < 0) break;
            // this group's first chunk of the tile (a group with none takes no stages)
            const uint32_t nchunks = h.nchunks;
            const uint32_t c_first = (uint32_t)((g - (int)(gchunk % G) + G) % G);
            gchunk += nchunks;
            if (c_first < nchunks) {
                const uint4* qt = qtab + h.qoff;
                const T* src = sm.src + h.src_off + h.pad_src;
                if constexpr (R::kChecked) {
                    if (use_checked) {
                        ws_consume_dispatch<R>(sm, h, src, qt, cur, g, j, c_first, seq, ov, hints, tr);
                    } else {
                        ws_consume_dispatch<RU>(sm, h, src, qt, cur, g, j, c_first, seq, ov, hints, tr);
                    }
                } else {
                    ws_consume_dispatch<R>(sm, h, src, qt, cur, g, j, c_first, seq, ov, hints, tr);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.src_empty[ss]);
        }
        if (ov) atomicOr(status, 1);
    }
    if (PL_WS_TRIGGER == 2) {
        // every output of this CTA stored and made visible device-wide, then
        // let the next layer's grid start its prologue
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
        }
    }
}

}  // namespace pl
