// C ABI of the B200 Store-zechin engine (include/permlab_b200.h).
//
// Host-side orchestration only: argument checks mirroring the reference's
// guards (reference proj/src/permanent.cpp:232-240, :143-149), device
// scratch from the stream-ordered allocator, kernel selection by order, and
// error mapping. No CPU arithmetic path exists: without a device every
// compute call fails with PL_ERR_NODEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <map>
#include <vector>
#include <type_traits>

#include "../../include/permlab_b200.h"
#include "sz_kernels.cuh"
#include "sz_ws.cuh"
#include "sz_lean.cuh"
#include "capi_internal.h"

namespace {

thread_local std::string g_err;

// Host binomial table C(s, l), s, l < 35 (the table builders below used to
// recompute every coefficient by a loop: 8.9 ms for the D = 14 low-term table).
uint32_t hbinom(int s, int l) {
    static const std::vector<uint32_t> t = [] {
        std::vector<uint32_t> v(pl::kBinomDim * pl::kBinomDim, 0);
        for (int a = 0; a < pl::kBinomDim; ++a)
            for (int b = 0; b <= a; ++b) v[a * pl::kBinomDim + b] = (uint32_t)pl::binom_u64(a, b);
        return v;
    }();
    return (l < 0 || l > s) ? 0u : t[s * pl::kBinomDim + l];
}

// PL_COLD_LOG=1: durations of the one-time builds (tables, tile lists, scratch
// allocations) on stderr -- where a cold first call spends its time.
struct ColdLog {
    const char* what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit ColdLog(const char* w) : what(w) {}
    ~ColdLog() {
        static const bool on = std::getenv("PL_COLD_LOG") != nullptr;
        if (on) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            std::fprintf(stderr, "[pl cold] %s %.2f ms\n", what, ms);
        }
    }
};

pl_status fail(pl_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

pl_status cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(PL_ERR_NOMEM, "%s: %s", what, cudaGetErrorString(e));
    }
    return fail(PL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

pl_status cuda_fail_if(cudaError_t e, const char* what) { return e == cudaSuccess ? PL_OK : cuda_fail(e, what); }

#define PL_CUDA(expr)                                        \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
    } while (0)

size_t elem_size(pl_dtype d) { return d == PL_C128 ? 16 : 8; }

bool valid_dtype(pl_dtype d) { return d == PL_I64 || d == PL_F64 || d == PL_C128; }

uint64_t max_layer(int n) {
    uint64_t m = 0;
    for (int k = 2; k <= n - 1; ++k) m = std::max<uint64_t>(m, pl::binom_u64(n, k));
    return m;
}

// ---------------------------------------------------------------- layer scratch
// Large-order scratch (two layers: up to 2 x 9.6 GB at n = 32 complex) comes
// from plain cudaMalloc blocks kept in a per-device cache: a first 19 GB
// cudaMallocAsync costs ~115 ms (and returning it to the OS as much again,
// profiles/r2/alloc_probe.cu), cudaMalloc ~2 ms. A call takes a free block of
// sufficient size (or allocates one), and hands it back when its stream
// reaches the end of the call (host callback), so concurrent calls never
// share scratch. pl_release_scratch() frees the idle blocks; with
// PL_SCRATCH_CACHE=0 every synchronous call does so before returning.
using plc::ScratchBlock;

// An idle block remembers the stream of its last use and an event recorded
// there at the end of that use: a call on the same stream reuses it at once
// (stream order), a call on another stream first waits for the event. No host
// callback sits in the stream (a cudaLaunchHostFunc node stalls the stream
// until a driver thread has run it: ~0.3 ms per C4 call, round 2).
struct IdleBlock {
    ScratchBlock b;
    cudaEvent_t ev = nullptr;  // null: no use pending
    cudaStream_t st = nullptr;
};

struct ScratchCache {
    std::mutex mu;
    std::vector<IdleBlock> idle;
};

ScratchCache& scratch_cache() {
    static ScratchCache* c = new ScratchCache;  // never destroyed: calls may still run at exit
    return *c;
}

bool scratch_caching() {
    static const bool on = [] {
        const char* e = std::getenv("PL_SCRATCH_CACHE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Block for a call on stream `st` (may be null: the caller then synchronises
// with the block's last use itself, see scratch_acquire_sync).
pl_status scratch_acquire_on(size_t bytes, cudaStream_t st, ScratchBlock* out) {
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    IdleBlock got;
    bool have = false;
    {
        ScratchCache& c = scratch_cache();
        std::lock_guard<std::mutex> lock(c.mu);
        int best = -1;
        for (int i = 0; i < (int)c.idle.size(); ++i) {
            const ScratchBlock& b = c.idle[i].b;
            if (b.dev == dev && b.bytes >= bytes && (best < 0 || b.bytes < c.idle[best].b.bytes)) best = i;
        }
        if (best >= 0) {
            got = c.idle[best];
            c.idle.erase(c.idle.begin() + best);
            have = true;
        }
    }
    if (have) {
        if (got.ev) {
            cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
            cudaError_t e = cudaSuccess;
            if (got.st != st && cap == cudaStreamCaptureStatusNone) {
                e = cudaStreamWaitEvent(st, got.ev, 0);
            } else if (got.st != st) {
                // a capture cannot depend on uncaptured work: wait for it on the host
                // (relaxed mode for this thread: a global-mode capture forbids the sync)
                cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
                cudaThreadExchangeStreamCaptureMode(&mode);
                e = cudaEventSynchronize(got.ev);
                cudaThreadExchangeStreamCaptureMode(&mode);
            }
            cudaEventDestroy(got.ev);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent(scratch)");
        }
        *out = got.b;
        return PL_OK;
    }
    void* p = nullptr;
    ColdLog cl("scratch cudaMalloc");
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        // idle blocks of this device may be holding the memory: drop them and retry
        cudaGetLastError();
        pl_release_scratch();
        e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(layer scratch)");
    *out = ScratchBlock{p, bytes, dev};
    return PL_OK;
}


// A block whose use has completed (the caller synchronised).
void scratch_return_idle(const ScratchBlock& b) {
    ScratchCache& c = scratch_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    c.idle.push_back(IdleBlock{b, nullptr, nullptr});
}

pl_status scratch_release_on_stream(const ScratchBlock& b, cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
    if (cap != cudaStreamCaptureStatusNone) {
        // captured into a CUDA graph: every replay uses this block, so the graph
        // owns it for the life of the process
        return PL_OK;
    }
    cudaEvent_t ev = nullptr;
    PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const cudaError_t e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) {
        cudaEventDestroy(ev);
        return cuda_fail(e, "cudaEventRecord(scratch)");
    }
    ScratchCache& c = scratch_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    c.idle.push_back(IdleBlock{b, ev, st});
    return PL_OK;
}

pl_status have_device() {
    static const int count = [] {
        ColdLog cl("device count");
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        return c;
    }();
    if (count == 0) return fail(PL_ERR_NODEVICE, "no CUDA device available (the engine has no CPU fallback)");
    // Per-call buffers of the host-pointer paths (inputs, outputs, status
    // words) come from the stream-ordered pool: keep up to PL_POOL_KEEP_MB
    // (default 1024) of freed pool memory mapped between calls, so a call
    // does not re-map its staging buffers (layer scratch is separate, above).
    static std::once_flag pool_once[64];
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
        std::call_once(pool_once[dev], [dev] {
            ColdLog cl("pool attributes");
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                const char* e = std::getenv("PL_POOL_KEEP_MB");
                uint64_t keep = (e ? std::strtoull(e, nullptr, 10) : 1024ull) << 20;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            cudaGetLastError();
        });
    }
    return PL_OK;
}

pl_status check_order(int n, const pl_limits* lim) {
    pl_limits d;
    pl_limits_default(&d);
    const pl_limits& L = lim ? *lim : d;
    if (n < 1) return fail(PL_ERR_ARG, "matrix order must be >= 1");
    if (n > L.subset_order_limit) {
        return fail(PL_ERR_LIMIT, "matrix order exceeds subset_order_limit (%d)", L.subset_order_limit);
    }
    if (n > PL_MAX_ORDER) return fail(PL_ERR_LIMIT, "column-subset algorithms support order <= %d", PL_MAX_ORDER);
    return PL_OK;
}

pl_status check_budget(pl_dtype dt, int n, const pl_limits* lim) {
    if (!lim || lim->memo_budget_bytes == 0) return PL_OK;
    if (pl_sz_scratch_bytes(dt, n) > lim->memo_budget_bytes) {
        return fail(PL_ERR_LIMIT, "store-zechin memo table exceeds the configured memory budget");
    }
    return PL_OK;
}

// ---------------------------------------------------------------- dispatch helpers

template <class F>
pl_status with_ring(pl_dtype dt, bool fma, F&& f) {
    switch (dt) {
        case PL_I64:
            return f(pl::RI64<true>{});
        case PL_F64:
            return fma ? f(pl::RF64<true>{}) : f(pl::RF64<false>{});
        case PL_C128:
            return fma ? f(pl::RC128<true>{}) : f(pl::RC128<false>{});
    }
    // internal: the residue passes of the exact big-integer path (bigint.cu)
    if (dt == plc::kModDtype) return f(pl::RModP{});
    return fail(PL_ERR_ARG, "unknown dtype");
}

int num_sms();

// Raise a kernel's MaxDynamicSharedMemorySize only when a launch needs more
// than any earlier one (the attribute is a per-kernel maximum: lowering it
// would invalidate larger launches of the same kernel).
template <class K>
cudaError_t set_smem_once(K kern, size_t bytes) {
    static std::mutex mu;
    static std::map<const void*, size_t> cur;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = cur[reinterpret_cast<const void*>(kern)];
    if (bytes <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

// Tile tickets of one layer range (see sz_ws.cuh): the valid high sets F of
// layer k (popcount in [max(0, k - D), min(k, H)]) from the range's first
// one on, in increasing order. valid_below(X) counts the valid F < X.
uint64_t valid_below(uint64_t X, int H, int fmin, int fmax) {
    uint64_t c = 0;
    int p = 0;
    for (int b = H; b >= 0; --b) {
        if (b == H) {
            if (X >> H) {  // X = 2^H: every valid F counts
                for (int j = fmin; j <= fmax; ++j) c += pl::binom_u64(H, j);
                return c;
            }
            continue;
        }
        if ((X >> b) & 1) {
            for (int j = std::max(0, fmin - p); j <= std::min(b, fmax - p); ++j) c += pl::binom_u64(b, j);
            ++p;
        }
    }
    return c;
}

struct Tickets {
    uint32_t rank0 = 0, ntiles = 0;
};

Tickets layer_tickets(int n, int k, int D, uint64_t r0, uint64_t r1) {
    const int H = n - D;
    const int fmin = std::max(0, k - D), fmax = std::min(k, H);
    const uint64_t F0 = pl_colex_unrank(k, r0) >> D;
    const uint64_t F1 = pl_colex_unrank(k, r1 - 1) >> D;
    Tickets t;
    t.rank0 = (uint32_t)valid_below(F0, H, fmin, fmax);
    t.ntiles = (uint32_t)(valid_below(F1 + 1, H, fmin, fmax) - t.rank0);
    return t;
}

// Every layer's list of valid high sets (sz_tile_list_kernel), generated on
// the device once per (device, n, D) -- at most a few tens of MB (n = 32:
// ~7.6 M entries) -- and freed by pl_release_scratch.
struct TileLists {
    uint32_t* buf = nullptr;
    std::vector<uint64_t> off;  // off[k]: first entry of layer k
};

std::mutex g_lists_mu;
std::map<std::vector<int>, TileLists>& lists_cache() {
    static auto* m = new std::map<std::vector<int>, TileLists>;
    return *m;
}

pl_status get_tile_lists(int n, int D, const uint32_t** layer_base, int k) {
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_lists_mu);
    auto& cache = lists_cache();
    const std::vector<int> key = {dev, n, D};
    auto it = cache.find(key);
    if (it == cache.end()) {
        ColdLog cl("tile lists");
        const int H = n - D;
        TileLists L;
        L.off.assign(n + 1, 0);
        uint64_t total = 0;
        for (int kk = 3; kk <= n - 1; ++kk) {
            L.off[kk] = total;
            const int fmin = std::max(0, kk - D), fmax = std::min(kk, H);
            total += valid_below(1ull << H, H, fmin, fmax);
        }
        L.off[n] = total;
        PL_CUDA(cudaMalloc(&L.buf, std::max<uint64_t>(total, 1) * sizeof(uint32_t)));
        cudaStream_t st;
        PL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (int kk = 3; kk <= n - 1; ++kk) {
            const int fmin = std::max(0, kk - D), fmax = std::min(kk, H);
            const uint32_t cnt = (uint32_t)(L.off[kk + 1] - L.off[kk]);
            if (cnt == 0) continue;
            const unsigned blocks = (unsigned)std::min<uint64_t>((cnt + 255) / 256, 4096);
            pl::sz_tile_list_kernel<<<blocks, 256, 0, st>>>(H, fmin, fmax, cnt, L.buf + L.off[kk]);
        }
        const cudaError_t e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        PL_CUDA(e);
        PL_CUDA(cudaGetLastError());
        it = cache.emplace(key, std::move(L)).first;
    }
    *layer_base = it->second.buf + it->second.off[k];
    return PL_OK;
}

// L2 hint mode of the layer kernel (bits 0-1 stream policy: 0 none, 1 evict-first beyond
// the reuse horizon, 2 + evict-last within it; bit 2 evict-first output stores; bits 8-15
// log2 of the horizon in tiles; bits 4+ are timing probes, see sz_ws.cuh). Default: far
// streams and output stores evict-first, horizon 2^9 tiles. PL_WS_HINTS overrides it.
uint32_t ws_hints() {
    static const uint32_t h = [] {
        const char* e = std::getenv("PL_WS_HINTS");
        return (e ? (uint32_t)std::strtoul(e, nullptr, 0) : 0x905u) & 0x7fffffffu;  // bit 31: see loaded_dep
    }();
    return h;
}

// Low-window width D of the tiled layer kernel: as wide as one tile source
// (C(D, D/2) entries) fits a shared-memory slot (ws_window), but leaving >= 10
// high columns so a layer has enough tiles (>= 2^10 high masks) to keep every
// SM busy. PL_WS_WINDOW narrows it for tuning.
int tile_window(size_t elem, int n) {
    static const int override_d = [] {
        const char* e = std::getenv("PL_WS_WINDOW");  // tuning/debug override of the window width
        return e ? std::atoi(e) : 0;
    }();
    if (override_d > 0) return std::max(1, std::min({override_d, pl::ws_window((int)elem), n - 1}));
    return std::max(1, std::min(pl::ws_window((int)elem), n - 10));
}

struct Qtab {
    uint4* ltab = nullptr;         // low-term table, 16 u16 entries (two uint4) per low subset
    uint32_t* offs = nullptr;      // offs[m]: first uint4 of the m-subsets
    uint2* binom_pairs = nullptr;  // [i * 35 + s] = (C(s, i), C(s, i - 1)), shared by every D
};

// Low-term table for window D on the current device, built once on the host.
// For the m-subset V of [0, D) of colex rank q, entry i (ascending v_i) is
//     rank_D(V \ {v_i}) | v_i << 12
// at u16 index 16 * (offs[m] / 2 + q) + i: the consumer reads its output's
// whole list with one or two 16-byte loads instead of unranking V.
pl_status get_qtab(int D, Qtab* out) {
    static_assert(pl::kWsLtabRankBits == 12, "ltab entry layout");
    static std::mutex mu;
    static std::map<std::pair<int, int>, Qtab> cache;
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, D});
    if (it != cache.end()) {
        *out = it->second;
        return PL_OK;
    }
    if (D > 14) return fail(PL_ERR_LIMIT, "layer window %d exceeds the low-term table layout (<= 14)", D);
    ColdLog cl("ltab build");
    std::vector<uint32_t> offs(D + 2, 0);
    for (int m = 0; m <= D; ++m) offs[m + 1] = offs[m] + 2u * (uint32_t)pl::binom_u64(D, m);
    std::vector<uint16_t> tab((size_t)offs[D + 1] * 8, 0);
    for (uint32_t mask = 0; mask < (1u << D); ++mask) {
        const int m = __builtin_popcount(mask);
        uint32_t r = 0;
        int i = 1;
        for (uint32_t mm = mask; mm; mm &= mm - 1, ++i) r += hbinom(__builtin_ctz(mm), i);
        uint16_t* e = &tab[(size_t)(offs[m] / 2 + r) * 16];
        int t = 0;
        for (uint32_t mm = mask; mm; mm &= mm - 1, ++t) {
            const int v = __builtin_ctz(mm);
            const uint32_t rest = mask & ~(1u << v);
            uint32_t rr = 0;
            int l = 1;
            for (uint32_t q = rest; q; q &= q - 1, ++l) rr += hbinom(__builtin_ctz(q), l);
            e[t] = (uint16_t)(rr | (uint32_t)v << pl::kWsLtabRankBits);
        }
    }
    Qtab q;
    std::vector<uint2> bp(pl::kBinomDim * pl::kBinomDim);
    for (int i = 0; i < pl::kBinomDim; ++i)
        for (int sc = 0; sc < pl::kBinomDim; ++sc)
            bp[i * pl::kBinomDim + sc] = make_uint2((uint32_t)pl::binom_u64(sc, i), i >= 1 ? (uint32_t)pl::binom_u64(sc, i - 1) : 0u);
    PL_CUDA(cudaMalloc(&q.binom_pairs, bp.size() * sizeof(uint2)));
    PL_CUDA(cudaMemcpy(q.binom_pairs, bp.data(), bp.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    PL_CUDA(cudaMalloc(&q.ltab, tab.size() * sizeof(uint16_t)));
    PL_CUDA(cudaMalloc(&q.offs, offs.size() * sizeof(uint32_t)));
    PL_CUDA(cudaMemcpy(q.ltab, tab.data(), tab.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    PL_CUDA(cudaMemcpy(q.offs, offs.data(), offs.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    cache[{dev, D}] = q;
    *out = q;
    return PL_OK;
}

int num_sms() {
    static int sms = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    });
    return sms;
}

// Compact low-term table of the lean kernel (sz_lean.cuh, ln_ltab): the m
// entries of the m-subset V of [0, D) in one uint4 (m <= 8) or two (m > 8);
// offs[m] in uint4 units. D <= 12: at most 70 KB (D = 10: 20 KB), L1-resident.
struct LtabCompact {
    uint4* ltab = nullptr;
    uint32_t* offs = nullptr;
};

pl_status get_ltab_compact(int D, LtabCompact* out) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, LtabCompact> cache;
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, D});
    if (it != cache.end()) {
        *out = it->second;
        return PL_OK;
    }
    if (D > pl::kLnMaxD) return fail(PL_ERR_LIMIT, "lean layer window %d exceeds %d", D, pl::kLnMaxD);
    ColdLog cl("compact ltab build");
    std::vector<uint32_t> offs(D + 2, 0);
    for (int m = 0; m <= D; ++m) offs[m + 1] = offs[m] + (m <= 8 ? 1u : 2u) * (uint32_t)pl::binom_u64(D, m);
    std::vector<uint16_t> tab((size_t)offs[D + 1] * 8, 0);
    for (uint32_t mask = 0; mask < (1u << D); ++mask) {
        const int m = __builtin_popcount(mask);
        uint32_t r = 0;
        int i = 1;
        for (uint32_t mm = mask; mm; mm &= mm - 1, ++i) r += hbinom(__builtin_ctz(mm), i);
        uint16_t* e = &tab[((size_t)offs[m] + (size_t)r * (m <= 8 ? 1 : 2)) * 8];
        int t = 0;
        for (uint32_t mm = mask; mm; mm &= mm - 1, ++t) {
            const int v = __builtin_ctz(mm);
            const uint32_t rest = mask & ~(1u << v);
            uint32_t rr = 0;
            int l = 1;
            for (uint32_t q = rest; q; q &= q - 1, ++l) rr += hbinom(__builtin_ctz(q), l);
            e[t] = (uint16_t)(rr | (uint32_t)v << pl::kWsLtabRankBits);
        }
    }
    LtabCompact q;
    PL_CUDA(cudaMalloc(&q.ltab, std::max<size_t>(tab.size(), 8) * sizeof(uint16_t)));
    PL_CUDA(cudaMalloc(&q.offs, offs.size() * sizeof(uint32_t)));
    PL_CUDA(cudaMemcpy(q.ltab, tab.data(), tab.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    PL_CUDA(cudaMemcpy(q.offs, offs.data(), offs.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    cache[{dev, D}] = q;
    *out = q;
    return PL_OK;
}

// Layer kernel choice: the lean kernel (sz_lean.cuh) for layers of at most
// PL_LEAN_MAX_MB (default 24) -- the outer layers, where the warp-specialised
// kernel's per-tile pipeline latency dominates (C4 k <= 8, k >= 17: 9-36 us
// against 11-46 us per layer, profiles/r2b) -- and the warp-specialised
// kernel (sz_ws.cuh) for the large middle layers, where its staged streams
// keep more loads in flight. PL_LAYER_KERNEL=lean|ws forces one.
bool use_lean_layer(size_t elem, int n, int k) {
    static const int force = [] {
        const char* e = std::getenv("PL_LAYER_KERNEL");
        if (e && std::string(e) == "lean") return 1;
        if (e && std::string(e) == "ws") return 0;
        return -1;
    }();
    if (force >= 0) return force == 1;
    static const uint64_t max_bytes = [] {
        const char* e = std::getenv("PL_LEAN_MAX_MB");
        return (e ? std::strtoull(e, nullptr, 10) : 24ull) << 20;
    }();
    return pl::binom_u64(n, k) * elem <= max_bytes;
}

int lean_window(int n) { return std::max(1, std::min(pl::kLnMaxD, n - 3)); }  // >= 8 high sets per layer

template <class K>
int blocks_per_sm(K kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<const void*, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(reinterpret_cast<const void*>(kern));
    if (it != cache.end()) return it->second;
    int b = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem) != cudaSuccess || b < 1) {
        cudaGetLastError();
        b = 1;
    }
    cache[reinterpret_cast<const void*>(kern)] = b;
    return b;
}

template <class R>
struct Unchecked {
    using type = R;
};
template <>
struct Unchecked<pl::RI64<true>> {
    using type = pl::RI64<false>;
};

// `tickets`: a device word that is zero when this launch starts (the layer
// kernel's tile counter; unused for k = 2).
// `nmat` > 1 (lean kernel only): the same layer of nmat matrices (contiguous
// from `a`, their buffers lstride elements apart; guard[b] per matrix).
template <class R>
pl_status launch_layer(int n, const void* a, int k, const void* prev, void* cur, uint64_t r0, uint64_t r1,
                       uint32_t* tickets, const int32_t* guard, int32_t* status, cudaStream_t st, uint32_t nmat = 1,
                       uint64_t lstride = 0, int top_cut = 0) {
    using T = typename R::T;
    if (r1 <= r0) return PL_OK;
    if (k == 2) {
        const unsigned blocks = (unsigned)std::min<uint64_t>((r1 - r0 + 255) / 256, 1024);
        pl::sz_base_layer_kernel<R><<<blocks, 256, 0, st>>>(static_cast<const T*>(a), n, static_cast<T*>(cur), r0, r1,
                                                            status);
        PL_CUDA(cudaGetLastError());
        return PL_OK;
    }
    if (nmat > 1 || use_lean_layer(sizeof(T), n, k)) {
        const int D = lean_window(n);
        LtabCompact lt;
        pl_status s = get_ltab_compact(D, &lt);
        if (s != PL_OK) return s;
        Qtab qb;
        s = get_qtab(D, &qb);  // binomial pairs
        if (s != PL_OK) return s;
        const Tickets tk = layer_tickets(n, k, D, r0, r1);
        const uint32_t* flist = nullptr;
        s = get_tile_lists(n, D, &flist, k);
        if (s != PL_OK) return s;
        const size_t smem = sizeof(pl::LnSmem<T>);
        auto kern = pl::sz_lean_kernel<R, typename Unchecked<R>::type>;
        constexpr int threads = pl::LnGeom<(int)sizeof(T)>::kThreads;
        static std::once_flag first_lean;
        std::call_once(first_lean, [&] {
            ColdLog cl("lean kernel attributes + occupancy (first use)");
            set_smem_once(kern, smem);
            blocks_per_sm(kern, threads, smem);
        });
        PL_CUDA(set_smem_once(kern, smem));
        const int per_sm = blocks_per_sm(kern, threads, smem);
        constexpr int wpb = pl::LnGeom<(int)sizeof(T)>::WPB;
        const unsigned grid = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>(((uint64_t)tk.ntiles * nmat + wpb - 1) / wpb, (uint64_t)num_sms() * per_sm));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        static const bool pdl_l = [] {
            const char* e = std::getenv("PL_WS_PDL");
            return !(e && e[0] == '0');
        }();
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_l ? 1 : 0;
        PL_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(a), n, k, D, static_cast<const T*>(prev),
                                   static_cast<T*>(cur), r0, r1, flist + tk.rank0, tk.ntiles, nmat, lstride,
                                   static_cast<const uint4*>(lt.ltab), static_cast<const uint32_t*>(lt.offs),
                                   static_cast<const uint2*>(qb.binom_pairs), guard, status, top_cut));
        return PL_OK;
    }
    const int D = tile_window(sizeof(T), n);
    Qtab q;
    pl_status s = get_qtab(D, &q);
    if (s != PL_OK) return s;
    static const int grid = [] {
        const char* e = std::getenv("PL_WS_GRID");  // tuning override of the layer-kernel grid
        return e ? std::max(1, std::min(atoi(e), num_sms())) : num_sms();
    }();
    const Tickets tk = layer_tickets(n, k, D, r0, r1);
    const uint32_t* flist = nullptr;
    s = get_tile_lists(n, D, &flist, k);
    if (s != PL_OK) return s;
    const size_t smem = pl::WsSmem<T>::bytes();
    auto kern = pl::sz_ws_kernel<R, typename Unchecked<R>::type>;
    {
        static std::once_flag first_ws;
        std::call_once(first_ws, [&] {
            ColdLog cl("ws kernel attributes (first use)");
            set_smem_once(kern, smem);
        });
    }
    PL_CUDA(set_smem_once(kern, smem));
    // PL_WS_TRACE=<file> PL_WS_TRACE_K=<k>: event trace of CTA 0 for layer k (debug)
    static const char* trace_path = std::getenv("PL_WS_TRACE");
    static const int trace_k = std::getenv("PL_WS_TRACE_K") ? atoi(std::getenv("PL_WS_TRACE_K")) : -1;
    unsigned long long* trace = nullptr;
    if (trace_path && k == trace_k) {
        const size_t tb = (size_t)4 * pl::kWsTraceCap * 2 * sizeof(unsigned long long);
        PL_CUDA(cudaMalloc(&trace, tb));
        PL_CUDA(cudaMemset(trace, 0, tb));
        PL_CUDA(cudaMemcpyToSymbol(pl::g_ws_trace, &trace, sizeof(trace)));
    }
    // programmatic dependent launch (see sz_ws_kernel): the grid's prologue
    // overlaps the tail of whatever precedes it on the stream
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(pl::WsGeom<(int)sizeof(T)>::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    static const bool pdl = [] {
        const char* e = std::getenv("PL_WS_PDL");  // debug: 0 disables programmatic dependent launch
        return !(e && e[0] == '0');
    }();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    PL_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(a), n, k, D, static_cast<const T*>(prev),
                               static_cast<T*>(cur), r0, r1, tickets, flist + tk.rank0, tk.ntiles,
                               static_cast<const uint4*>(q.ltab), static_cast<const uint32_t*>(q.offs),
                               static_cast<const uint2*>(q.binom_pairs), guard, status,
                               ws_hints() | (uint32_t)(top_cut & 7) << 28));
    if (trace) {
        PL_CUDA(cudaStreamSynchronize(st));
        std::vector<unsigned long long> hb((size_t)4 * pl::kWsTraceCap * 2);
        PL_CUDA(cudaMemcpy(hb.data(), trace, hb.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        unsigned long long* null = nullptr;
        PL_CUDA(cudaMemcpyToSymbol(pl::g_ws_trace, &null, sizeof(null)));
        PL_CUDA(cudaFree(trace));
        if (FILE* fp = std::fopen(trace_path, "wb")) {
            std::fwrite(hb.data(), sizeof(unsigned long long), hb.size(), fp);
            std::fclose(fp);
        }
    }
    return PL_OK;
}

template <class R>
pl_status launch_top(int n, const void* a, const void* last, void* out, const int32_t* guard, int32_t* status,
                     cudaStream_t st) {
    using T = typename R::T;
    pl::sz_top_kernel<R><<<1, 32, 0, st>>>(static_cast<const T*>(a), n, static_cast<const T*>(last),
                                           static_cast<T*>(out), guard, status);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

// Full single-matrix layer DP for one device-resident matrix (n >= 3).
// tickets[k] (k < n) must be zero.
template <class R>
pl_status run_layers(int n, const void* a_dev, void* out_dev, void* buf0, void* buf1, uint32_t* tickets,
                     const int32_t* guard, int32_t* status, cudaStream_t st) {
    void* prev = buf0;
    void* cur = buf1;
    pl_status s = launch_layer<R>(n, a_dev, 2, nullptr, prev, 0, pl::binom_u64(n, 2), nullptr, guard, status, st);
    if (s != PL_OK) return s;
    for (int k = 3; k <= n - 1; ++k) {
        s = launch_layer<R>(n, a_dev, k, prev, cur, 0, pl::binom_u64(n, k), tickets + k, guard, status, st);
        if (s != PL_OK) return s;
        std::swap(prev, cur);
    }
    return launch_top<R>(n, a_dev, prev, out_dev, guard, status, st);
}

// Batches of large orders whose layers all fit the lean kernel (n <= ~22):
// every layer of a group of matrices in one launch (tiles of all the group's
// matrices), instead of one DP (n - 2 launches) per matrix. The group is
// sized so its two layer buffers per matrix fit batch_scratch_bytes() (2 GB).
// PL_BATCH_LAYERS=0: one matrix at a time.
bool batch_layers_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PL_BATCH_LAYERS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// scratch per group of a large-order batch (PL_BATCH_SCRATCH_MB: tests force small groups)
size_t batch_scratch_bytes() {
    static const size_t b = [] {
        const char* e = std::getenv("PL_BATCH_SCRATCH_MB");
        return (e ? std::strtoull(e, nullptr, 10) : 2048ull) << 20;
    }();
    return b;
}

template <class R>
pl_status run_layers_batch(int n, int64_t count, const void* a_dev, void* out_dev, int32_t* status_dev,
                           cudaStream_t st, ScratchBlock* held) {
    using T = typename R::T;
    const uint64_t ml = max_layer(n);
    const uint64_t stride = (ml + 8 + 31) & ~uint64_t(31);  // elements per matrix buffer (256-byte aligned, slack)
    const int64_t group = std::max<int64_t>(1, std::min<int64_t>(count, (int64_t)(batch_scratch_bytes() / (2 * stride * sizeof(T)))));
    constexpr size_t kHead = 256;
    const size_t gbytes = ((size_t)group * sizeof(int32_t) + 255) & ~size_t(255);
    ScratchBlock blk;
    pl_status s = scratch_acquire_on(kHead + gbytes + 2 * (size_t)group * stride * sizeof(T), st, &blk);
    if (s != PL_OK) return s;
    int32_t* guards = reinterpret_cast<int32_t*>(static_cast<char*>(blk.ptr) + kHead);
    T* buf0 = reinterpret_cast<T*>(static_cast<char*>(blk.ptr) + kHead + gbytes);
    T* buf1 = buf0 + (size_t)group * stride;
    for (int64_t g0 = 0; g0 < count && s == PL_OK; g0 += group) {
        const uint32_t nm = (uint32_t)std::min<int64_t>(group, count - g0);
        const T* ag = static_cast<const T*>(a_dev) + (size_t)g0 * n * n;
        T* og = static_cast<T*>(out_dev) + g0;
        const int32_t* gd = nullptr;
        if constexpr (R::kChecked) {
            pl::sz_guard_i64_batch_kernel<<<(nm + 127) / 128, 128, 0, st>>>(reinterpret_cast<const long long*>(ag), n,
                                                                             nm, guards);
            gd = guards;
        }
        const uint64_t c2 = pl::binom_u64(n, 2) * nm;
        pl::sz_base_layer_batch_kernel<R><<<(unsigned)std::min<uint64_t>((c2 + 255) / 256, 4096), 256, 0, st>>>(
            ag, n, buf0, stride, nm, status_dev);
        PL_CUDA(cudaGetLastError());
        T* prev = buf0;
        T* cur = buf1;
        for (int k = 3; k <= n - 1 && s == PL_OK; ++k) {
            s = launch_layer<R>(n, ag, k, prev, cur, 0, pl::binom_u64(n, k), nullptr, gd, status_dev, st, nm, stride);
            std::swap(prev, cur);
        }
        pl::sz_top_batch_kernel<R><<<(nm + 127) / 128, 128, 0, st>>>(ag, n, prev, stride, og, nm, status_dev);
        PL_CUDA(cudaGetLastError());
    }
    if (held) {
        *held = blk;
        return s;
    }
    const pl_status s2 = scratch_release_on_stream(blk, st);
    return s != PL_OK ? s : s2;
}

// Device-side batch compute: a_dev/out_dev device pointers, enqueue only.
// `held`: a synchronous caller takes the large-order scratch block and
// returns it to the cache after its stream synchronisation; otherwise a host
// callback on the stream returns it.
pl_status enqueue_batch(pl_dtype dt, int n, int64_t count, const void* a_dev, void* out_dev, bool fma,
                        int32_t* status_dev, cudaStream_t st, ScratchBlock* held = nullptr) {
    if (count == 0) return PL_OK;
    if (plc::small_order_batch(dt, n)) {
        // n <= 14: register / shared-memory batch kernels (csrc/batch.cu, a module of its own)
        return plc::launch_small_batch(dt, fma, n, count, a_dev, out_dev, status_dev, st);
    }
    // Large orders: one layer DP per matrix through global scratch (a cached
    // cudaMalloc block; returned to the cache when the stream gets there).
    const size_t es = elem_size(dt);
    const uint64_t ml = max_layer(n);
    if (count >= 2 && use_lean_layer(es, n, n / 2) && batch_layers_enabled()) {
        return with_ring(dt, fma, [&](auto r) {
            return run_layers_batch<decltype(r)>(n, count, a_dev, out_dev, status_dev, st, held);
        });
    }
    if (plc::blk_supported(dt, n)) {
        // float rings: the register-blocked engine (sz_blk.cuh), one launch per super-layer
        ScratchBlock blk;
        pl_status s = scratch_acquire_on(plc::blk_scratch_bytes(dt, n), st, &blk);
        if (s != PL_OK) return s;
        for (int64_t b = 0; b < count && s == PL_OK; ++b) {
            s = plc::run_blocks(dt, fma, n, static_cast<const char*>(a_dev) + (size_t)b * n * n * es,
                                static_cast<char*>(out_dev) + (size_t)b * es, blk.ptr, status_dev, st);
        }
        if (held) {
            *held = blk;
            return s;
        }
        const pl_status s2 = scratch_release_on_stream(blk, st);
        return s != PL_OK ? s : s2;
    }
    // Head: tile tickets of every layer (64 words) and the int64 guard flag.
    // Layer buffers carry 64 bytes of slack: 8-byte rings stage 16-byte aligned
    // spans that may read one element past a layer's last entry.
    // Each buffer starts 256-byte aligned (TMA bulk copies need 16).
    constexpr size_t kHead = 512;
    const size_t stride = (ml * es + 64 + 255) & ~size_t(255);
    ScratchBlock blk;
    pl_status s = scratch_acquire_on(kHead + 2 * stride, st, &blk);
    if (s != PL_OK) return s;
    uint32_t* tickets = static_cast<uint32_t*>(blk.ptr);
    int32_t* guards = reinterpret_cast<int32_t*>(static_cast<char*>(blk.ptr) + 256);
    char* bufs = static_cast<char*>(blk.ptr) + kHead;
    for (int64_t b = 0; b < count && s == PL_OK; ++b) {
        const char* ab = static_cast<const char*>(a_dev) + (size_t)b * n * n * es;
        char* ob = static_cast<char*>(out_dev) + (size_t)b * es;
        s = cuda_fail_if(cudaMemsetAsync(blk.ptr, 0, kHead, st), "cudaMemsetAsync(tickets)");
        if (s != PL_OK) break;
        if (dt == PL_I64) {
            pl::sz_guard_i64_kernel<<<1, 1, 0, st>>>(reinterpret_cast<const long long*>(ab), n, guards);
        }
        s = with_ring(dt, fma, [&](auto r) {
            return run_layers<decltype(r)>(n, ab, ob, bufs, bufs + stride, tickets, guards, status_dev, st);
        });
    }
    if (held) {
        *held = blk;
        return s;
    }
    const pl_status s2 = scratch_release_on_stream(blk, st);
    return s != PL_OK ? s : s2;
}

// Host-pointer batches of batched orders: the batch moves in chunks so that the
// upload of chunk i + 1 (copy stream), the kernel of chunk i (the caller's
// stream) and the download of chunk i - 1 (second copy stream, the other PCIe
// direction) overlap; the call then costs about the upload alone.
constexpr size_t kPipeMinBytes = size_t(8) << 20;
constexpr size_t kPipeChunkBytes = size_t(8) << 20;
#ifndef PL_HOST_UP_DEFAULT
#define PL_HOST_UP_DEFAULT 1
#endif
constexpr int kDefaultUpStreams = PL_HOST_UP_DEFAULT;

constexpr int kMaxUpStreams = 4;

struct CopyStreams {
    cudaStream_t up[kMaxUpStreams] = {};
    cudaStream_t down = nullptr;
};

// Upload streams of the host pipeline: chunk c goes up on stream c mod N, so N
// copies can be in flight on different copy engines (PL_HOST_UP_STREAMS).
int host_up_streams() {
    static const int nup = [] {
        const char* e = std::getenv("PL_HOST_UP_STREAMS");
        return e ? std::max(1, std::min(kMaxUpStreams, atoi(e))) : kDefaultUpStreams;
    }();
    return nup;
}

pl_status copy_streams(CopyStreams* out) {
    static thread_local std::map<int, CopyStreams> cache;  // per thread and device
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    auto it = cache.find(dev);
    if (it == cache.end()) {
        CopyStreams cs;
        for (int i = 0; i < kMaxUpStreams; ++i) PL_CUDA(cudaStreamCreateWithFlags(&cs.up[i], cudaStreamNonBlocking));
        PL_CUDA(cudaStreamCreateWithFlags(&cs.down, cudaStreamNonBlocking));
        it = cache.emplace(dev, cs).first;
    }
    *out = it->second;
    return PL_OK;
}

pl_status pipelined_host_batch(pl_dtype dt, int n, int64_t count, const void* a, void* out, void* a_dev,
                               void* out_dev, bool fma, int32_t* status_dev, cudaStream_t st) {
    CopyStreams cs;
    pl_status s = copy_streams(&cs);
    if (s != PL_OK) return s;
    const size_t es = elem_size(dt);
    const size_t mat_bytes = (size_t)n * n * es;
    static const size_t chunk_bytes = [] {
        const char* e = std::getenv("PL_HOST_CHUNK_MB");  // tuning: chunk size of the host pipeline
        return e ? std::max<size_t>(1, (size_t)atoi(e)) << 20 : kPipeChunkBytes;
    }();
    const int64_t per = std::max<int64_t>(32, (int64_t)(chunk_bytes / mat_bytes) / 32 * 32);
    const int64_t nchunks = (count + per - 1) / per;
    std::vector<cudaEvent_t> evs;
    auto make_event = [&](cudaEvent_t* e) -> pl_status {
        PL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        evs.push_back(*e);
        return PL_OK;
    };
    const int nup = (int)std::min<int64_t>(host_up_streams(), nchunks);
    cudaEvent_t start;
    s = make_event(&start);
    if (s == PL_OK) s = cuda_fail_if(cudaEventRecord(start, st), "cudaEventRecord");
    for (int i = 0; i < nup && s == PL_OK; ++i)
        s = cuda_fail_if(cudaStreamWaitEvent(cs.up[i], start, 0), "cudaStreamWaitEvent");
    if (s == PL_OK) s = cuda_fail_if(cudaStreamWaitEvent(cs.down, start, 0), "cudaStreamWaitEvent");
    for (int64_t c = 0; c < nchunks && s == PL_OK; ++c) {
        const int64_t b0 = c * per, b1 = std::min<int64_t>(count, b0 + per);
        const size_t off_in = (size_t)b0 * mat_bytes, len_in = (size_t)(b1 - b0) * mat_bytes;
        cudaEvent_t up_done, k_done;
        if ((s = make_event(&up_done)) != PL_OK || (s = make_event(&k_done)) != PL_OK) break;
        cudaStream_t up = cs.up[c % nup];
        s = cuda_fail_if(cudaMemcpyAsync(static_cast<char*>(a_dev) + off_in, static_cast<const char*>(a) + off_in,
                                         len_in, cudaMemcpyHostToDevice, up), "cudaMemcpyAsync(in)");
        if (s == PL_OK) s = cuda_fail_if(cudaEventRecord(up_done, up), "cudaEventRecord");
        if (s == PL_OK) s = cuda_fail_if(cudaStreamWaitEvent(st, up_done, 0), "cudaStreamWaitEvent");
        if (s == PL_OK)
            s = enqueue_batch(dt, n, b1 - b0, static_cast<const char*>(a_dev) + off_in,
                              static_cast<char*>(out_dev) + (size_t)b0 * es, fma, status_dev, st);
        if (s == PL_OK) s = cuda_fail_if(cudaEventRecord(k_done, st), "cudaEventRecord");
        if (s == PL_OK) s = cuda_fail_if(cudaStreamWaitEvent(cs.down, k_done, 0), "cudaStreamWaitEvent");
        if (s == PL_OK)
            s = cuda_fail_if(cudaMemcpyAsync(static_cast<char*>(out) + (size_t)b0 * es,
                                             static_cast<char*>(out_dev) + (size_t)b0 * es, (size_t)(b1 - b0) * es,
                                             cudaMemcpyDeviceToHost, cs.down),
                             "cudaMemcpyAsync(out)");
    }
    // the caller's stream continues after every download (and every upload)
    for (int i = 0; i < nup && s == PL_OK; ++i) {
        cudaEvent_t up_all;
        if ((s = make_event(&up_all)) != PL_OK) break;
        s = cuda_fail_if(cudaEventRecord(up_all, cs.up[i]), "cudaEventRecord");
        if (s == PL_OK) s = cuda_fail_if(cudaStreamWaitEvent(st, up_all, 0), "cudaStreamWaitEvent");
    }
    cudaEvent_t down_all;
    if (s == PL_OK && (s = make_event(&down_all)) == PL_OK) {
        s = cuda_fail_if(cudaEventRecord(down_all, cs.down), "cudaEventRecord");
        if (s == PL_OK) s = cuda_fail_if(cudaStreamWaitEvent(st, down_all, 0), "cudaStreamWaitEvent");
    }
    for (cudaEvent_t e : evs) cudaEventDestroy(e);  // destruction is deferred until the event completes
    return s;
}

// Synchronous wrapper: owns device copies for host pointers and a status
// word; waits and maps the status word to PL_ERR_OVERFLOW.
pl_status run_batch(pl_dtype dt, int n, int64_t count, const void* a, void* out, uint32_t flags,
                    int32_t* status_dev_user, cudaStream_t st) {
    const bool dev_ptrs = flags & PL_FLAG_DEVICE_PTRS;
    const bool fma = flags & PL_FLAG_FMA;
    const bool async = flags & PL_FLAG_ASYNC;
    if (async) {
        if (!dev_ptrs) return fail(PL_ERR_ARG, "PL_FLAG_ASYNC requires PL_FLAG_DEVICE_PTRS");
        if (!status_dev_user) return fail(PL_ERR_ARG, "PL_FLAG_ASYNC requires a device status word");
        return enqueue_batch(dt, n, count, a, out, fma, status_dev_user, st);
    }
    const size_t es = elem_size(dt);
    const size_t in_bytes = (size_t)count * n * n * es;
    const size_t out_bytes = (size_t)count * es;
    void* a_dev = const_cast<void*>(a);
    void* out_dev = out;
    int32_t* status_dev = nullptr;
    PL_CUDA(cudaMallocAsync((void**)&status_dev, sizeof(int32_t), st));
    PL_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int32_t), st));
    if (!dev_ptrs) {
        PL_CUDA(cudaMallocAsync(&a_dev, std::max<size_t>(in_bytes, 16), st));
        PL_CUDA(cudaMallocAsync(&out_dev, std::max<size_t>(out_bytes, 16), st));
    }
    pl_status s = PL_OK;
    bool out_copied = false;
    ScratchBlock held;
    static const bool host_pipe = [] {
        const char* e = std::getenv("PL_HOST_PIPE");  // 0: one upload, one kernel, one download (A/B)
        return !(e && e[0] == '0');
    }();
    if (!dev_ptrs && host_pipe && n <= 14 && in_bytes >= kPipeMinBytes) {
        s = pipelined_host_batch(dt, n, count, a, out, a_dev, out_dev, fma, status_dev, st);
        out_copied = true;
    } else {
        if (!dev_ptrs) PL_CUDA(cudaMemcpyAsync(a_dev, a, in_bytes, cudaMemcpyHostToDevice, st));
        s = enqueue_batch(dt, n, count, a_dev, out_dev, fma, status_dev, st, &held);
    }
    int32_t status_host = 0;
    if (s == PL_OK) {
        if (!dev_ptrs && !out_copied) {
            const cudaError_t e = cudaMemcpyAsync(out, out_dev, out_bytes, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(out)");
        }
        const cudaError_t e2 = cudaMemcpyAsync(&status_host, status_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (s == PL_OK && e2 != cudaSuccess) s = cuda_fail(e2, "cudaMemcpyAsync(status)");
    }
    if (!dev_ptrs) {
        cudaFreeAsync(a_dev, st);
        cudaFreeAsync(out_dev, st);
    }
    cudaFreeAsync(status_dev, st);
    const cudaError_t e3 = cudaStreamSynchronize(st);
    if (s == PL_OK && e3 != cudaSuccess) s = cuda_fail(e3, "cudaStreamSynchronize");
    if (held.ptr) {
        if (e3 == cudaSuccess) {
            scratch_return_idle(held);
        } else {
            cudaFree(held.ptr);  // the stream failed: do not recycle a block that may still be in use
        }
    }
    if (!scratch_caching()) pl_release_scratch();
    if (s == PL_OK && (status_host & PL_STATUS_BIT_OVERFLOW)) {
        s = fail(PL_ERR_OVERFLOW,
                 "int64 overflow: an intermediate sub-permanent does not fit the exact int64 ring");
    }
    return s;
}

pl_status common_checks(pl_dtype dt, int n, int64_t count, const void* a, void* out, const pl_limits* lim) {
    if (!valid_dtype(dt)) return fail(PL_ERR_ARG, "unknown dtype %d", (int)dt);
    if (count < 0) return fail(PL_ERR_ARG, "negative batch count");
    if (count > 0 && (!a || !out)) return fail(PL_ERR_ARG, "null matrix or output pointer");
    pl_status s = check_order(n, lim);
    if (s != PL_OK) return s;
    s = check_budget(dt, n, lim);
    if (s != PL_OK) return s;
    return have_device();
}

}  // namespace

namespace plc {

pl_status fail_msg(pl_status s, const char* msg) { return fail(s, "%s", msg); }
pl_status cuda_error(cudaError_t e, const char* what) { return cuda_fail(e, what); }
pl_status device_ready() { return have_device(); }
int sm_count() { return num_sms(); }
namespace {
thread_local bool tl_input_ready = false;
}
bool input_ready_hint() { return tl_input_ready; }
void set_input_ready_hint(bool on) { tl_input_ready = on; }
pl_status set_modulus(const pl::ModParams* mp, cudaStream_t st) {
    PL_CUDA(cudaMemcpyToSymbolAsync(pl::c_modp, mp, sizeof(pl::ModParams), 0, cudaMemcpyHostToDevice, st));
    return PL_OK;
}
pl_status enqueue_batch(pl_dtype dt, int n, int64_t count, const void* a_dev, void* out_dev, bool fma,
                        int32_t* status_dev, cudaStream_t st) {
    return ::enqueue_batch(dt, n, count, a_dev, out_dev, fma, status_dev, st);
}
pl_status check_order_limits(int n, const pl_limits* lim) { return check_order(n, lim); }
pl_status check_budget_limits(pl_dtype dt, int n, const pl_limits* lim) { return check_budget(dt, n, lim); }
pl_status layer(pl_dtype dt, bool fma, int n, const void* a, int k, const void* prev, void* cur, uint64_t r0,
                uint64_t r1, uint32_t* tickets, const int32_t* guard, int32_t* status, cudaStream_t st, int top_cut) {
    return with_ring(dt, fma, [&](auto r) {
        return launch_layer<decltype(r)>(n, a, k, prev, cur, r0, r1, tickets, guard, status, st, 1, 0, top_cut);
    });
}
pl_status top_terms(pl_dtype dt, bool fma, int n, const void* a, int k, const void* prev, void* cur, uint64_t base,
                    uint64_t len, int nsrc, const int* cols, const uint64_t* src_bases, bool init_first, int32_t* status,
                    cudaStream_t st) {
    if (len == 0 || nsrc == 0) return PL_OK;
    if (nsrc > 8) return fail(PL_ERR_ARG, "at most 8 top columns");
    pl::TopSrc src{};
    for (int i = 0; i < nsrc; ++i) {
        src.col[i] = cols[i];
        src.base[i] = src_bases[i];
    }
    return with_ring(dt, fma, [&](auto r) {
        using R = decltype(r);
        using T = typename R::T;
        const unsigned blocks = (unsigned)std::min<uint64_t>((len + 255) / 256, (uint64_t)num_sms() * 8);
        pl::sz_top_terms_kernel<R><<<blocks, 256, 0, st>>>(static_cast<const T*>(a), n, k, static_cast<const T*>(prev),
                                                           static_cast<T*>(cur), base, len, nsrc, src, init_first ? 1 : 0,
                                                           status);
        PL_CUDA(cudaGetLastError());
        return PL_OK;
    });
}
pl_status top(pl_dtype dt, bool fma, int n, const void* a, const void* last, void* out, const int32_t* guard,
              int32_t* status, cudaStream_t st) {
    return with_ring(dt, fma, [&](auto r) { return launch_top<decltype(r)>(n, a, last, out, guard, status, st); });
}
pl_status guard_i64(int n, const void* a, int32_t* guard, cudaStream_t st) {
    pl::sz_guard_i64_kernel<<<1, 1, 0, st>>>(static_cast<const long long*>(a), n, guard);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}
pl_status scratch_get(size_t bytes, cudaStream_t st, ScratchBlock* out) { return ::scratch_acquire_on(bytes, st, out); }
pl_status scratch_put(const ScratchBlock& b, cudaStream_t st) { return ::scratch_release_on_stream(b, st); }

}  // namespace plc

extern "C" {

const char* pl_version(void) { return "permlab-b200 0.1.0 (sm_100a)"; }

const char* pl_last_error(void) { return g_err.c_str(); }

void pl_limits_default(pl_limits* out) {
    if (!out) return;
    out->subset_order_limit = PL_MAX_ORDER;
    out->memo_budget_bytes = 0;
    out->num_gpus = 0;
}

int32_t pl_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

uint64_t pl_binom(int32_t s, int32_t k) {
    if (s < 0 || k < 0 || k > s || s > 64) return 0;
    return pl::binom_u64(s, k);
}

uint64_t pl_colex_rank(uint64_t mask) {
    uint64_t r = 0;
    int i = 1;
    while (mask) {
        const int s = __builtin_ctzll(mask);
        r += pl::binom_u64(s, i++);
        mask &= mask - 1;
    }
    return r;
}

uint64_t pl_colex_unrank(int32_t k, uint64_t rank) {
    uint64_t mask = 0;
    int s = 63;
    for (int i = k; i >= 1; --i) {
        while (s >= 0 && pl::binom_u64(s, i) > rank) --s;
        if (s < 0) return 0;
        mask |= 1ull << s;
        rank -= pl::binom_u64(s, i);
        --s;
    }
    return mask;
}

uint64_t pl_sz_scratch_bytes(pl_dtype dtype, int32_t n) {
    if (n < 3 || n > 64) return 0;
    return 2 * max_layer(n) * elem_size(dtype);
}

pl_status pl_sz_counts(int32_t n, uint64_t* mults, uint64_t* adds) {
    if (n < 1 || n > 63 || !mults || !adds) return fail(PL_ERR_ARG, "bad arguments to pl_sz_counts");
    if (n == 1) {
        *mults = 0;
        *adds = 0;
    } else if (n == 2) {
        *mults = 2;
        *adds = 1;
    } else {
        const uint64_t half = 1ull << (n - 1);
        *mults = (uint64_t)n * half - (uint64_t)n;
        *adds = (uint64_t)n * half - 2 * half + 1;
    }
    return PL_OK;
}

pl_status pl_sz_diagnostics(int32_t n, uint64_t* misses, uint64_t* distinct) {
    if (n < 1 || n > 63 || !misses || !distinct) return fail(PL_ERR_ARG, "bad arguments to pl_sz_diagnostics");
    const uint64_t v = n == 1 ? 0 : n == 2 ? 1 : (1ull << n) - (uint64_t)n - 2;
    *misses = v;
    *distinct = v;
    return PL_OK;
}

pl_status pl_sz_permanent_batch(pl_dtype dtype, int32_t n, int64_t count, const void* a, void* out, uint32_t flags,
                                const pl_limits* limits, void* stream, int32_t* status_dev) {
    pl_status s = common_checks(dtype, n, count, a, out, limits);
    if (s != PL_OK) return s;
    if (limits && limits->num_gpus >= 1) {
        return plc::run_multi(dtype, n, count, a, out, flags, limits, nullptr, static_cast<cudaStream_t>(stream));
    }
    // device pointers only: a host batch is uploaded by this call, so its input is never "ready"
    plc::set_input_ready_hint((flags & PL_FLAG_INPUT_READY) && (flags & PL_FLAG_DEVICE_PTRS));
    s = run_batch(dtype, n, count, a, out, flags, status_dev, static_cast<cudaStream_t>(stream));
    plc::set_input_ready_hint(false);
    return s;
}

pl_status pl_sz_permanent(pl_dtype dtype, int32_t n, const void* a, void* out, uint32_t flags,
                          const pl_limits* limits, void* stream) {
    if (flags & PL_FLAG_ASYNC) return fail(PL_ERR_ARG, "pl_sz_permanent is synchronous; use the batch entry point");
    pl_status s = common_checks(dtype, n, 1, a, out, limits);
    if (s != PL_OK) return s;
    if (limits && limits->num_gpus >= 1) {
        return plc::run_multi(dtype, n, 1, a, out, flags, limits, nullptr, static_cast<cudaStream_t>(stream));
    }
    return run_batch(dtype, n, 1, a, out, flags, nullptr, static_cast<cudaStream_t>(stream));
}

pl_status pl_sz_layer(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev, void* cur_dev,
                      uint64_t r0, uint64_t r1, uint32_t flags, const int32_t* guard_dev, int32_t* status_dev,
                      void* stream) {
    if (!valid_dtype(dtype)) return fail(PL_ERR_ARG, "unknown dtype");
    if (n < 3 || n > PL_MAX_ORDER) return fail(PL_ERR_ARG, "layer order out of range");
    if (k < 2 || k > n - 1) return fail(PL_ERR_ARG, "layer index k must be in [2, n-1]");
    if (r1 > pl::binom_u64(n, k) || r0 > r1) return fail(PL_ERR_ARG, "rank range outside the layer");
    if (!a_dev || !cur_dev || (k > 2 && !prev_dev) || !status_dev) return fail(PL_ERR_ARG, "null device pointer");
    if (dtype == PL_I64 && !guard_dev) return fail(PL_ERR_ARG, "int64 layers need the guard flag");
    pl_status s = have_device();
    if (s != PL_OK) return s;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t* tickets = nullptr;
    if (k > 2) {  // a zeroed tile counter for this launch, stream-ordered
        PL_CUDA(cudaMallocAsync((void**)&tickets, sizeof(uint32_t), st));
        PL_CUDA(cudaMemsetAsync(tickets, 0, sizeof(uint32_t), st));
    }
    s = with_ring(dtype, flags & PL_FLAG_FMA, [&](auto r) {
        return launch_layer<decltype(r)>(n, a_dev, k, prev_dev, cur_dev, r0, r1, tickets, guard_dev, status_dev,
                                         st);
    });
    if (tickets) cudaFreeAsync(tickets, st);
    return s;
}

void pl_release_scratch(void) {
    std::vector<IdleBlock> drop;
    {
        ScratchCache& c = scratch_cache();
        std::lock_guard<std::mutex> lock(c.mu);
        drop.swap(c.idle);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (const IdleBlock& ib : drop) {
        cudaSetDevice(ib.b.dev);
        if (ib.ev) {
            cudaEventSynchronize(ib.ev);  // its last use has finished
            cudaEventDestroy(ib.ev);
        }
        cudaFree(ib.b.ptr);
    }
    {
        // the cached tile lists: wait for every device's work that may still read them
        std::lock_guard<std::mutex> lock(g_lists_mu);
        for (auto& kv : lists_cache()) {
            cudaSetDevice(kv.first[0]);
            cudaDeviceSynchronize();
            cudaFree(kv.second.buf);
        }
        lists_cache().clear();
        plc::blk_release_tables();  // every device was synchronised above (or has no tables)
    }
    cudaSetDevice(cur);
    cudaGetLastError();
}

pl_status pl_sz_top(pl_dtype dtype, int32_t n, const void* a_dev, const void* last_dev, void* out_dev,
                    uint32_t flags, const int32_t* guard_dev, int32_t* status_dev, void* stream) {
    if (!valid_dtype(dtype)) return fail(PL_ERR_ARG, "unknown dtype");
    if (n < 3 || n > PL_MAX_ORDER) return fail(PL_ERR_ARG, "order out of range");
    if (!a_dev || !last_dev || !out_dev || !status_dev) return fail(PL_ERR_ARG, "null device pointer");
    pl_status s = have_device();
    if (s != PL_OK) return s;
    return with_ring(dtype, flags & PL_FLAG_FMA, [&](auto r) {
        return launch_top<decltype(r)>(n, a_dev, last_dev, out_dev, guard_dev, status_dev,
                                       static_cast<cudaStream_t>(stream));
    });
}

pl_status pl_sz_guard_i64(int32_t n, const int64_t* a_dev, int32_t* guard_dev, void* stream) {
    if (n < 1 || n > PL_MAX_ORDER || !a_dev || !guard_dev) return fail(PL_ERR_ARG, "bad guard arguments");
    pl_status s = have_device();
    if (s != PL_OK) return s;
    pl::sz_guard_i64_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const long long*>(a_dev), n, guard_dev);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

}  // extern "C"
