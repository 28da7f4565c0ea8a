// Batch kernels of small orders (n <= 14) and their launch logic: the register
// kernels (n <= 5), the warp / CTA shared-memory kernels (6 <= n <= 14), the
// pair / FP32-exact pack kernels. A translation unit (and so a CUDA module) of
// its own: a module is loaded as a whole on first use, and this one holds
// ~140 of the library's ~180 kernel instantiations, so a large-order call
// (capi.cu's layer kernels) no longer pays for loading it (cold C4 call
// 48 -> 22 ms, round 2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/permlab_b200.h"
#include "capi_internal.h"
#include "sz_batch.cuh"
#include "sz_kernels.cuh"
#include "sz_batch_blk.cuh"

namespace {

pl_status fail(pl_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return plc::fail_msg(s, buf);
}

#define PL_CUDA(expr)                                              \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return plc::cuda_error(_e, #expr);  \
    } while (0)

size_t elem_size(pl_dtype d) { return d == PL_C128 ? 16 : 8; }

uint64_t max_layer(int n) {
    uint64_t m = 0;
    for (int k = 2; k <= n - 1; ++k) m = std::max<uint64_t>(m, pl::binom_u64(n, k));
    return m;
}

int num_sms() { return plc::sm_count(); }

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
    return fail(PL_ERR_ARG, "unknown dtype");
}

// Raise a kernel's MaxDynamicSharedMemorySize only when a launch needs more
// than any earlier one (the attribute is a per-kernel maximum).
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

constexpr int kRegsMaxOrder = 5;  // n = 6 spills in registers; it runs in the shared-memory kernel

// Batch kernel choice for n <= 5: the pipelined kernel for inputs of 64 MiB
// and more (1.6 M c128 5x5: 6.1 vs 5.5 TB/s), the per-warp TMA kernel below
// that (equal at C2's 40 MB, faster for C1's int64) and for misaligned input.
// PL_BATCH_KERNEL=warp|pipe forces one (A/B timing, profiles/batch_ab.py).
bool use_pipe_kernel(size_t in_bytes) {
    static const int force = [] {
        const char* e = std::getenv("PL_BATCH_KERNEL");
        if (e && std::string(e) == "warp") return 0;
        if (e && std::string(e) == "pipe") return 1;
        return -1;
    }();
    return force >= 0 ? force == 1 : in_bytes >= (size_t(64) << 20);
}

// Launch with programmatic stream serialisation (the batch kernels wait for
// the previous grid with griddepcontrol.wait before touching memory, so a
// back-to-back stream of batches overlaps launch and ramp with the previous
// tail). PL_BATCH_PDL=0 launches plainly.
template <class K, class... Args>
cudaError_t launch_pdl(K kern, unsigned grid, unsigned threads, size_t smem, cudaStream_t st, Args... args) {
    static const bool pdl = [] {
        const char* e = std::getenv("PL_BATCH_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <class R, int N>
pl_status launch_regs_n(const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st) {
    using T = typename R::T;
    if (use_pipe_kernel((size_t)count * N * N * sizeof(T)) && (reinterpret_cast<uintptr_t>(a) & 15u) == 0) {
        using Pg = pl::PipeGeom<T, N>;
        auto kern = pl::sz_batch_pipe_kernel<R, N>;
        PL_CUDA(set_smem_once(kern, Pg::kSmem));
        const int64_t nfull = count / 32;
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(nfull, num_sms()));
        PL_CUDA(launch_pdl(kern, (unsigned)blocks, Pg::kThreads, Pg::kSmem, st, static_cast<const T*>(a),
                           static_cast<T*>(out), count, status));
        return PL_OK;
    }
    using Gm = pl::BatchGeom<T, N>;
    auto kern = pl::sz_batch_tma_kernel<R, N>;
    PL_CUDA(set_smem_once(kern, Gm::kSmem));
    // resident CTAs per SM (per instantiation; thread-safe static initialisation)
    static const int per_sm = [kern] {
        int v = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, Gm::kThreads, Gm::kSmem) != cudaSuccess) {
            cudaGetLastError();
            v = 1;
        }
        return std::max(v, 1);
    }();
    const int64_t batches = (count + Gm::kBatch - 1) / Gm::kBatch;
    const int64_t blocks = std::min<int64_t>((batches + Gm::kWarps - 1) / Gm::kWarps, (int64_t)num_sms() * per_sm);
    PL_CUDA(launch_pdl(kern, (unsigned)blocks, Gm::kThreads, Gm::kSmem, st, static_cast<const T*>(a),
                       static_cast<T*>(out), count, status, plc::input_ready_hint() ? 1 : 0));
    return PL_OK;
}

template <class R>
pl_status launch_regs(int n, const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st) {
    switch (n) {
        case 1: return launch_regs_n<R, 1>(a, out, count, status, st);
        case 2: return launch_regs_n<R, 2>(a, out, count, status, st);
        case 3: return launch_regs_n<R, 3>(a, out, count, status, st);
        case 4: return launch_regs_n<R, 4>(a, out, count, status, st);
        case 5: return launch_regs_n<R, 5>(a, out, count, status, st);
    }
    return fail(PL_ERR_ARG, "register kernel order out of range");
}

size_t smem_per_warp(pl_dtype dt, int n) {
    return ((((size_t)n * n + 1) & ~size_t(1)) + 2 * (((size_t)max_layer(n) + 1) & ~size_t(1))) * elem_size(dt);
}

constexpr size_t kSmemCap = 200 * 1024;
constexpr int kSmemMaxOrder = 14;  // predecessor ranks must fit 12 bits (C(14,7) = 3432)

bool smem_fits(pl_dtype dt, int n) { return n <= kSmemMaxOrder && smem_per_warp(dt, n) <= kSmemCap; }

struct Ptab {
    uint16_t* tab = nullptr;
    uint32_t* off = nullptr;
    uint32_t* tab32[3] = {nullptr, nullptr, nullptr};  // byte-offset entries for 8-, 16- and 32-byte elements
    const uint32_t* t32(size_t es) const { return tab32[es == 32 ? 2 : es == 16 ? 1 : 0]; }
    // layers >= 3 with two terms per word (the byte-coefficient FP32 packs): word p * C(n,k) + r of
    // layer k (first word off2[k]) = entry 2p | entry 2p + 1 << 16 of subset r, entries as in `tab`
    uint32_t* tab2 = nullptr;
    uint32_t* off2 = nullptr;
};

// Predecessor table of order n (see sz_batch_smem_kernel), built once per
// (device, n) on the host and cached.
pl_status get_ptab(int n, Ptab* out) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, Ptab> cache;
    int dev = 0;
    PL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, n});
    if (it != cache.end()) {
        *out = it->second;
        return PL_OK;
    }
    std::vector<uint32_t> off(n + 2, 0);
    off[2] = 0;
    off[3] = (uint32_t)pl::binom_u64(n, 2);
    for (int k = 3; k <= n; ++k) off[k + 1] = off[k] + (k < n ? (uint32_t)(k * pl::binom_u64(n, k)) : 0u);
    std::vector<uint16_t> tab(off[n + 1] ? off[n + 1] : 1);
    for (int j2 = 1; j2 < n; ++j2)
        for (int j1 = 0; j1 < j2; ++j1) tab[off[2] + j1 + j2 * (j2 - 1) / 2] = (uint16_t)(j1 | (j2 << 8));
    for (int k = 3; k < n; ++k) {
        const uint64_t ck = pl::binom_u64(n, k);
        uint64_t mask = (1ull << k) - 1;
        for (uint64_t r = 0; r < ck; ++r) {
            int i = 0;
            for (uint64_t m = mask; m; m &= m - 1, ++i) {
                const int s = __builtin_ctzll(m);
                tab[off[k] + i * ck + r] = (uint16_t)(pl_colex_rank(mask & ~(1ull << s)) | ((uint32_t)s << 12));
            }
            const uint64_t c = mask & (~mask + 1), rr = mask + c;  // Gosper: next k-subset in colex order
            mask = (((rr ^ mask) >> 2) / c) | rr;
        }
    }
    Ptab p;
    for (int w = 0; w < 3; ++w) {
        // layers >= 3 as byte offsets: (rank * es) | (column * es) << 16 (es = 8, 16, 32;
        // 32 only where the largest rank * 32 fits 16 bits, n <= 13)
        const uint32_t es = w == 0 ? 8u : w == 1 ? 16u : 32u;
        if (es * (uint32_t)max_layer(n) >= 65536u) continue;
        std::vector<uint32_t> t32(tab.size(), 0);
        for (int k = 3; k < n; ++k)
            for (uint32_t x = off[k]; x < off[k + 1]; ++x)
                t32[x] = (uint32_t)(tab[x] & 0xfffu) * es | ((uint32_t)(tab[x] >> 12) * es) << 16;
        PL_CUDA(cudaMalloc(&p.tab32[w], t32.size() * sizeof(uint32_t)));
        PL_CUDA(cudaMemcpy(p.tab32[w], t32.data(), t32.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    {
        std::vector<uint32_t> off2(n + 2, 0);
        for (int k = 3; k <= n; ++k)
            off2[k + 1] = off2[k] + (k < n ? (uint32_t)(((k + 1) / 2) * pl::binom_u64(n, k)) : 0u);
        std::vector<uint32_t> t2(off2[n + 1] ? off2[n + 1] : 1, 0);
        for (int k = 3; k < n; ++k) {
            const uint64_t ck = pl::binom_u64(n, k);
            for (int i = 0; i < k; ++i)
                for (uint64_t r = 0; r < ck; ++r)
                    t2[off2[k] + (i / 2) * ck + r] |= (uint32_t)tab[off[k] + i * ck + r] << (16 * (i & 1));
        }
        PL_CUDA(cudaMalloc(&p.tab2, t2.size() * sizeof(uint32_t)));
        PL_CUDA(cudaMalloc(&p.off2, off2.size() * sizeof(uint32_t)));
        PL_CUDA(cudaMemcpy(p.tab2, t2.data(), t2.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        PL_CUDA(cudaMemcpy(p.off2, off2.data(), off2.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    PL_CUDA(cudaMalloc(&p.tab, tab.size() * sizeof(uint16_t)));
    PL_CUDA(cudaMalloc(&p.off, off.size() * sizeof(uint32_t)));
    PL_CUDA(cudaMemcpy(p.tab, tab.data(), tab.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    PL_CUDA(cudaMemcpy(p.off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    cache[{dev, n}] = p;
    *out = p;
    return PL_OK;
}


template <class R, int N>
pl_status launch_smem_n(pl_dtype dt, const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st,
                        const Ptab& pt) {
    using T = typename R::T;
    const size_t smem = smem_per_warp(dt, N) + 32;  // one matrix per CTA
    auto kern = pl::sz_batch_smem_kernel<R, N>;
    PL_CUDA(set_smem_once(kern, smem));
    int per_sm = 1;
    PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl::kSmemThreads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t blocks = std::min<int64_t>(count, (int64_t)num_sms() * per_sm);
    if (plc::input_ready_hint()) {  // PL_FLAG_INPUT_READY: see launch_f32_pack_n
        PL_CUDA(launch_pdl(kern, (unsigned)blocks, (unsigned)pl::kSmemThreads, smem, st, static_cast<const T*>(a),
                           static_cast<T*>(out), count, (int)N, (int)max_layer(N), (const uint16_t*)pt.tab,
                           (const uint32_t*)pt.off, pt.t32(sizeof(T)), status, 1));
        return PL_OK;
    }
    kern<<<(unsigned)blocks, pl::kSmemThreads, smem, st>>>(static_cast<const T*>(a), static_cast<T*>(out), count, N,
                                              (int)max_layer(N), pt.tab, pt.off, pt.t32(sizeof(T)), status, 0);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

// Pack kernel for 8-byte rings, 10 <= n <= 14: P matrices per CTA in lockstep.
// P = 2 by default (C3 197 -> 182 us); P = 4 (PL_BATCH_PACK=4, n <= 13, where 16-bit
// byte offsets of 32-byte packs fit) measured slower (233 us: fewer packs per SM);
// PL_BATCH_PACK=1 runs the one-matrix kernel.
int pack_width(int n) {
    static const int force = [] {
        const char* e = std::getenv("PL_BATCH_PACK");
        return e ? atoi(e) : 0;
    }();
    if (force == 1) return 1;
    if (force == 4 && n <= 13) return 4;
    return 2;
}

template <class R, int N, int P>
pl_status launch_pack_n(const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st, const Ptab& pt) {
    using T = typename R::T;
    const int maxc = (int)max_layer(N);
    const size_t smem = (size_t)(N * N + 2 * maxc) * 8 * P + 64;  // pack layout (the single layout fits inside)
    auto kern = pl::sz_batch_smem_pack_kernel<R, N, P>;
    PL_CUDA(set_smem_once(kern, smem));
    int per_sm = 1;
    PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl::pack_threads<N>(), smem));
    per_sm = std::max(per_sm, 1);
    const int64_t packs = (count + P - 1) / P;
    const int64_t blocks = std::min<int64_t>(packs, (int64_t)num_sms() * per_sm);
    kern<<<(unsigned)blocks, pl::pack_threads<N>(), smem, st>>>(static_cast<const T*>(a), static_cast<T*>(out), count, maxc,
                                                          pt.tab, pt.off, pt.t32(8), pt.t32(8 * P), status);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

// int64, 10 <= n <= 14: the FP32-exact four-matrix pack kernel (PL_BATCH_F32=0: the
// double pack kernel).
bool use_f32_pack() {
    static const bool on = [] {
        const char* e = std::getenv("PL_BATCH_F32");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int N, int P>
pl_status launch_f32_pack_n(const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st,
                            const Ptab& pt) {
    const int maxc = (int)max_layer(N);
    // 4P-byte packs (the single layout fits inside) + the byte-packed coefficient words
    const size_t smem = (size_t)(N * N + 2 * maxc) * 4 * P + (size_t)N * N * 4 + 64;
    auto kern = pl::sz_batch_f32_pack_kernel<N, P>;
    PL_CUDA(set_smem_once(kern, smem));
    int per_sm = 1;
    PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl::kF32Threads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t packs = (count + P - 1) / P;
    const int64_t blocks = std::min<int64_t>(packs, (int64_t)num_sms() * per_sm);
    if (plc::input_ready_hint()) {
        // PL_FLAG_INPUT_READY: programmatic dependent launch, loads before the previous grid is done
        // (C3 72 -> 64 us per step in a stream of batches: no launch gap and the next grid's CTAs
        // fill the slots the last, partial round leaves idle)
        PL_CUDA(launch_pdl(kern, (unsigned)blocks, (unsigned)pl::kF32Threads, smem, st,
                           static_cast<const long long*>(a), static_cast<long long*>(out), count, maxc,
                           (const uint16_t*)pt.tab, (const uint32_t*)pt.off, pt.t32(8), pt.t32(4 * P),
                           (const uint32_t*)pt.tab2, (const uint32_t*)pt.off2, status, 1));
        return PL_OK;
    }
    // plain launch otherwise: with the attribute but the wait up front the dependent CTAs only sit in
    // the freed slots (measured 77 against 72 us per step)
    kern<<<(unsigned)blocks, pl::kF32Threads, smem, st>>>(static_cast<const long long*>(a),
                                                         static_cast<long long*>(out), count, maxc, pt.tab,
                                                         pt.off, pt.t32(8), pt.t32(4 * P), pt.tab2, pt.off2, status,
                                                         0);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

// int64, 10 <= n <= 12: the register-blocked FP32-exact pack kernel (sz_batch_blk.cuh);
// opt-in with PL_BATCH_F32_BLK=1 (measured slower than the subset-per-thread pack kernel
// above: C3 171 vs 121 us per call, profiles/r2c/NOTES.md).
bool use_f32_blk() {
    static const bool on = [] {
        const char* e = std::getenv("PL_BATCH_F32_BLK");
        return e && e[0] == '1';
    }();
    return on;
}

template <int N>
pl_status launch_f32_blk_n(const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st,
                           const Ptab& pt) {
    const uint4* wtab = nullptr;
    pl_status s = plc::blk_wtab(&wtab);
    if (s != PL_OK) return s;
    const int maxc = (int)max_layer(N);
    constexpr size_t smem = pl::f32_blk_smem_bytes<N>();
    auto kern = pl::sz_batch_f32_blk_kernel<N>;
    PL_CUDA(set_smem_once(kern, smem));
    int per_sm = 1;
    PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl::kF32BlkThreads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t packs = (count + 3) / 4;
    const int64_t blocks = std::min<int64_t>(packs, (int64_t)num_sms() * per_sm);
    kern<<<(unsigned)blocks, pl::kF32BlkThreads, smem, st>>>(static_cast<const long long*>(a),
                                                            static_cast<long long*>(out), count, maxc, pt.tab,
                                                            pt.off, pt.t32(8), wtab, status);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

// Warp-per-matrix kernel for 8-byte rings, 6 <= n <= 9 (PL_BATCH_SMEM=cta forces the CTA
// kernel). Measured (profiles/c3_ab.py): n = 8 x 50k int64 104 -> 74 us; equal at n = 10;
// slower at n = 12 (C3: 205 -> 293 us), where a matrix's layers take ~16 KB and a warp per
// matrix leaves too few warps per SM, so n >= 10 keeps the CTA-per-matrix kernel.
template <class R, int N>
pl_status launch_warp_n(const void* a, void* out, int64_t count, int32_t* status, cudaStream_t st, const Ptab& pt) {
    using T = typename R::T;
    const size_t smem = (size_t)pl::kWarpKernelWarps * pl::warp_kernel_stride<N>() * sizeof(T);
    auto kern = pl::sz_batch_warp_kernel<R, N>;
    PL_CUDA(set_smem_once(kern, smem));
    int per_sm = 1;
    PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * pl::kWarpKernelWarps, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t blocks = std::min<int64_t>((count + pl::kWarpKernelWarps - 1) / pl::kWarpKernelWarps,
                                             (int64_t)num_sms() * per_sm);
    if (plc::input_ready_hint()) {  // PL_FLAG_INPUT_READY: see launch_f32_pack_n
        PL_CUDA(launch_pdl(kern, (unsigned)blocks, (unsigned)(32 * pl::kWarpKernelWarps), smem, st,
                           static_cast<const T*>(a), static_cast<T*>(out), count, (const uint16_t*)pt.tab,
                           (const uint32_t*)pt.off, pt.t32(sizeof(T)), status, 1));
        return PL_OK;
    }
    kern<<<(unsigned)blocks, 32 * pl::kWarpKernelWarps, smem, st>>>(static_cast<const T*>(a), static_cast<T*>(out),
                                                                   count, pt.tab, pt.off, pt.t32(sizeof(T)), status,
                                                                   0);
    PL_CUDA(cudaGetLastError());
    return PL_OK;
}

bool use_warp_kernel() {
    static const bool warp = [] {
        const char* e = std::getenv("PL_BATCH_SMEM");
        return !(e && std::string(e) == "cta");
    }();
    return warp;
}

// 6 <= n <= 14: the shared-memory kernels, specialised per order.
template <class R>
pl_status launch_smem(pl_dtype dt, int n, const void* a, void* out, int64_t count, int32_t* status,
                      cudaStream_t st) {
    Ptab pt;
    pl_status s = get_ptab(n, &pt);
    if (s != PL_OK) return s;
    if constexpr (sizeof(typename R::T) == 8) {
        if (use_warp_kernel()) {
            switch (n) {
#define PL_WARP_N(NN) \
    case NN:          \
        return launch_warp_n<R, NN>(a, out, count, status, st, pt);
                PL_WARP_N(6) PL_WARP_N(7) PL_WARP_N(8) PL_WARP_N(9)
#undef PL_WARP_N
            }
        }
        if constexpr (std::is_same_v<R, pl::RI64<true>>) {
            if (n >= 10 && n <= 14 && count >= 4 && use_f32_pack()) {
                static const int p8 = [] {
                    const char* e = std::getenv("PL_BATCH_F32_P");  // 8: eight-matrix packs (n <= 13)
                    return e && atoi(e) == 8;
                }();
                if (p8 && n <= 13) {
                    switch (n) {
                        case 10: return launch_f32_pack_n<10, 8>(a, out, count, status, st, pt);
                        case 11: return launch_f32_pack_n<11, 8>(a, out, count, status, st, pt);
                        case 12: return launch_f32_pack_n<12, 8>(a, out, count, status, st, pt);
                        case 13: return launch_f32_pack_n<13, 8>(a, out, count, status, st, pt);
                    }
                }
                if (n <= 12 && use_f32_blk()) {
                    switch (n) {
                        case 10: return launch_f32_blk_n<10>(a, out, count, status, st, pt);
                        case 11: return launch_f32_blk_n<11>(a, out, count, status, st, pt);
                        case 12: return launch_f32_blk_n<12>(a, out, count, status, st, pt);
                    }
                }
                switch (n) {
                    case 10: return launch_f32_pack_n<10, 4>(a, out, count, status, st, pt);
                    case 11: return launch_f32_pack_n<11, 4>(a, out, count, status, st, pt);
                    case 12: return launch_f32_pack_n<12, 4>(a, out, count, status, st, pt);
                    case 13: return launch_f32_pack_n<13, 4>(a, out, count, status, st, pt);
                    case 14: return launch_f32_pack_n<14, 4>(a, out, count, status, st, pt);
                }
            }
        }
        const int P = n >= 10 && n <= 14 ? pack_width(n) : 1;
        if (P > 1 && count >= 2) {
            switch (n * 8 + P) {
#define PL_PACK_N(NN, PP) \
    case NN * 8 + PP:     \
        return launch_pack_n<R, NN, PP>(a, out, count, status, st, pt);
                PL_PACK_N(10, 2) PL_PACK_N(11, 2) PL_PACK_N(12, 2) PL_PACK_N(13, 2) PL_PACK_N(14, 2)
                PL_PACK_N(10, 4) PL_PACK_N(11, 4) PL_PACK_N(12, 4) PL_PACK_N(13, 4)
#undef PL_PACK_N
            }
        }
    }
    switch (n) {
#define PL_SMEM_N(NN) \
    case NN:          \
        return launch_smem_n<R, NN>(dt, a, out, count, status, st, pt);
        PL_SMEM_N(6) PL_SMEM_N(7) PL_SMEM_N(8) PL_SMEM_N(9) PL_SMEM_N(10) PL_SMEM_N(11) PL_SMEM_N(12)
        PL_SMEM_N(13) PL_SMEM_N(14)
#undef PL_SMEM_N
    }
    return fail(PL_ERR_ARG, "shared-memory kernel order out of range");
}


}  // namespace

namespace plc {

bool small_order_batch(pl_dtype dt, int n) { return n <= kRegsMaxOrder || smem_fits(dt, n); }

pl_status launch_small_batch(pl_dtype dt, bool fma, int n, int64_t count, const void* a_dev, void* out_dev,
                             int32_t* status_dev, cudaStream_t st) {
    if (n <= kRegsMaxOrder) {
        return with_ring(dt, fma, [&](auto r) { return launch_regs<decltype(r)>(n, a_dev, out_dev, count, status_dev, st); });
    }
    return with_ring(dt, fma,
                     [&](auto r) { return launch_smem<decltype(r)>(dt, n, a_dev, out_dev, count, status_dev, st); });
}

}  // namespace plc
