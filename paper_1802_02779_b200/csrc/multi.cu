// Multi-GPU Store-zechin inside one process (C ABI, include/permlab_b200.h).
//
// The reference is single-threaded (reference proj/src/permanent.cpp:310-316);
// this is the engine's addition for C/C++ callers of the drop-in boundary:
// pl_limits.num_gpus = g >= 1 runs a large-order matrix (n >= 15) as ONE
// layer DP sharded over devices 0..g-1, with single-process NCCL
// communicators (ncclCommInitAll) and one stream per device:
//
//   * top-column blocks (g = 2^t, n - t >= 3): device d computes the
//     k-subsets whose top-t-column pattern is P_d (bit i of d <-> column
//     n - t + i), one contiguous colex range of C(n - t, k - |P_d|) ranks;
//     after each layer it sends its block to the devices d | 2^i and receives
//     the blocks of d & ~2^i (ncclSend / ncclRecv in one group): about
//     (t / 2) / 2^t of a layer per device instead of an all-gather's
//     (2^t - 1) / 2^t. Layer n - 1 is sent to device 0 for the top level.
//   * equal slices + in-place all-gather (any other g, and g = 1): every
//     layer is cut into g padded slices of ceil(C(n,k) / g) ranks and
//     replicated by ncclAllGather after it is computed.
//
// Every output is computed once by the same layer kernel on a rank range
// (plc::layer), so results are bitwise those of the single-device path. The
// same plans drive the torch.distributed version (sharded.py); the plan
// functions are exported (pl_shard_*) so the CPU suite checks both agree.
// Batches of smaller orders are split by matrix across the devices, with no
// collective. NCCL is loaded with dlopen on first use (libnccl.so.2).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/permlab_b200.h"
#include "capi_internal.h"
#include "ring.cuh"

namespace {

// ---------------------------------------------------------------- plans

int top_columns(int world) {
    if (world < 1 || (world & (world - 1)) != 0) return -1;
    int t = 0;
    while ((1 << t) < world) ++t;
    return t;
}

bool block_plan(int n, int world) {
    const int t = top_columns(world);
    return t >= 1 && n - t >= 3;
}

void top_block(int n, int k, int world, int g, uint64_t* r0, uint64_t* r1) {
    const int t = top_columns(world);
    int cols[32], nc = 0;
    for (int i = 0; i < t; ++i)
        if ((g >> i) & 1) cols[nc++] = n - t + i;
    const int m = k - nc;
    if (m < 0 || m > n - t) {
        *r0 = *r1 = 0;
        return;
    }
    uint64_t base = 0;
    for (int l = 0; l < nc; ++l) base += pl::binom_u64(cols[l], m + l + 1);
    *r0 = base;
    *r1 = base + pl::binom_u64(n - t, m);
}

uint64_t slice_len(int n, int k, int world) {
    const uint64_t total = pl::binom_u64(n, k);
    return (total + world - 1) / world;
}

void slice_range(int n, int k, int world, int g, uint64_t* r0, uint64_t* r1) {
    const uint64_t total = pl::binom_u64(n, k), per = slice_len(n, k, world);
    *r0 = std::min<uint64_t>((uint64_t)g * per, total);
    *r1 = std::min<uint64_t>((uint64_t)(g + 1) * per, total);
}

struct Xop {
    int recv;  // 0 send, 1 receive
    int peer;
    uint64_t r0, r1;
};

// Point-to-point exchange after layer k under the block plan (k < n - 1).
int block_exchange(int n, int k, int world, int g, Xop* ops) {
    const int t = top_columns(world);
    int c = 0;
    for (int i = 0; i < t; ++i) {
        const int partner = g ^ (1 << i);
        uint64_t r0, r1;
        if ((g >> i) & 1) {  // receive block P \ {n - t + i}
            top_block(n, k, world, partner, &r0, &r1);
            if (r1 > r0) ops[c++] = Xop{1, partner, r0, r1};
        } else {  // send own block to P u {n - t + i}
            top_block(n, k, world, g, &r0, &r1);
            if (r1 > r0) ops[c++] = Xop{0, partner, r0, r1};
        }
    }
    return c;
}

// Top-column terms of device g's block of layer k (block plan): its range,
// the columns c in P_g ascending and the bases of the blocks P_g \ {c} of
// layer k - 1 (same offsets, received from their owners); init_first when the
// block has no other term (lower part empty: S = P_g).
struct TopTerms {
    uint64_t base = 0, len = 0;
    int nsrc = 0;
    int cols[8];
    uint64_t sbase[8];
    bool init_first = false;
};

TopTerms block_top_terms(int n, int k, int world, int g) {
    TopTerms tt;
    const int t = top_columns(world);
    uint64_t r0, r1;
    top_block(n, k, world, g, &r0, &r1);
    tt.base = r0;
    tt.len = r1 - r0;
    int bits = 0;
    for (int i = 0; i < t; ++i) {
        if (!((g >> i) & 1)) continue;
        ++bits;
        uint64_t s0, s1;
        top_block(n, k - 1, world, g & ~(1 << i), &s0, &s1);
        tt.cols[tt.nsrc] = n - t + i;
        tt.sbase[tt.nsrc] = s0;
        ++tt.nsrc;
    }
    tt.init_first = k == bits;
    return tt;
}

// PL_SHARD_OVERLAP=0: the block plan exchanges each layer before the next
// one starts (no partial layers).
bool shard_overlap() {
    static const bool on = [] {
        const char* e = std::getenv("PL_SHARD_OVERLAP");
        return !(e && e[0] == '0');
    }();
    return on;
}

// ---------------------------------------------------------------- NCCL (dlopen)

struct Nccl {
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const Nccl& nccl() {
    static Nccl api = [] {
        Nccl a;
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            a.error = std::string("NCCL is not available (dlopen libnccl.so.2: ") + dlerror() + ")";
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
        };
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.AllGather, "ncclAllGather");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    return api;
}

pl_status nccl_fail(ncclResult_t r, const char* what) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
    return plc::fail_msg(PL_ERR_NCCL, buf);
}

#define PL_NCCL(expr)                                             \
    do {                                                          \
        ncclResult_t _r = (expr);                                 \
        if (_r != ncclSuccess) return nccl_fail(_r, #expr);       \
    } while (0)

// Communicators and streams of one device set, created once per process.
struct DeviceGroup {
    std::vector<int> devs;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    std::vector<cudaStream_t> xstreams;  // exchange streams (block plan, overlapped)
    std::vector<cudaEvent_t> done, xdone;  // layer final on streams[g] / exchange landed on xstreams[g]
    std::mutex run;  // one sharded DP at a time per device set (NCCL ops must be issued in the same order)
};

pl_status device_group(const std::vector<int>& devs, DeviceGroup** out) {
    static std::mutex mu;
    static std::map<std::vector<int>, DeviceGroup*> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(devs);
    if (it != cache.end()) {
        *out = it->second;
        return PL_OK;
    }
    const Nccl& api = nccl();
    if (!api.error.empty()) return plc::fail_msg(PL_ERR_NCCL, api.error.c_str());
    auto* g = new DeviceGroup;
    g->devs = devs;
    g->comms.resize(devs.size());
    g->streams.resize(devs.size());
    g->xstreams.resize(devs.size());
    g->done.resize(devs.size());
    g->xdone.resize(devs.size());
    int cur = 0;
    PLC_CUDA(cudaGetDevice(&cur));
    for (size_t i = 0; i < devs.size(); ++i) {
        PLC_CUDA(cudaSetDevice(devs[i]));
        PLC_CUDA(cudaStreamCreateWithFlags(&g->streams[i], cudaStreamNonBlocking));
        PLC_CUDA(cudaStreamCreateWithFlags(&g->xstreams[i], cudaStreamNonBlocking));
        PLC_CUDA(cudaEventCreateWithFlags(&g->done[i], cudaEventDisableTiming));
        PLC_CUDA(cudaEventCreateWithFlags(&g->xdone[i], cudaEventDisableTiming));
    }
    PLC_CUDA(cudaSetDevice(cur));
    PL_NCCL(api.CommInitAll(g->comms.data(), (int)devs.size(), devs.data()));
    PLC_CUDA(cudaSetDevice(cur));
    cache[devs] = g;
    *out = g;
    return PL_OK;
}

pl_status check_devices(int num_gpus, const int32_t* devices, std::vector<int>* out) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        count = 0;
    }
    if (count == 0) return plc::fail_msg(PL_ERR_NODEVICE, "no CUDA device available (the engine has no CPU fallback)");
    if (num_gpus < 1) return plc::fail_msg(PL_ERR_ARG, "num_gpus must be >= 1");
    out->clear();
    for (int i = 0; i < num_gpus; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= count) {
            char buf[128];
            std::snprintf(buf, sizeof buf, "device %d requested, %d visible", d, count);
            return plc::fail_msg(PL_ERR_ARG, buf);
        }
        if (std::find(out->begin(), out->end(), d) != out->end()) {
            return plc::fail_msg(PL_ERR_ARG, "duplicate device in the device list");
        }
        out->push_back(d);
    }
    return PL_OK;
}

size_t esize(pl_dtype d) { return d == PL_C128 ? 16 : 8; }

// Head of every device's scratch block: tile tickets (64 words), guard,
// status word, top-level output.
constexpr size_t kTickets = 0, kGuard = 256, kStatus = 260, kOut = 384, kHead = 512;

// One large matrix, layer DP sharded over the group. `a` is host or device
// memory (UVA copies), `out` likewise (one element).
pl_status sharded_dp(DeviceGroup& G, pl_dtype dt, int n, const void* a, void* out, bool fma) {
    const Nccl& api = nccl();
    const int world = (int)G.devs.size();
    const size_t es = esize(dt);
    const bool blocks = block_plan(n, world);
    uint64_t cap = 0;  // entries per layer buffer
    for (int k = 2; k <= n - 1; ++k)
        cap = std::max<uint64_t>(cap, blocks ? pl::binom_u64(n, k) : slice_len(n, k, world) * world);
    const size_t stride = (cap * es + 64 + 255) & ~size_t(255);
    const size_t mat_bytes = (size_t)n * n * es;
    const size_t mat_off = kHead + 2 * stride;
    std::vector<plc::ScratchBlock> blk(world);
    int cur_dev = 0;
    PLC_CUDA(cudaGetDevice(&cur_dev));
    pl_status s = PL_OK;
    auto dev_ptr = [&](int g, size_t off) { return static_cast<char*>(blk[g].ptr) + off; };
    for (int g = 0; g < world && s == PL_OK; ++g) {
        PLC_CUDA(cudaSetDevice(G.devs[g]));
        s = plc::scratch_get(mat_off + ((mat_bytes + 255) & ~size_t(255)), G.streams[g], &blk[g]);
        if (s != PL_OK) break;
        PLC_CUDA(cudaMemsetAsync(blk[g].ptr, 0, kHead, G.streams[g]));
        PLC_CUDA(cudaMemcpyAsync(dev_ptr(g, mat_off), a, mat_bytes, cudaMemcpyDefault, G.streams[g]));
        if (dt == PL_I64) {
            s = plc::guard_i64(n, dev_ptr(g, mat_off), reinterpret_cast<int32_t*>(dev_ptr(g, kGuard)), G.streams[g]);
        }
    }
    char* bufs[64][2];
    for (int g = 0; g < world && s == PL_OK; ++g) {
        bufs[g][0] = dev_ptr(g, kHead);
        bufs[g][1] = dev_ptr(g, kHead + stride);
    }
    int pi = 0;  // layer k lands in bufs[.][pi ^ 1] ... prev = bufs[.][pi]
    const bool overlap = blocks && shard_overlap() && n - 1 >= 3;
    const int tcols = top_columns(world);
    for (int k = 2; overlap && k <= n - 1 && s == PL_OK; ++k) {
        // Overlapped block plan. Layer k of device g: the partial layer (every
        // term but the top columns', from g's own block of layer k - 1) runs on
        // streams[g] while the exchange of layer k - 1 runs on xstreams[g];
        // then the top-column terms from the received blocks. The top columns
        // are the highest, so their terms come last in the reference's
        // ascending order: partial + top terms is the same rounding sequence.
        const int ci = k == 2 ? 0 : (pi ^ 1);
        if (k >= 3) {
            // exchange of layer k - 1 (final on streams[g], event done[g])
            PL_NCCL(api.GroupStart());
            for (int g = 0; g < world; ++g) {
                PLC_CUDA(cudaSetDevice(G.devs[g]));
                PLC_CUDA(cudaStreamWaitEvent(G.xstreams[g], G.done[g], 0));
                Xop ops[32];
                const int no = block_exchange(n, k - 1, world, g, ops);
                for (int i = 0; i < no; ++i) {
                    char* p = bufs[g][pi] + ops[i].r0 * es;
                    const size_t bytes = (ops[i].r1 - ops[i].r0) * es;
                    if (ops[i].recv) PL_NCCL(api.Recv(p, bytes, ncclUint8, ops[i].peer, G.comms[g], G.xstreams[g]));
                    else PL_NCCL(api.Send(p, bytes, ncclUint8, ops[i].peer, G.comms[g], G.xstreams[g]));
                }
            }
            PL_NCCL(api.GroupEnd());
            for (int g = 0; g < world; ++g) {
                PLC_CUDA(cudaSetDevice(G.devs[g]));
                PLC_CUDA(cudaEventRecord(G.xdone[g], G.xstreams[g]));
            }
        }
        for (int g = 0; g < world && s == PL_OK; ++g) {
            uint64_t r0, r1;
            top_block(n, k, world, g, &r0, &r1);
            PLC_CUDA(cudaSetDevice(G.devs[g]));
            if (r1 > r0) {
                s = plc::layer(dt, fma, n, dev_ptr(g, mat_off), k, k == 2 ? nullptr : bufs[g][pi], bufs[g][ci], r0, r1,
                               reinterpret_cast<uint32_t*>(dev_ptr(g, kTickets)) + k,
                               reinterpret_cast<const int32_t*>(dev_ptr(g, kGuard)),
                               reinterpret_cast<int32_t*>(dev_ptr(g, kStatus)), G.streams[g], k == 2 ? 0 : tcols);
            }
            if (s != PL_OK) break;
            if (k >= 3) {
                PLC_CUDA(cudaStreamWaitEvent(G.streams[g], G.xdone[g], 0));
                const TopTerms tt = block_top_terms(n, k, world, g);
                if (tt.len) {
                    s = plc::top_terms(dt, fma, n, dev_ptr(g, mat_off), k, bufs[g][pi], bufs[g][ci], tt.base, tt.len,
                                       tt.nsrc, tt.cols, tt.sbase, tt.init_first,
                                       reinterpret_cast<int32_t*>(dev_ptr(g, kStatus)), G.streams[g]);
                }
            }
            PLC_CUDA(cudaEventRecord(G.done[g], G.streams[g]));
        }
        if (s != PL_OK) break;
        if (k == n - 1) {  // layer n - 1: every owner sends its entries to device 0
            PL_NCCL(api.GroupStart());
            for (int g = 0; g < world; ++g) {
                for (int h = 1; h < world; ++h) {
                    uint64_t r0, r1;
                    top_block(n, k, world, h, &r0, &r1);
                    if (r1 <= r0) continue;
                    if (g == 0) PL_NCCL(api.Recv(bufs[0][ci] + r0 * es, (r1 - r0) * es, ncclUint8, h, G.comms[0], G.streams[0]));
                    if (g == h) PL_NCCL(api.Send(bufs[h][ci] + r0 * es, (r1 - r0) * es, ncclUint8, 0, G.comms[h], G.streams[h]));
                }
            }
            PL_NCCL(api.GroupEnd());
        }
        pi = ci;
    }
    for (int k = 2; !overlap && k <= n - 1 && s == PL_OK; ++k) {
        const int ci = k == 2 ? 0 : (pi ^ 1);
        for (int g = 0; g < world && s == PL_OK; ++g) {
            uint64_t r0, r1;
            if (blocks) top_block(n, k, world, g, &r0, &r1);
            else slice_range(n, k, world, g, &r0, &r1);
            if (r1 <= r0) continue;
            PLC_CUDA(cudaSetDevice(G.devs[g]));
            s = plc::layer(dt, fma, n, dev_ptr(g, mat_off), k, k == 2 ? nullptr : bufs[g][pi], bufs[g][ci], r0, r1,
                           reinterpret_cast<uint32_t*>(dev_ptr(g, kTickets)) + k,
                           reinterpret_cast<const int32_t*>(dev_ptr(g, kGuard)),
                           reinterpret_cast<int32_t*>(dev_ptr(g, kStatus)), G.streams[g]);
        }
        if (s != PL_OK) break;
        // exchange: every device's copy of layer k gets what its next layer reads
        PL_NCCL(api.GroupStart());
        for (int g = 0; g < world; ++g) {
            if (!blocks) {
                const size_t bytes = slice_len(n, k, world) * es;
                PL_NCCL(api.AllGather(bufs[g][ci] + (size_t)g * bytes, bufs[g][ci], bytes, ncclUint8, G.comms[g],
                                      G.streams[g]));
            } else if (k < n - 1) {
                Xop ops[32];
                const int no = block_exchange(n, k, world, g, ops);
                for (int i = 0; i < no; ++i) {
                    char* p = bufs[g][ci] + ops[i].r0 * es;
                    const size_t bytes = (ops[i].r1 - ops[i].r0) * es;
                    if (ops[i].recv) PL_NCCL(api.Recv(p, bytes, ncclUint8, ops[i].peer, G.comms[g], G.streams[g]));
                    else PL_NCCL(api.Send(p, bytes, ncclUint8, ops[i].peer, G.comms[g], G.streams[g]));
                }
            } else {  // layer n - 1: every owner sends its entries to device 0
                for (int h = 1; h < world; ++h) {
                    uint64_t r0, r1;
                    top_block(n, k, world, h, &r0, &r1);
                    if (r1 <= r0) continue;
                    if (g == 0) PL_NCCL(api.Recv(bufs[0][ci] + r0 * es, (r1 - r0) * es, ncclUint8, h, G.comms[0], G.streams[0]));
                    if (g == h) PL_NCCL(api.Send(bufs[h][ci] + r0 * es, (r1 - r0) * es, ncclUint8, 0, G.comms[h], G.streams[h]));
                }
            }
        }
        PL_NCCL(api.GroupEnd());
        pi = ci;
    }
    int32_t status = 0;
    if (s == PL_OK) {
        PLC_CUDA(cudaSetDevice(G.devs[0]));
        s = plc::top(dt, fma, n, dev_ptr(0, mat_off), bufs[0][pi], dev_ptr(0, kOut),
                     reinterpret_cast<const int32_t*>(dev_ptr(0, kGuard)), reinterpret_cast<int32_t*>(dev_ptr(0, kStatus)),
                     G.streams[0]);
        if (s == PL_OK) {
            const cudaError_t e = cudaMemcpyAsync(out, dev_ptr(0, kOut), es, cudaMemcpyDefault, G.streams[0]);
            if (e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(out)");
        }
    }
    for (int g = 0; g < world; ++g) {
        if (!blk[g].ptr) continue;
        cudaSetDevice(G.devs[g]);
        int32_t st = 0;
        const cudaError_t e = cudaMemcpyAsync(&st, dev_ptr(g, kStatus), sizeof st, cudaMemcpyDeviceToHost, G.streams[g]);
        const pl_status sp = plc::scratch_put(blk[g], G.streams[g]);
        const cudaError_t e2 = cudaStreamSynchronize(G.streams[g]);
        if (s == PL_OK && e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(status)");
        if (s == PL_OK && e2 != cudaSuccess) s = plc::cuda_error(e2, "cudaStreamSynchronize");
        if (s == PL_OK) s = sp;
        status |= st;
    }
    cudaSetDevice(cur_dev);
    if (s == PL_OK && (status & PL_STATUS_BIT_OVERFLOW)) {
        s = plc::fail_msg(PL_ERR_OVERFLOW, "int64 overflow: an intermediate sub-permanent does not fit the exact int64 ring");
    }
    return s;
}

// A batch of smaller orders split by matrix across the group (no collective).
pl_status split_batch(DeviceGroup& G, pl_dtype dt, int n, int64_t count, const void* a, void* out, uint32_t flags,
                      const pl_limits* lim) {
    const int world = (int)G.devs.size();
    const size_t es = esize(dt), mat_bytes = (size_t)n * n * es;
    const int64_t per = (count + world - 1) / world;
    int cur_dev = 0;
    PLC_CUDA(cudaGetDevice(&cur_dev));
    (void)lim;
    // every device's share is enqueued on its own stream before any wait, so
    // the devices run concurrently
    pl_status s = PL_OK;
    std::vector<void*> dev_in(world, nullptr), dev_out(world, nullptr);
    std::vector<int32_t*> dev_status(world, nullptr);
    const bool dev_ptrs = flags & PL_FLAG_DEVICE_PTRS;
    for (int g = 0; g < world && s == PL_OK; ++g) {
        const int64_t b0 = std::min<int64_t>(count, g * per), b1 = std::min<int64_t>(count, b0 + per);
        if (b1 <= b0) continue;
        PLC_CUDA(cudaSetDevice(G.devs[g]));
        cudaStream_t st = G.streams[g];
        PLC_CUDA(cudaMallocAsync(&dev_in[g], (size_t)(b1 - b0) * mat_bytes, st));
        PLC_CUDA(cudaMallocAsync(&dev_out[g], (size_t)(b1 - b0) * es, st));
        PLC_CUDA(cudaMallocAsync((void**)&dev_status[g], sizeof(int32_t), st));
        PLC_CUDA(cudaMemsetAsync(dev_status[g], 0, sizeof(int32_t), st));
        PLC_CUDA(cudaMemcpyAsync(dev_in[g], static_cast<const char*>(a) + (size_t)b0 * mat_bytes,
                                 (size_t)(b1 - b0) * mat_bytes, cudaMemcpyDefault, st));
        s = plc::enqueue_batch(dt, n, b1 - b0, dev_in[g], dev_out[g], flags & PL_FLAG_FMA, dev_status[g], st);
        if (s != PL_OK) break;
        PLC_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + (size_t)b0 * es, dev_out[g], (size_t)(b1 - b0) * es,
                                 dev_ptrs ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, st));
    }
    int32_t status = 0;
    for (int g = 0; g < world; ++g) {
        if (!dev_in[g]) continue;
        cudaSetDevice(G.devs[g]);
        int32_t sv = 0;
        cudaMemcpyAsync(&sv, dev_status[g], sizeof sv, cudaMemcpyDeviceToHost, G.streams[g]);
        cudaFreeAsync(dev_in[g], G.streams[g]);
        cudaFreeAsync(dev_out[g], G.streams[g]);
        cudaFreeAsync(dev_status[g], G.streams[g]);
        const cudaError_t e = cudaStreamSynchronize(G.streams[g]);
        if (s == PL_OK && e != cudaSuccess) s = plc::cuda_error(e, "cudaStreamSynchronize");
        status |= sv;
    }
    cudaSetDevice(cur_dev);
    if (s == PL_OK && (status & PL_STATUS_BIT_OVERFLOW)) {
        s = plc::fail_msg(PL_ERR_OVERFLOW, "int64 overflow: an intermediate sub-permanent does not fit the exact int64 ring");
    }
    return s;
}

}  // namespace

namespace plc {

// Entry of pl_sz_permanent / pl_sz_permanent_batch when limits->num_gpus >= 1.
pl_status run_multi(pl_dtype dt, int n, int64_t count, const void* a, void* out, uint32_t flags,
                    const pl_limits* lim, const int32_t* devices, cudaStream_t caller) {
    if (flags & PL_FLAG_ASYNC) return fail_msg(PL_ERR_ARG, "the multi-GPU path is synchronous (no PL_FLAG_ASYNC)");
    std::vector<int> devs;
    pl_status s = check_devices(lim->num_gpus, devices, &devs);
    if (s != PL_OK) return s;
    // inputs the caller produced on its stream must be complete
    PLC_CUDA(cudaStreamSynchronize(caller));
    DeviceGroup* G = nullptr;
    s = device_group(devs, &G);
    if (s != PL_OK) return s;
    std::lock_guard<std::mutex> lock(G->run);
    if (count == 0) return PL_OK;
    if (n < 15) return split_batch(*G, dt, n, count, a, out, flags, lim);
    const size_t es = esize(dt), mat_bytes = (size_t)n * n * es;
    for (int64_t b = 0; b < count && s == PL_OK; ++b) {
        s = sharded_dp(*G, dt, n, static_cast<const char*>(a) + (size_t)b * mat_bytes, static_cast<char*>(out) + b * es,
                       flags & PL_FLAG_FMA);
    }
    return s;
}

}  // namespace plc

extern "C" {

int32_t pl_shard_plan(int32_t n, int32_t world) {
    if (n < 3 || world < 1) return -1;
    return block_plan(n, world) ? PL_SHARD_BLOCKS : PL_SHARD_ALLGATHER;
}

pl_status pl_shard_range(int32_t n, int32_t world, int32_t rank, int32_t k, uint64_t* r0, uint64_t* r1) {
    if (n < 3 || n > PL_MAX_ORDER || world < 1 || world > 64 || rank < 0 || rank >= world || k < 2 || k > n - 1 ||
        !r0 || !r1) {
        return plc::fail_msg(PL_ERR_ARG, "bad arguments to pl_shard_range");
    }
    if (block_plan(n, world)) top_block(n, k, world, rank, r0, r1);
    else slice_range(n, k, world, rank, r0, r1);
    return PL_OK;
}

int32_t pl_shard_exchange(int32_t n, int32_t world, int32_t rank, int32_t k, uint64_t* ops, int32_t max_ops) {
    if (n < 3 || n > PL_MAX_ORDER || world < 1 || world > 64 || rank < 0 || rank >= world || k < 2 || k > n - 1) return -1;
    Xop x[64];
    int c = 0;
    if (!block_plan(n, world)) {
        return 0;  // the all-gather plan replicates the whole layer
    }
    if (k < n - 1) {
        c = block_exchange(n, k, world, rank, x);
    } else {
        for (int h = 1; h < world; ++h) {
            uint64_t r0, r1;
            top_block(n, k, world, h, &r0, &r1);
            if (r1 <= r0) continue;
            if (rank == 0) x[c++] = Xop{1, h, r0, r1};
            if (rank == h) x[c++] = Xop{0, 0, r0, r1};
        }
    }
    if (ops) {
        for (int i = 0; i < c && i < max_ops; ++i) {
            ops[4 * i] = (uint64_t)x[i].recv;
            ops[4 * i + 1] = (uint64_t)x[i].peer;
            ops[4 * i + 2] = x[i].r0;
            ops[4 * i + 3] = x[i].r1;
        }
    }
    return c;
}

pl_status pl_shard_block_partial(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev,
                                 void* cur_dev, int32_t world, int32_t rank, uint32_t flags, const int32_t* guard_dev,
                                 int32_t* status_dev, void* stream) {
    if (!block_plan(n, world) || rank < 0 || rank >= world) return plc::fail_msg(PL_ERR_ARG, "not a block-plan rank");
    if (k < 3 || k > n - 1) return plc::fail_msg(PL_ERR_ARG, "layer index k must be in [3, n-1]");
    if (!a_dev || !prev_dev || !cur_dev || !status_dev) return plc::fail_msg(PL_ERR_ARG, "null device pointer");
    if (dtype == PL_I64 && !guard_dev) return plc::fail_msg(PL_ERR_ARG, "int64 layers need the guard flag");
    pl_status s = plc::device_ready();
    if (s != PL_OK) return s;
    uint64_t r0, r1;
    top_block(n, k, world, rank, &r0, &r1);
    if (r1 <= r0) return PL_OK;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t* tickets = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&tickets, sizeof(uint32_t), st));
    PLC_CUDA(cudaMemsetAsync(tickets, 0, sizeof(uint32_t), st));
    s = plc::layer(dtype, flags & PL_FLAG_FMA, n, a_dev, k, prev_dev, cur_dev, r0, r1, tickets, guard_dev, status_dev,
                   st, top_columns(world));
    cudaFreeAsync(tickets, st);
    return s;
}

pl_status pl_shard_block_top_terms(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev,
                                   void* cur_dev, int32_t world, int32_t rank, uint32_t flags, int32_t* status_dev,
                                   void* stream) {
    if (!block_plan(n, world) || rank < 0 || rank >= world) return plc::fail_msg(PL_ERR_ARG, "not a block-plan rank");
    if (k < 3 || k > n - 1) return plc::fail_msg(PL_ERR_ARG, "layer index k must be in [3, n-1]");
    if (!a_dev || !prev_dev || !cur_dev || !status_dev) return plc::fail_msg(PL_ERR_ARG, "null device pointer");
    pl_status s = plc::device_ready();
    if (s != PL_OK) return s;
    const TopTerms tt = block_top_terms(n, k, world, rank);
    return plc::top_terms(dtype, flags & PL_FLAG_FMA, n, a_dev, k, prev_dev, cur_dev, tt.base, tt.len, tt.nsrc,
                          tt.cols, tt.sbase, tt.init_first, status_dev, static_cast<cudaStream_t>(stream));
}

pl_status pl_sz_permanent_multi(pl_dtype dtype, int32_t n, int64_t count, const void* a, void* out, uint32_t flags,
                                const pl_limits* limits, int32_t num_gpus, const int32_t* devices) {
    pl_limits lim;
    pl_limits_default(&lim);
    if (limits) lim = *limits;
    lim.num_gpus = num_gpus;
    if (dtype != PL_I64 && dtype != PL_F64 && dtype != PL_C128) return plc::fail_msg(PL_ERR_ARG, "unknown dtype");
    if (count < 0) return plc::fail_msg(PL_ERR_ARG, "negative batch count");
    if (count > 0 && (!a || !out)) return plc::fail_msg(PL_ERR_ARG, "null matrix or output pointer");
    pl_status s = plc::check_order_limits(n, &lim);
    if (s != PL_OK) return s;
    s = plc::check_budget_limits(dtype, n, &lim);
    if (s != PL_OK) return s;
    return plc::run_multi(dtype, n, count, a, out, flags, &lim, devices, nullptr);
}

}  // extern "C"
