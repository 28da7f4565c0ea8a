// C ABI of the device boson-sampling driver (include/permlab_b200.h,
// "boson sampling" section): outcome probabilities of output patterns of an
// m-mode interferometer, replacing the reference's per-pattern loop
// extract_submatrix -> store_zechin_permanent -> |per|^2 / prod occ!
// (reference proj/src/boson.cpp:207-240, 250-269). Kernels: sz_boson.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/permlab_b200.h"
#include "capi_internal.h"
#include "sz_boson.cuh"

namespace {

constexpr size_t kBosonSmemCap = 200 * 1024;

// The reference's input-mode checks (boson.cpp:63-77), same messages.
pl_status check_modes(int32_t m, int32_t n, const int32_t* modes) {
    if (m < 1) return plc::fail_msg(PL_ERR_ARG, "mode count must be >= 1");
    if (n < 1 || !modes) return plc::fail_msg(PL_ERR_ARG, "at least one input mode is required");
    std::vector<char> seen((size_t)m, 0);
    for (int i = 0; i < n; ++i) {
        if (modes[i] < 0 || modes[i] >= m) return plc::fail_msg(PL_ERR_ARG, "input mode index out of range");
        if (seen[(size_t)modes[i]]) return plc::fail_msg(PL_ERR_ARG, "input modes must be distinct");
        seen[(size_t)modes[i]] = 1;
    }
    return PL_OK;
}

// C(a, l) saturating at UINT64_MAX.
uint64_t binom_sat(uint64_t a, int l) {
    if (l < 0 || (uint64_t)l > a) return 0;
    unsigned __int128 r = 1;
    for (int i = 1; i <= l; ++i) {
        r = r * (a - (uint64_t)l + (uint64_t)i) / (uint64_t)i;
        if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
    }
    return (uint64_t)r;
}

size_t table_bytes(int m, int n) { return (size_t)(n + 1) * (size_t)(m + n) * sizeof(uint64_t); }

template <class R, int N, bool VS>
pl_status launch_fused(const pl::BosonParams& p, bool enumerate, cudaStream_t st) {
    const size_t smem = (enumerate ? table_bytes(p.m, N) : 0) + (VS ? (size_t)p.m * N * sizeof(double2) : 0);
    auto kern = pl::sz_boson_kernel<R, N, VS>;
    {
        // the attribute is a per-kernel maximum: raise it monotonically, under a lock
        static std::mutex mu;
        static size_t have = 0;  // per instantiation
        std::lock_guard<std::mutex> lock(mu);
        if (smem > have) {
            PLC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            have = smem;
        }
    }
    int per_sm = 1;
    PLC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl::kBosonThreads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t want = (p.count + pl::kBosonThreads - 1) / pl::kBosonThreads;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)plc::sm_count() * per_sm));
    if (p.early) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3(pl::kBosonThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        PLC_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
        return PL_OK;
    }
    kern<<<(unsigned)blocks, pl::kBosonThreads, smem, st>>>(p);
    PLC_CUDA(cudaGetLastError());
    return PL_OK;
}

template <class R, int N>
pl_status launch_fused_v(const pl::BosonParams& p, bool enumerate, cudaStream_t st) {
    const size_t tb = enumerate ? table_bytes(p.m, N) : 0;
    if (tb > kBosonSmemCap) return plc::fail_msg(PL_ERR_LIMIT, "mode count too large for the enumeration table");
    if (tb + (size_t)p.m * N * sizeof(double2) <= kBosonSmemCap) return launch_fused<R, N, true>(p, enumerate, st);
    return launch_fused<R, N, false>(p, enumerate, st);
}

template <class R>
pl_status launch_fused_n(int n, const pl::BosonParams& p, bool enumerate, cudaStream_t st) {
    switch (n) {
        case 1: return launch_fused_v<R, 1>(p, enumerate, st);
        case 2: return launch_fused_v<R, 2>(p, enumerate, st);
        case 3: return launch_fused_v<R, 3>(p, enumerate, st);
        case 4: return launch_fused_v<R, 4>(p, enumerate, st);
        case 5: return launch_fused_v<R, 5>(p, enumerate, st);
        case 6: return launch_fused_v<R, 6>(p, enumerate, st);
    }
    return plc::fail_msg(PL_ERR_ARG, "fused boson kernel order out of range");
}

pl_status launch_fused_any(bool fma, int n, const pl::BosonParams& p, bool enumerate, cudaStream_t st) {
    return fma ? launch_fused_n<pl::RC128<true>>(n, p, enumerate, st)
               : launch_fused_n<pl::RC128<false>>(n, p, enumerate, st);
}

// Enqueue probabilities for `count` given row lists (device pointers).
pl_status enqueue_rows(int32_t m, const double2* u_dev, int32_t n, const int32_t* modes, int64_t count,
                       const int32_t* rows_dev, double* probs_dev, bool fma, int32_t* status_dev, cudaStream_t st) {
    if (count == 0) return PL_OK;
    if (n <= pl::kBosonMaxFused) {
        pl::BosonParams p = {};
        p.u = u_dev;
        p.m = m;
        for (int j = 0; j < n; ++j) p.in[j] = modes[j];
        p.count = count;
        p.rows = rows_dev;
        p.probs = probs_dev;
        p.status = status_dev;
        return launch_fused_any(fma, n, p, false, st);
    }
    // larger orders: materialise the submatrices for the batched permanent kernels
    double2* sub = nullptr;
    double2* per = nullptr;
    int32_t* bad = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&sub, (size_t)count * n * n * sizeof(double2), st));
    PLC_CUDA(cudaMallocAsync((void**)&per, (size_t)count * sizeof(double2), st));
    PLC_CUDA(cudaMallocAsync((void**)&bad, (size_t)count * sizeof(int32_t), st));
    PLC_CUDA(cudaMemsetAsync(bad, 0, (size_t)count * sizeof(int32_t), st));
    pl::BosonGather g = {};
    g.u = u_dev;
    g.m = m;
    g.n = n;
    for (int j = 0; j < n; ++j) g.in[j] = modes[j];
    g.rows = rows_dev;
    g.count = count;
    g.sub = sub;
    g.bad = bad;
    g.status = status_dev;
    const int blocks = plc::sm_count() * 8;
    pl::sz_boson_gather_kernel<<<blocks, 256, 0, st>>>(g);
    PLC_CUDA(cudaGetLastError());
    pl_status s = plc::enqueue_batch(PL_C128, n, count, sub, per, fma, status_dev, st);
    if (s == PL_OK) {
        if (fma) pl::sz_boson_norm_kernel<true><<<blocks, 256, 0, st>>>(per, rows_dev, n, count, bad, probs_dev);
        else pl::sz_boson_norm_kernel<false><<<blocks, 256, 0, st>>>(per, rows_dev, n, count, bad, probs_dev);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) s = plc::cuda_error(e, "sz_boson_norm_kernel");
    }
    cudaFreeAsync(sub, st);
    cudaFreeAsync(per, st);
    cudaFreeAsync(bad, st);
    return s;
}

// Synchronous driver around an enqueue: device copies of host buffers, a
// status word, the wait, and status -> error mapping.
template <class Enq>
pl_status run_sync(int32_t m, const void* u, size_t rows_bytes, const int32_t* rows, int64_t count, double* probs,
                   uint32_t flags, int32_t* status_user, cudaStream_t st, Enq&& enq) {
    const bool dev = flags & PL_FLAG_DEVICE_PTRS;
    if (flags & PL_FLAG_ASYNC) {
        if (!dev) return plc::fail_msg(PL_ERR_ARG, "PL_FLAG_ASYNC requires PL_FLAG_DEVICE_PTRS");
        return enq(static_cast<const double2*>(u), rows, probs, status_user);
    }
    const double2* u_dev = static_cast<const double2*>(u);
    const int32_t* rows_dev = rows;
    double* probs_dev = probs;
    int32_t* status_dev = nullptr;
    PLC_CUDA(cudaMallocAsync((void**)&status_dev, sizeof(int32_t), st));
    PLC_CUDA(cudaMemsetAsync(status_dev, 0, sizeof(int32_t), st));
    if (!dev) {
        double2* ud = nullptr;
        PLC_CUDA(cudaMallocAsync((void**)&ud, (size_t)m * m * sizeof(double2), st));
        PLC_CUDA(cudaMemcpyAsync(ud, u, (size_t)m * m * sizeof(double2), cudaMemcpyHostToDevice, st));
        u_dev = ud;
        if (rows_bytes) {
            int32_t* rd = nullptr;
            PLC_CUDA(cudaMallocAsync((void**)&rd, rows_bytes, st));
            PLC_CUDA(cudaMemcpyAsync(rd, rows, rows_bytes, cudaMemcpyHostToDevice, st));
            rows_dev = rd;
        }
        PLC_CUDA(cudaMallocAsync((void**)&probs_dev, std::max<size_t>((size_t)count * sizeof(double), 16), st));
    }
    pl_status s = enq(u_dev, rows_dev, probs_dev, status_dev);
    int32_t status_host = 0;
    if (s == PL_OK && !dev && count > 0) {
        const cudaError_t e = cudaMemcpyAsync(probs, probs_dev, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(probs)");
    }
    if (s == PL_OK) {
        const cudaError_t e = cudaMemcpyAsync(&status_host, status_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = plc::cuda_error(e, "cudaMemcpyAsync(status)");
    }
    if (!dev) {
        cudaFreeAsync(const_cast<double2*>(u_dev), st);
        if (rows_bytes) cudaFreeAsync(const_cast<int32_t*>(rows_dev), st);
        cudaFreeAsync(probs_dev, st);
    }
    cudaFreeAsync(status_dev, st);
    const cudaError_t e3 = cudaStreamSynchronize(st);
    if (s == PL_OK && e3 != cudaSuccess) s = plc::cuda_error(e3, "cudaStreamSynchronize");
    if (s == PL_OK && (status_host & PL_STATUS_BIT_ROWS)) {
        s = plc::fail_msg(PL_ERR_ARG, "output rows must be nondecreasing mode indices in [0, m)");
    }
    if (s == PL_OK && (status_host & PL_STATUS_BIT_OVERFLOW)) {
        s = plc::fail_msg(PL_ERR_OVERFLOW, "int64 overflow");  // unreachable for the complex ring
    }
    return s;
}

}  // namespace

extern "C" {

uint64_t pl_boson_pattern_count(int32_t m, int32_t n) {
    if (m < 1 || n < 0) return 0;
    const uint64_t c = binom_sat((uint64_t)m + (uint64_t)n - 1, n);
    return c == UINT64_MAX ? 0 : c;
}

pl_status pl_boson_unrank_pattern(int32_t m, int32_t n, uint64_t index, int32_t* rows) {
    if (m < 1 || n < 1 || !rows) return plc::fail_msg(PL_ERR_ARG, "bad arguments to pl_boson_unrank_pattern");
    const uint64_t total = pl_boson_pattern_count(m, n);
    if (total == 0 || index >= total) return plc::fail_msg(PL_ERR_ARG, "pattern index out of range");
    // the device kernel's search (sz_boson.cuh boson_unrank), on the host
    int prev = 0;
    for (int i = 0; i < n; ++i) {
        const int len = n - 1 - i;
        const uint64_t top = binom_sat((uint64_t)(m - prev + len), len + 1);
        int lo = prev, hi = m - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (top - binom_sat((uint64_t)(m - mid + len), len + 1) <= index) lo = mid;
            else hi = mid - 1;
        }
        index -= top - binom_sat((uint64_t)(m - lo + len), len + 1);
        rows[i] = lo;
        prev = lo;
    }
    return PL_OK;
}

pl_status pl_boson_probabilities(int32_t m, const void* u, int32_t n, const int32_t* input_modes, int64_t count,
                                 const int32_t* out_rows, double* probs, uint32_t flags, const pl_limits* limits,
                                 void* stream, int32_t* status_dev) {
    pl_status s = check_modes(m, n, input_modes);
    if (s != PL_OK) return s;
    s = plc::check_order_limits(n, limits);
    if (s != PL_OK) return s;
    if (count < 0) return plc::fail_msg(PL_ERR_ARG, "negative pattern count");
    if (!u || (count > 0 && (!out_rows || !probs))) return plc::fail_msg(PL_ERR_ARG, "null unitary, rows or output pointer");
    if ((flags & PL_FLAG_ASYNC) && !status_dev) return plc::fail_msg(PL_ERR_ARG, "PL_FLAG_ASYNC requires a device status word");
    s = plc::device_ready();
    if (s != PL_OK) return s;
    const bool fma = flags & PL_FLAG_FMA;
    std::vector<int32_t> modes(input_modes, input_modes + n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return run_sync(m, u, (size_t)count * n * sizeof(int32_t), out_rows, count, probs, flags, status_dev, st,
                    [&](const double2* ud, const int32_t* rd, double* pd, int32_t* sd) {
                        return enqueue_rows(m, ud, n, modes.data(), count, rd, pd, fma, sd, st);
                    });
}

pl_status pl_boson_distribution(int32_t m, const void* u, int32_t n, const int32_t* input_modes, uint64_t first,
                                int64_t count, double* probs, uint32_t flags, void* stream) {
    pl_status s = check_modes(m, n, input_modes);
    if (s != PL_OK) return s;
    if (n > pl::kBosonMaxFused) {
        return plc::fail_msg(PL_ERR_LIMIT, "full distributions are enumerated for at most 6 photons");
    }
    const uint64_t total = pl_boson_pattern_count(m, n);
    if (total == 0 || total > (1ull << 62)) return plc::fail_msg(PL_ERR_LIMIT, "outcome count exceeds the 64-bit index range");
    if (count < 0 || first > total || (uint64_t)count > total - first) {
        return plc::fail_msg(PL_ERR_ARG, "pattern range outside the distribution");
    }
    if (!u || (count > 0 && !probs)) return plc::fail_msg(PL_ERR_ARG, "null unitary or output pointer");
    if (table_bytes(m, n) > kBosonSmemCap) return plc::fail_msg(PL_ERR_LIMIT, "mode count too large for the enumeration table");
    s = plc::device_ready();
    if (s != PL_OK) return s;
    const bool fma = flags & PL_FLAG_FMA;
    std::vector<int32_t> modes(input_modes, input_modes + n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return run_sync(m, u, 0, nullptr, count, probs, flags, nullptr, st,
                    [&](const double2* ud, const int32_t*, double* pd, int32_t* sd) -> pl_status {
                        if (count == 0) return PL_OK;
                        pl::BosonParams p = {};
                        p.u = ud;
                        p.m = m;
                        for (int j = 0; j < n; ++j) p.in[j] = modes[j];
                        p.first = first;
                        p.count = count;
                        p.rows = nullptr;
                        p.probs = pd;
                        p.status = sd;
                        p.early = ((flags & PL_FLAG_INPUT_READY) && (flags & PL_FLAG_DEVICE_PTRS)) ? 1 : 0;
                        return launch_fused_any(fma, n, p, true, st);
                    });
}

}  // extern "C"
