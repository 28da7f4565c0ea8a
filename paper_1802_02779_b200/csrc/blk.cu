// Host side of the register-blocked layer engine (sz_blk.cuh): tables per
// (device, order, register columns), scratch sizing and the launch chain of one
// large matrix. Replaces the arithmetic of the reference's SzEval::eval /
// run_top (proj/src/permanent.cpp:151-199) for the float rings.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/permlab_b200.h"
#include "capi_internal.h"
#include "sz_blk.cuh"

namespace {

struct BlkTables {
    uint32_t* tb = nullptr;      // [(NW + 1)][2^H] first row of tile (F, j)
    uint32_t* flist = nullptr;   // valid F of every super-layer, increasing
    std::vector<uint64_t> fl_off;  // fl_off[j]: first flist entry of super-layer j (size NW + 2)
    std::vector<uint64_t> rows;    // rows[j]: rows of super-layer j
    int H = 0, NW = 0;
};

std::mutex g_mu;
std::map<std::vector<int>, BlkTables>& tables_cache() {
    static auto* m = new std::map<std::vector<int>, BlkTables>;
    return *m;
}
std::map<int, uint4*>& wtab_cache() {
    static auto* m = new std::map<int, uint4*>;
    return *m;
}

// rows and tiles of super-layer j in closed form: sum over f = popc(F)
void layer_shape(int H, int j, uint64_t* tiles, uint64_t* rows) {
    uint64_t t = 0, r = 0;
    for (int f = 0; f <= H; ++f) {
        const int m = j - f;
        if (m < 0 || m > pl::kBlkDW) continue;
        const uint64_t c = pl::binom_u64(H, f);
        t += c;
        r += c * pl::blk_rows9(m);
    }
    *tiles = t;
    *rows = r;
}

pl_status get_wtab(const uint4** out) {
    int dev = 0;
    PLC_CUDA(cudaGetDevice(&dev));
    auto& cache = wtab_cache();
    auto it = cache.find(dev);
    if (it == cache.end()) {
        // entry t (ascending window column w_t) of the m-subset V of colex rank q:
        // rank9(V \ {w_t}) | w_t << 7, 12 bits each; entries 0-4 in the low 64 bits,
        // 5-8 in the high 64 bits
        std::vector<uint64_t> tab(2 * 512, 0);
        auto rank9 = [](uint32_t mask) {
            uint32_t r = 0;
            int i = 1;
            for (uint32_t mm = mask; mm; mm &= mm - 1, ++i) r += (uint32_t)pl::binom_u64(__builtin_ctz(mm), i);
            return r;
        };
        for (uint32_t mask = 0; mask < 512; ++mask) {
            const int m = __builtin_popcount(mask);
            uint64_t* e = &tab[2 * (size_t)(pl::blk_moff9(m) + rank9(mask))];
            int t = 0;
            for (uint32_t mm = mask; mm; mm &= mm - 1, ++t) {
                const uint32_t w = (uint32_t)__builtin_ctz(mm);
                const uint64_t fld = rank9(mask & ~(1u << w)) | w << 7;
                if (t < 5)
                    e[0] |= fld << (12 * t);
                else
                    e[1] |= fld << (12 * (t - 5));
            }
        }
        uint4* d = nullptr;
        PLC_CUDA(cudaMalloc(&d, tab.size() * sizeof(uint64_t)));
        PLC_CUDA(cudaMemcpy(d, tab.data(), tab.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        it = cache.emplace(dev, d).first;
    }
    *out = it->second;
    return PL_OK;
}

pl_status get_tables(int n, int LC, const BlkTables** out) {
    int dev = 0;
    PLC_CUDA(cudaGetDevice(&dev));
    auto& cache = tables_cache();
    const std::vector<int> key = {dev, n, LC};
    auto it = cache.find(key);
    if (it == cache.end()) {
        BlkTables t;
        t.NW = n - LC;
        t.H = t.NW - pl::kBlkDW;
        t.fl_off.assign(t.NW + 2, 0);
        t.rows.assign(t.NW + 1, 0);
        for (int j = 0; j <= t.NW; ++j) {
            uint64_t tiles = 0;
            layer_shape(t.H, j, &tiles, &t.rows[j]);
            t.fl_off[j + 1] = t.fl_off[j] + tiles;
            if (t.rows[j] >= pl::kBlkInvalid) return plc::fail_msg(PL_ERR_LIMIT, "block engine: super-layer too large");
        }
        uint64_t* off_dev = nullptr;
        PLC_CUDA(cudaMalloc(&t.tb, ((size_t)(t.NW + 1) << t.H) * sizeof(uint32_t)));
        PLC_CUDA(cudaMalloc(&t.flist, std::max<uint64_t>(t.fl_off[t.NW + 1], 1) * sizeof(uint32_t)));
        PLC_CUDA(cudaMalloc(&off_dev, t.fl_off.size() * sizeof(uint64_t)));
        PLC_CUDA(cudaMemcpy(off_dev, t.fl_off.data(), t.fl_off.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        cudaStream_t st;
        PLC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        pl::blk_tables_kernel<<<t.NW + 1, 1024, 0, st>>>(t.H, t.tb, t.flist, off_dev);
        const cudaError_t e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        cudaFree(off_dev);
        PLC_CUDA(e);
        PLC_CUDA(cudaGetLastError());
        it = cache.emplace(key, std::move(t)).first;
    }
    *out = &it->second;
    return PL_OK;
}

template <class R>
pl_status run_ring(int n, const void* a_dev, void* out_dev, void* scratch, int32_t* status, cudaStream_t st) {
    using T = typename R::T;
    constexpr int LC = pl::blk_reg_cols((int)sizeof(T));
    const BlkTables* tabs = nullptr;
    const uint4* wtab = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        pl_status s = get_tables(n, LC, &tabs);
        if (s != PL_OK) return s;
        s = get_wtab(&wtab);
        if (s != PL_OK) return s;
    }
    uint64_t max_rows = 0;
    for (uint64_t r : tabs->rows) max_rows = std::max(max_rows, r);
    constexpr size_t kHead = 256;
    uint32_t* tickets = static_cast<uint32_t*>(scratch);
    T* buf[2] = {reinterpret_cast<T*>(static_cast<char*>(scratch) + kHead),
                 reinterpret_cast<T*>(static_cast<char*>(scratch) + kHead + max_rows * pl::kBlkRowBytes)};
    PLC_CUDA(cudaMemsetAsync(scratch, 0, kHead, st));
    auto kern = pl::sz_blk_kernel<R, LC>;
    constexpr size_t smem = (size_t)pl::kBlkWarps * pl::kBlkRowBytes +
                            (size_t)pl::kBlkWarps * pl::kBlkSlots * pl::BlkRing<T, LC>::kSlotBytes;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    PLC_CUDA(attr_err);
    static const bool pdl = [] {
        const char* e = std::getenv("PL_WS_PDL");
        return !(e && e[0] == '0');
    }();
    static const int per_sm = [] {
        const char* e = std::getenv("PL_BLK_CTAS");  // tuning: CTAs per SM in the grid
        return e ? std::max(1, atoi(e)) : 4;
    }();
    static const uint32_t hints = [] {
        const char* e = std::getenv("PL_BLK_HINTS");  // timing probes (wrong results), see sz_blk.cuh
        return e ? (uint32_t)std::strtoul(e, nullptr, 0) : 0u;
    }();
    const size_t nF = (size_t)1 << tabs->H;
    for (int j = 0; j <= tabs->NW; ++j) {
        const uint32_t ntiles = (uint32_t)(tabs->fl_off[j + 1] - tabs->fl_off[j]);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)std::max<uint32_t>(1, std::min<uint32_t>(ntiles, (uint32_t)(plc::sm_count() * per_sm))));
        cfg.blockDim = dim3(32 * pl::kBlkWarps);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        const T* prev = buf[(j + 1) & 1];
        T* cur = buf[j & 1];
        PLC_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(a_dev), n, j, prev, cur, static_cast<T*>(out_dev),
                                    tickets + j, static_cast<const uint32_t*>(tabs->flist + tabs->fl_off[j]), ntiles,
                                    static_cast<const uint32_t*>(tabs->tb + (size_t)j * nF),
                                    static_cast<const uint32_t*>(j ? tabs->tb + (size_t)(j - 1) * nF : nullptr), wtab,
                                    status, hints));
    }
    return PL_OK;
}

}  // namespace

namespace plc {

// Off by default (measured slower than the per-layer kernels):
// PL_BLK=1 turns the engine on; PL_BLK_MIN_N moves the smallest order it takes.
bool blk_supported(pl_dtype dt, int n) {
    static const bool on = [] {
        const char* e = std::getenv("PL_BLK");
        return e && e[0] == '1';
    }();
    static const int min_n = [] {
        const char* e = std::getenv("PL_BLK_MIN_N");
        return e ? atoi(e) : 15;
    }();
    if (!on || (dt != PL_F64 && dt != PL_C128)) return false;
    const int LC = pl::blk_reg_cols(dt == PL_C128 ? 16 : 8);
    return n >= std::max(min_n, LC + pl::kBlkDW + 1) && n <= PL_MAX_ORDER;
}

size_t blk_scratch_bytes(pl_dtype dt, int n) {
    const int LC = pl::blk_reg_cols(dt == PL_C128 ? 16 : 8);
    const int NW = n - LC, H = NW - pl::kBlkDW;
    uint64_t max_rows = 0;
    for (int j = 0; j <= NW; ++j) {
        uint64_t tiles = 0, rows = 0;
        layer_shape(H, j, &tiles, &rows);
        max_rows = std::max(max_rows, rows);
    }
    return 256 + 2 * (size_t)max_rows * pl::kBlkRowBytes;
}

pl_status run_blocks(pl_dtype dt, bool fma, int n, const void* a_dev, void* out_dev, void* scratch, int32_t* status,
                     cudaStream_t st) {
    if (dt == PL_F64)
        return fma ? run_ring<pl::RF64<true>>(n, a_dev, out_dev, scratch, status, st)
                   : run_ring<pl::RF64<false>>(n, a_dev, out_dev, scratch, status, st);
    if (dt == PL_C128)
        return fma ? run_ring<pl::RC128<true>>(n, a_dev, out_dev, scratch, status, st)
                   : run_ring<pl::RC128<false>>(n, a_dev, out_dev, scratch, status, st);
    return fail_msg(PL_ERR_ARG, "block engine: unsupported dtype");
}

pl_status blk_wtab(const uint4** out) {
    std::lock_guard<std::mutex> lock(g_mu);
    return get_wtab(out);
}

void blk_release_tables() {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto& kv : tables_cache()) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaSetDevice(kv.first[0]);
        cudaDeviceSynchronize();  // work that may still read them
        cudaFree(kv.second.tb);
        cudaFree(kv.second.flist);
        cudaSetDevice(dev);
    }
    tables_cache().clear();
}

}  // namespace plc
