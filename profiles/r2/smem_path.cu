// Microbenchmark: does the L1/shared-memory data path limit the layer
// kernel's operand traffic, and which staging path is cheapest per byte?
//   lds     : LDS.128, lane-contiguous (conflict-free), 16 warps per SM
//   ldg_l2  : LDG.128 coalesced from an L2-resident buffer, L1::no_allocate
//   ldg_l1  : LDG.128 from a 64 KB buffer (L1 hits)
//   mix     : half the warps lds, half ldg_l2 (shared data path?)
//   tma_lds : one warp streams cp.async.bulk (L2 -> smem) into a ring while
//             15 warps LDS from other slots (does TMA fill cost LDS bandwidth?)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_path smem_path.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ double4 lds128(const void* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
    return make_double4(v.x, v.y, 0, 0);
}

__device__ __forceinline__ double2 ldg_na(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ldg_ca(const double2* p) {
    double2 v;
    asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

constexpr int kThreads = 512;
constexpr int kSmemElems = 8192;  // 128 KB of double2

// mode 0: lds all warps; 1: ldg_l2 all warps; 2: ldg_l1; 3: mix; 4: tma + lds
__global__ void __launch_bounds__(kThreads, 1) bench(int mode, const double2* __restrict__ big, size_t big_elems,
                                                     const double2* __restrict__ small, int iters, double* sink) {
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) uint64_t bar[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSmemElems; i += blockDim.x) sm[i] = make_double2(i, -i);
    if (threadIdx.x == 0)
        for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    double ax = 0, ay = 0;
    const bool do_lds = mode == 0 || (mode == 3 && warp < 8) || (mode == 4 && warp > 0);
    const bool do_l2 = mode == 1 || (mode == 3 && warp >= 8);
    if (mode == 4 && warp == 0) {
        // TMA producer: 4 slots of 8 KB at the end of the smem buffer (elements 6144..8191),
        // streaming consecutive 8 KB pieces of `big` (L2 resident), waiting for each landing
        if (lane == 0) {
            size_t off = (size_t)blockIdx.x * 4096;
            for (int it = 0; it < iters; ++it) {
                const int s = it & 3;
                if (it >= 4) {
                    // wait for the copy issued 4 iterations ago into this slot
                    const unsigned par = ((it - 4) >> 2) & 1;
                    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(&bar[s])), "r"(par) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(8192u) : "memory");
                off = (off + 512) % (big_elems - 512);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + 6144 + s * 512)), "l"(big + off), "r"(8192u), "r"(smem_u32(&bar[s])) : "memory");
            }
            for (int it = iters; it < iters + 4; ++it) {
                const int s = it & 3;
                const unsigned par = ((it - 4) >> 2) & 1;
                asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(&bar[s])), "r"(par) : "memory");
            }
        }
    } else if (do_lds) {
        // each warp sweeps lane-contiguous 16-byte words of elements 0..6143, 8 loads in flight
        int base = (warp * 32 + lane) % 6144;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double4 v = lds128(sm + ((base + u * 512) % 6144));
                ax += v.x;
                ay += v.y;
            }
            base = (base + 97 * 32) % 6144;
        }
    } else if (do_l2) {
        size_t idx = ((size_t)blockIdx.x * 16 + warp) * 32 * 64 + lane;
        for (int it = 0; it < iters; ++it) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ldg_na(big + (idx + u * 32) % big_elems);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                ax += v[u].x;
                ay += v[u].y;
            }
            idx = (idx + 256 * 148 * 16) % big_elems;
        }
    } else if (mode == 2) {
        int idx = (warp * 32 + lane) % 4096;
        for (int it = 0; it < iters; ++it) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ldg_ca(small + ((idx + u * 512) & 4095));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                ax += v[u].x;
                ay += v[u].y;
            }
            idx = (idx + 97 * 32) & 4095;
        }
    }
    if (ax + ay == 12345.678) sink[threadIdx.x] = ax;
}

int main() {
    const size_t big_elems = (size_t)48 << 20 >> 4;  // 48 MB: L2 resident
    double2 *big, *small;
    double* sink;
    CK(cudaMalloc(&big, big_elems * 16));
    CK(cudaMalloc(&small, 4096 * 16));
    CK(cudaMalloc(&sink, 4096 * 8));
    CK(cudaMemset(big, 0, big_elems * 16));
    CK(cudaMemset(small, 0, 4096 * 16));
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t smem = kSmemElems * 16;
    CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const char* names[] = {"lds (16 warps)", "ldg_l2 no_allocate (16 warps)", "ldg_l1 hits (16 warps)",
                           "mix: 8 warps lds + 8 warps ldg_l2", "tma 8KB ring (1 warp) + 15 warps lds"};
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) bench<<<sms, kThreads, smem>>>(mode, big, big_elems, small, iters, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        bench<<<sms, kThreads, smem>>>(mode, big, big_elems, small, iters, sink);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        // bytes per SM: warps doing each kind x iters x 8 loads x 512 B
        double lds_warps = mode == 0 ? 16 : mode == 3 ? 8 : mode == 4 ? 15 : 0;
        double ldg_warps = (mode == 1 || mode == 2) ? 16 : mode == 3 ? 8 : 0;
        double lds_b = lds_warps * iters * 8 * 512.0, ldg_b = ldg_warps * iters * 8 * 512.0;
        double tma_b = mode == 4 ? iters * 8192.0 : 0;
        double cyc = ms * 1e-3 * clk * 1e3;  // at the nominal max clock
        printf("%-40s %8.3f ms  lds %6.1f B/clk/SM  ldg %6.1f B/clk/SM  tma %6.1f B/clk/SM  total %6.1f  (%.2f TB/s chip)\n",
               names[mode], ms, lds_b / cyc, ldg_b / cyc, tma_b / cyc, (lds_b + ldg_b + tma_b) / cyc,
               (lds_b + ldg_b + tma_b) * sms / (ms * 1e-3) / 1e12);
    }
    return 0;
}
