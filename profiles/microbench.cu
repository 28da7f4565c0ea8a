// Roofline denominators the driver does not measure:
// FP64 DFMA / DMUL+DADD issue rate, L2-resident read bandwidth, HBM read
// bandwidth and INT64-multiply rate on this B200. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu && ./microbench
// Prints one JSON object.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                    \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmul_dadd_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            x0 = __dmul_rn(x0, a); x1 = __dadd_rn(x1, b); x2 = __dmul_rn(x2, a); x3 = __dadd_rn(x3, b);
            x4 = __dmul_rn(x4, a); x5 = __dadd_rn(x5, b); x6 = __dmul_rn(x6, a); x7 = __dadd_rn(x7, b);
            x0 = __dadd_rn(x0, b); x1 = __dmul_rn(x1, a); x2 = __dadd_rn(x2, b); x3 = __dmul_rn(x3, a);
            x4 = __dadd_rn(x4, b); x5 = __dmul_rn(x5, a); x6 = __dadd_rn(x6, b); x7 = __dmul_rn(x7, a);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void imad64_kernel(long long* out, int iters, long long a, long long b) {
    long long x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

// Grid-stride LDG.128 read of `bytes`, `reps` times; sums to defeat DCE.
__global__ void read_kernel(const double2* __restrict__ p, size_t n, int reps, double* out) {
    double s = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            double2 v = __ldcg(p + i);
            s += v.x + v.y;
        }
    }
    if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ p, double2* __restrict__ q, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) q[i] = p[i];
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double* dout;
    CK(cudaMalloc(&dout, sizeof(double) * sms * 8 * 1024));
    float ms;
    const int blocks = sms * 4, threads = 512, iters = 2000;

    dfma_kernel<<<blocks, threads>>>(dout, 10, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double dfma_per_s = (double)blocks * threads * iters * 64 / (ms * 1e-3);

    dmul_dadd_kernel<<<blocks, threads>>>(dout, 10, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    dmul_dadd_kernel<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double dop_per_s = (double)blocks * threads * iters * 64 / (ms * 1e-3);

    imad64_kernel<<<blocks, threads>>>((long long*)dout, 10, 3, 7);
    CK(cudaEventRecord(e0));
    imad64_kernel<<<blocks, threads>>>((long long*)dout, iters, 3, 7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double imad_per_s = (double)blocks * threads * iters * 32 / (ms * 1e-3);

    // L2-resident reads: 48 MiB, read 40 times
    const size_t l2_bytes = 48ull << 20;
    double2* buf;
    CK(cudaMalloc(&buf, 8ull << 30));
    CK(cudaMemset(buf, 0, 8ull << 30));
    read_kernel<<<sms * 8, 512>>>(buf, l2_bytes / 16, 2, dout);
    CK(cudaEventRecord(e0));
    read_kernel<<<sms * 8, 512>>>(buf, l2_bytes / 16, 40, dout);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double l2_gbs = (double)l2_bytes * 40 / (ms * 1e-3) / 1e9;

    // HBM reads: 4 GiB once
    const size_t hbm_bytes = 4ull << 30;
    read_kernel<<<sms * 8, 512>>>(buf, hbm_bytes / 16, 1, dout);
    CK(cudaEventRecord(e0));
    read_kernel<<<sms * 8, 512>>>(buf, hbm_bytes / 16, 1, dout);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double hbm_read_gbs = (double)hbm_bytes / (ms * 1e-3) / 1e9;

    // HBM copy 2 GiB -> 2 GiB (read + write bytes)
    copy_kernel<<<sms * 8, 512>>>(buf, buf + (2ull << 30) / 16, (2ull << 30) / 16);
    CK(cudaEventRecord(e0));
    copy_kernel<<<sms * 8, 512>>>(buf, buf + (2ull << 30) / 16, (2ull << 30) / 16);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double copy_gbs = 2.0 * (2ull << 30) / (ms * 1e-3) / 1e9;

    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"sms\": %d, \"dfma_per_s\": %.4e, \"fp64_fma_tflops\": %.2f, \"dmul_dadd_per_s\": %.4e, "
           "\"imad64_per_s\": %.4e, \"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"hbm_copy_gbs\": %.1f, "
           "\"clock_khz_attr\": %d}\n",
           sms, dfma_per_s, 2 * dfma_per_s / 1e12, dop_per_s, imad_per_s, l2_gbs, hbm_read_gbs, copy_gbs, clk);
    return 0;
}
