// L2 residency probe: every SM re-reads a working set of W bytes R times
// (grid-stride, 16-byte loads); effective bandwidth vs W shows the usable L2
// capacity for data shared by all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/l2probe profiles/l2probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void reread(const double2* __restrict__ p, size_t n, int reps, double* sink) {
    double acc = 0;
    for (int r = 0; r < reps; ++r) {
        // rotate the start so each pass touches lines in a different order per CTA
        const size_t off = (size_t)r * 977 * 32;
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            const double2 v = __ldg(p + (i + off) % n);
            acc += v.x + v.y;
        }
    }
    if (acc == 1234.5) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxb = (size_t)1 << 30;
    double2* p;
    double* sink;
    cudaMalloc(&p, maxb);
    cudaMalloc(&sink, 8);
    cudaMemset(p, 0, maxb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int mbs[] = {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 160, 256, 1024};
    for (int mb : mbs) {
        const size_t bytes = (size_t)mb << 20, n = bytes / 16;
        const int reps = 20;
        reread<<<sms * 4, 512>>>(p, n, 2, sink);
        cudaEventRecord(e0);
        reread<<<sms * 4, 512>>>(p, n, reps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("W %5d MB: %8.1f GB/s\n", mb, (double)bytes * reps / ms / 1e6);
    }
    return 0;
}
