// Cold-call cost probe: what does a first large allocation cost?
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void touch(char* p, size_t n) { for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 4096; i < n; i += (size_t)gridDim.x * blockDim.x * 4096) p[i] = 1; }
int main() {
    double t = now(); cudaFree(0); printf("context %.1f ms\n", now() - t);
    cudaStream_t s; cudaStreamCreate(&s);
    for (size_t gb : {1, 4, 19}) {
        size_t n = gb << 30; void* p;
        t = now(); cudaMalloc(&p, n); cudaDeviceSynchronize(); double a = now() - t;
        t = now(); touch<<<1184, 256>>>((char*)p, n); cudaDeviceSynchronize(); double b = now() - t;
        t = now(); cudaFree(p); double c = now() - t;
        t = now(); cudaMallocAsync(&p, n, s); cudaStreamSynchronize(s); double d = now() - t;
        t = now(); touch<<<1184, 256, 0, s>>>((char*)p, n); cudaStreamSynchronize(s); double e = now() - t;
        t = now(); cudaFreeAsync(p, s); cudaStreamSynchronize(s); double f = now() - t;
        t = now(); cudaMallocAsync(&p, n, s); cudaStreamSynchronize(s); double g = now() - t;
        cudaFreeAsync(p, s); cudaStreamSynchronize(s);
        printf("%2zu GB: cudaMalloc %.1f ms, first touch %.1f, cudaFree %.1f | mallocAsync %.1f, touch %.1f, freeAsync+sync %.1f, mallocAsync again %.1f\n", gb, a, b, c, d, e, f, g);
    }
    return 0;
}
