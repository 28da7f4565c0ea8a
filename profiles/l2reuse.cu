// L2 reuse-distance probe: all SMs sweep a large array front to back; every
// chunk is read twice, by the lead sweep and again by a lag sweep d bytes
// behind it. DRAM bytes / array bytes = 1 when the lag reads hit L2, 2 when
// they miss. Run under ncu (dram__bytes_read.sum) for several d.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/l2reuse profiles/l2reuse.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void sweep(const double2* __restrict__ p, size_t nchunks, size_t chunk, size_t lag, double* sink) {
    double acc = 0;
    for (size_t c = blockIdx.x; c < nchunks + lag; c += gridDim.x) {
        if (c < nchunks) {
            const double2* q = p + c * chunk;
            for (size_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += __ldcg(q + i).x;
        }
        if (c >= lag && c - lag < nchunks) {
            const double2* q = p + (c - lag) * chunk;
            for (size_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += __ldcg(q + i).y;
        }
    }
    if (acc == 1234.5) *sink = acc;
}

int main(int argc, char** argv) {
    const size_t bytes = (size_t)4 << 30, chunk_bytes = 64 << 10;  // 4 GB array, 64 KB chunks
    const size_t chunk = chunk_bytes / 16, nchunks = bytes / chunk_bytes;
    double2* p;
    double* sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(p, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int mbs[] = {8, 16, 32, 48, 64, 80, 96, 112, 128};
    for (int mb : mbs) {
        const size_t lag = ((size_t)mb << 20) / chunk_bytes;
        sweep<<<sms * 2, 512>>>(p, nchunks, chunk, lag, sink);
        cudaDeviceSynchronize();
        printf("lag %d MB done\n", mb);
    }
    return 0;
}
