// Which SMs share an L2 partition? Two sweeps with a lagged re-read (see
// l2reuse.cu) run at once on disjoint SM sets A and B over disjoint arrays.
// If A and B sit on different dies, each sweep keeps its die's L2 to itself
// and the lagged re-reads hit more often than when A and B are mixed.
// One CTA per SM (large dynamic smem); set membership by %smid:
//   mode 0: smid < nsm/2 ; mode 1: smid even ; mode 2: (smid / 2) even ; mode 3: (smid/4) even
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned tickets[2];

__global__ void sweep2(const double2* __restrict__ p, const double2* __restrict__ q, size_t nchunks, size_t chunk,
                       size_t lag, int mode, int per_set, double* sink) {
    extern __shared__ unsigned char pad[];
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int nsm = gridDim.x;
    bool inA = mode == 0 ? smid < (unsigned)nsm / 2 : mode == 1 ? (smid & 1) == 0 : mode == 2 ? ((smid >> 1) & 1) == 0 : ((smid >> 2) & 1) == 0;
    __shared__ unsigned t;
    if (threadIdx.x == 0) t = atomicAdd(&tickets[inA ? 0 : 1], 1u);
    __syncthreads();
    const double2* base = inA ? p : q;
    double acc = pad[0];
    for (size_t c = t; c < nchunks + lag; c += per_set) {
        if (c < nchunks) {
            const double2* r = base + c * chunk;
            for (size_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += __ldcg(r + i).x;
        }
        if (c >= lag && c - lag < nchunks) {
            const double2* r = base + (c - lag) * chunk;
            for (size_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += __ldcg(r + i).y;
        }
    }
    if (acc == 1234.5) *sink = acc;
}

int main() {
    const size_t bytes = (size_t)2 << 30, chunk_bytes = 64 << 10;
    const size_t chunk = chunk_bytes / 16, nchunks = bytes / chunk_bytes;
    double2 *p, *q;
    double* sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&q, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(p, 0, bytes);
    cudaMemset(q, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 150 * 1024;
    cudaFuncSetAttribute(sweep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 4; ++mode) {
        for (int mb : {24, 40}) {
            unsigned z[2] = {0, 0};
            cudaMemcpyToSymbol(tickets, z, sizeof(z));
            const size_t lag = ((size_t)mb << 20) / chunk_bytes;
            sweep2<<<sms, 512, smem>>>(p, q, nchunks, chunk, lag, mode, sms / 2, sink);
            cudaDeviceSynchronize();
            printf("mode %d lag %d MB: %s\n", mode, mb, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
