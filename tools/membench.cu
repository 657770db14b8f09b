// tools/membench.cu -- HBM access-granularity probe for the LU data layout.
// Each warp reads `run` consecutive 256 B rows (32 lanes x 8 B) starting at a
// pseudo-random row of a large buffer; reports achieved GB/s for several run
// lengths, plus a streaming baseline.  Build: nvcc -O3 -arch=sm_100a membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void gather_runs(const double* __restrict__ buf, size_t rows, int run, int iters,
                            double* sink) {
    const int lane = threadIdx.x & 31;
    const size_t w = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        const size_t r0 = mix(w * 1315423911ull + it) % (rows - run);
        const double* p = buf + r0 * 32 + lane;
        double v[8];
        for (int z = 0; z < run; z += 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = z + q < run ? p[size_t(z + q) * 32] : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += v[q];
        }
    }
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void stream_read(const double4* __restrict__ buf, size_t n, double* sink) {
    double acc = 0.0;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const double4 v = buf[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.678) sink[0] = acc;
}

int main() {
    const size_t bytes = size_t(16) << 30;  // 16 GiB
    double* buf;
    double* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 0, bytes);
    const size_t rows = bytes / 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_read<<<148 * 8, 256>>>(reinterpret_cast<const double4*>(buf), bytes / 32, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("stream read 16 GiB: %.0f GB/s\n", bytes / ms / 1e6);
    }
    const int runs[] = {1, 2, 4, 8, 16, 32, 64};
    for (int run : runs) {
        for (int warps_per_sm : {16, 32, 64}) {
            const int threads = 256, blocks = 148 * warps_per_sm / 8;
            const int iters = int((size_t(4) << 30) / (size_t(blocks) * 8 * run * 256)) + 1;
            gather_runs<<<blocks, threads>>>(buf, rows, run, 1, sink);
            cudaEventRecord(a);
            gather_runs<<<blocks, threads>>>(buf, rows, run, iters, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            const double moved = double(blocks) * 8 * iters * run * 256;
            printf("run %2d rows (%5d B) warps/SM %2d: %.0f GB/s\n", run, run * 256, warps_per_sm,
                   moved / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
