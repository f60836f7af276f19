// Microbenchmark: fp64 / fp32 RED throughput into a 16 MB table on one B200, by the number
// of lanes of a warp instruction that share a 32-byte sector or an address.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rate red_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// group: lanes per group that share a sector (mode 1) or an address (mode 2); mode 0: all distinct
template <typename T>
__global__ void k_red(T* g, uint32_t n_mask, int iters, int group, int mode) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        uint32_t base = hash32(tid / (mode ? group : 1) * 7919u + it * 104729u) & n_mask;
        uint32_t idx;
        if (mode == 1) idx = (base & ~3u) | (lane % group & 3);       // same 32B sector (4 doubles)
        else if (mode == 3) idx = (base & ~3u) | (lane & 3);          // group lanes in one sector, 4 addresses
        else idx = base;                                              // same address if mode 2
        atomicAdd(g + idx, (T)1);
    }
}

int main() {
    const uint32_t n = 1u << 21;  // 2M doubles = 16 MB
    double* gd; float* gf;
    cudaMalloc(&gd, n * 8); cudaMalloc(&gf, n * 4);
    cudaMemset(gd, 0, n * 8); cudaMemset(gf, 0, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = 148 * 16, threads = 256, iters = 256;
    const double ops = (double)blocks * threads * iters;
    struct { int group, mode; const char* name; } cases[] = {
        {1, 0, "distinct addresses"}, {2, 1, "2 lanes per sector"}, {4, 1, "4 lanes per sector"},
        {2, 2, "2 lanes per address"}, {8, 2, "8 lanes per address"}, {32, 2, "32 lanes per address"},
        {8, 3, "8 lanes/sector, 4 addr"}, {32, 3, "32 lanes/sector, 4 addr"}};
    for (auto c : cases) {
        for (int f = 0; f < 2; ++f) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (f == 0) k_red<double><<<blocks, threads>>>(gd, n - 1, iters, c.group, c.mode);
                else k_red<float><<<blocks, threads>>>(gf, n - 1, iters, c.group, c.mode);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("%-24s %s: %.3g thread-REDs/s\n", c.name, f ? "f32" : "f64", ops / (ms * 1e-3));
            }
        }
    }
    return 0;
}
