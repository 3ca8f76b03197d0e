// Microbenchmark: random 4-byte gathers over a working set of S bytes.
// Reports gathers/s and effective bytes per gather (from timing only) to find
// the effective L2 capacity for randomly gathered data on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__global__ void gather(const int *a, uint32_t n, uint32_t iters, int *out, uint32_t salt) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    int acc = 0;
    for (uint32_t i = 0; i < iters; i += 4) {
        uint32_t h0 = hash32(t * 0x9E3779B9u + i * 0x85ebca6bu + salt);
        uint32_t h1 = hash32(h0 + 1), h2 = hash32(h0 + 2), h3 = hash32(h0 + 3);
        acc += a[h0 % n] + a[h1 % n] + a[h2 % n] + a[h3 % n];
    }
    if (acc == 0x7fffffff) out[0] = acc;
}
__global__ void red_min(int *a, uint32_t n, uint32_t iters, uint32_t salt) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t i = 0; i < iters; i++) {
        uint32_t h = hash32(t * 0x9E3779B9u + i * 0x85ebca6bu + salt);
        atomicMin(a + (h % n), (int)(h >> 8));
    }
}
int main() {
    int dev = 0; cudaSetDevice(dev);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t maxS = (size_t)400 << 20;
    int *a, *out; cudaMalloc(&a, maxS); cudaMalloc(&out, 64); cudaMemset(a, 1, maxS);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = sms * 8, block = 256; const uint32_t iters = 256;
    double total = (double)grid * block * iters;
    printf("%10s %14s %14s %14s\n", "MB", "Ggather/s", "B/gather@6.5TB", "GredMin/s");
    for (size_t mb : {8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 200, 400}) {
        uint32_t n = (uint32_t)((mb << 20) / 4);
        for (int w = 0; w < 3; w++) gather<<<grid, block>>>(a, n, iters, out, w);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; r++) gather<<<grid, block>>>(a, n, iters, out, 100 + r);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double gps = 5 * total / (ms * 1e-3);
        for (int w = 0; w < 2; w++) red_min<<<grid, block>>>(a, n, iters / 4, w);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; r++) red_min<<<grid, block>>>(a, n, iters / 4, 100 + r);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        double rps = 5 * total / 4 / (ms2 * 1e-3);
        printf("%10zu %14.1f %14.1f %14.1f\n", mb, gps / 1e9, 6.5e12 / gps, rps / 1e9);
    }
    return 0;
}
