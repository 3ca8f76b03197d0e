// Random 4-B gathers with different load flavours (plain / nc / L2 cache-hint
// evict_last / nc+no_allocate+evict_first) at several working-set sizes.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int MODE>
__device__ __forceinline__ int ld(const int *p, uint64_t pol) {
    int v;
    if (MODE == 0) v = *(volatile const int *)p;
    else if (MODE == 1) v = __ldg(p);
    else if (MODE == 2) asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    else if (MODE == 3) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    else if (MODE == 4) asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
    else asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <int MODE>
__global__ void gather(const int *a, uint32_t n, uint32_t iters, int *out, uint32_t salt) {
    uint64_t pol;
    if (MODE == 3) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    int acc = 0;
    for (uint32_t i = 0; i < iters; i += 4) {
        uint32_t h0 = hash32(t * 0x9E3779B9u + i * 0x85ebca6bu + salt);
        uint32_t h1 = hash32(h0 + 1), h2 = hash32(h0 + 2), h3 = hash32(h0 + 3);
        acc += ld<MODE>(a + h0 % n, pol) + ld<MODE>(a + h1 % n, pol) + ld<MODE>(a + h2 % n, pol) + ld<MODE>(a + h3 % n, pol);
    }
    if (acc == 0x7fffffff) out[0] = acc;
}
template <int MODE>
double run(const int *a, uint32_t n, int *out, int grid, int block, uint32_t iters) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; w++) gather<MODE><<<grid, block>>>(a, n, iters, out, w);
    cudaEventRecord(e0);
    for (int r = 0; r < 4; r++) gather<MODE><<<grid, block>>>(a, n, iters, out, 100 + r);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return 4.0 * grid * block * iters / (ms * 1e-3) / 1e9;
}
int main(int argc, char **argv) {
    if (argc > 1) {
        size_t g = (size_t)atoi(argv[1]);
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    }
    size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit: %zu\n", cur);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t maxS = (size_t)400 << 20;
    int *a, *out; cudaMalloc(&a, maxS); cudaMalloc(&out, 64); cudaMemset(a, 1, maxS);
    const int grid = sms * 8, block = 256; const uint32_t iters = 256;
    printf("%6s %9s %9s %9s %9s %9s %9s   (G gathers/s)\n", "MB", "volatile", "ldg", "hint_last", "nc_first", "plain", "cg");
    for (size_t mb : {32, 64, 100, 200, 400}) {
        uint32_t n = (uint32_t)((mb << 20) / 4);
        printf("%6zu %9.1f %9.1f %9.1f %9.1f %9.1f %9.1f\n", mb, run<0>(a, n, out, grid, block, iters), run<1>(a, n, out, grid, block, iters),
               run<2>(a, n, out, grid, block, iters), run<3>(a, n, out, grid, block, iters), run<4>(a, n, out, grid, block, iters),
               run<5>(a, n, out, grid, block, iters));
    }
    return 0;
}
