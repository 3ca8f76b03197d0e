// Random 4-B gathers over a W-MB window WHILE streaming a large array (the
// relax kernels' mix): does the window stay L2-resident next to evict-first
// streams?  Per thread and step: one 16-B streamed load (evict_first or
// plain) and G random gathers (evict_last), optionally a RED.MIN on the
// gathered address.  Prints G gathers/s and streamed GB/s.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// MARK: 0 none, 1 RED.OR on a bitmap, 2 plain byte store to a flag array
template <int G, bool FIRST, bool RED, bool HINT = false, int MARK = 0>
__global__ void mix(const int *win, uint32_t nwin, const uint4 *stream, uint64_t nstream, int *wr, uint32_t iters,
                    int *out, uint32_t salt, uint32_t *bm, uint8_t *flags) {
    uint64_t pf, pl;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    int acc = 0;
    for (uint32_t i = 0; i < iters; i++) {
        const uint64_t si = ((uint64_t)i * nt + t) % nstream;
        uint4 s;
        if (FIRST)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(s.x), "=r"(s.y), "=r"(s.z), "=r"(s.w) : "l"(stream + si), "l"(pf));
        else
            s = stream[si];
        acc += (int)(s.x ^ s.w);
        uint32_t h = hash32(t * 0x9E3779B9u + i * 0x85ebca6bu + salt);
#pragma unroll
        for (int g = 0; g < G; g++) {
            const uint32_t idx = hash32(h + g) % nwin;
            int v;
            asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(win + idx), "l"(pl));
            acc += v;
            if (RED && (h & (7u << (4 * g))) < (3u << (4 * g))) {   // ~3/8 of the gathers reduce
                if (HINT)
                    asm volatile("red.relaxed.gpu.global.min.L2::cache_hint.s32 [%0], %1, %2;" :: "l"(wr + idx), "r"(v - 1), "l"(pl) : "memory");
                else
                    atomicMin(wr + idx, v - 1);
                if (MARK == 1) atomicOr(bm + (idx >> 5), 1u << (idx & 31));
                if (MARK == 2) flags[idx] = (uint8_t)(i + 1);
            }
        }
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

uint32_t *g_bm;
uint8_t *g_flags;
template <int G, bool FIRST, bool RED, bool HINT = false, int MARK = 0>
void run(const char *tag, int *win, uint32_t nwin, const uint4 *stream, uint64_t nstream, int *out, int grid,
         int block, uint32_t iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; w++) mix<G, FIRST, RED, HINT, MARK><<<grid, block>>>(win, nwin, stream, nstream, win, iters, out, w, g_bm, g_flags);
    cudaEventRecord(e0);
    for (int r = 0; r < 4; r++) mix<G, FIRST, RED, HINT, MARK><<<grid, block>>>(win, nwin, stream, nstream, win, iters, out, 9 + r, g_bm, g_flags);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double steps = 4.0 * grid * block * iters;
    printf("%-22s win %5.0f MB  gathers %6.1f G/s  stream %6.0f GB/s\n", tag, nwin * 4.0 / (1 << 20),
           steps * G / (ms * 1e-3) / 1e9, steps * 16 / (ms * 1e-3) / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxw = (size_t)128 << 20, sbytes = (size_t)2 << 30;
    int *win, *out;
    uint4 *stream;
    cudaMalloc(&win, maxw); cudaMalloc(&out, 64); cudaMalloc(&stream, sbytes);
    cudaMemset(win, 0x11, maxw); cudaMemset(stream, 1, sbytes);
    cudaMalloc(&g_bm, maxw / 32); cudaMalloc(&g_flags, maxw / 4);
    const int grid = sms * 8, block = 256;
    const uint32_t iters = 256;
    const uint64_t ns = sbytes / 16;
    for (int persist = 0; persist < 1; persist++) {
        if (persist) {   // the library's optional persisting set-aside (max) -- no window: hints only
            int mp = 0;
            cudaDeviceGetAttribute(&mp, cudaDevAttrMaxPersistingL2CacheSize, 0);
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mp);
            printf("-- persisting L2 set-aside %d bytes\n", mp);
        }
        for (size_t mb : {24, 50, 64, 100}) {
            const uint32_t nw = (uint32_t)((mb << 20) / 4);
            run<2, true, false>("G2 stream-first", win, nw, stream, ns, out, grid, block, iters);
            run<2, true, true>("G2 first +RED", win, nw, stream, ns, out, grid, block, iters);
            run<2, true, true, true>("G2 first +RED(hint)", win, nw, stream, ns, out, grid, block, iters);
            run<2, true, true, false, 1>("G2 +RED +bitmap OR", win, nw, stream, ns, out, grid, block, iters);
            run<2, true, true, false, 2>("G2 +RED +byte store", win, nw, stream, ns, out, grid, block, iters);
        }
    }
    return 0;
}
