// The L2 ceiling of the relax step with the issue overhead taken out: per
// thread and iteration, U independent random 4-B gathers over a W-MB window
// (evict_last) next to a streamed 8 B per gather (evict_first), and for a
// fraction of them a RED.MIN to a random window address (value independent
// of the gathers: fire-and-forget) plus optionally a RED.OR on an n-bit
// bitmap.  All addresses are computed up front, so up to U gathers per
// thread are in flight.  Prints gathers/s and REDs/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2probe4 tools/l2probe4.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// RED_PER8: REDs per 8 gathers (0..8); MARK: also RED.OR the bitmap bit; DEP:
// the RED value depends on the gathered value (the relax step's data flow)
template <int U, int RED_PER8, bool MARK, bool DEP>
__global__ void __launch_bounds__(256) mix(int *win, uint32_t nwin, const uint2 *stream, uint64_t nstream,
                                           uint32_t iters, int *out, uint32_t salt, uint32_t *bm) {
    uint64_t pf, pl;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    int acc = 0;
    for (uint32_t i = 0; i < iters; i++) {
        uint32_t idx[U];
        int v[U];
        uint2 s[U];
#pragma unroll
        for (int g = 0; g < U; g++) {   // streamed 8 B per gather (nstream a power of two)
            const uint64_t si = (((uint64_t)i * nt + t) * U + g) & (nstream - 1);
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                         : "=r"(s[g].x), "=r"(s[g].y) : "l"(stream + si), "l"(pf));
        }
#pragma unroll
        for (int g = 0; g < U; g++) {   // independent of the stream: multiply-shift into [0, nwin)
            idx[g] = (uint32_t)(((uint64_t)hash32(t * 0x9E3779B9u + (i * U + g) * 0x85ebca6bu + salt) * nwin) >> 32);
            asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v[g]) : "l"(win + idx[g]), "l"(pl));
        }
#pragma unroll
        for (int g = 0; g < U; g++) acc += (int)s[g].x;
#pragma unroll
        for (int g = 0; g < U; g++) {
            if ((g & 7) < RED_PER8) {
                const int val = DEP ? v[g] - 1 : (int)(idx[g] ^ i);
                atomicMin(win + idx[g], val);
                if (MARK) atomicOr(bm + (idx[g] >> 5), 1u << (idx[g] & 31));
            } else {
                acc += v[g];
            }
        }
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

template <int U, int RED_PER8, bool MARK, bool DEP>
void run(const char *tag, int *win, uint32_t nwin, const uint2 *stream, uint64_t nstream, int *out, int grid,
         uint32_t iters, uint32_t *bm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    mix<U, RED_PER8, MARK, DEP><<<grid, 256>>>(win, nwin, stream, nstream, iters, out, 1, bm);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) mix<U, RED_PER8, MARK, DEP><<<grid, 256>>>(win, nwin, stream, nstream, iters, out, 9 + r, bm);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double g = 3.0 * grid * 256 * iters * U;
    printf("%-26s U=%d grid=%5d win %4.0f MB  gathers %6.1f G/s  REDs %6.1f G/s  stream %5.0f GB/s  (%s)\n", tag, U,
           grid, nwin * 4.0 / (1 << 20), g / (ms * 1e-3) / 1e9, g * RED_PER8 / 8 / (ms * 1e-3) / 1e9,
           g * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxw = (size_t)128 << 20, sbytes = (size_t)2 << 30;
    int *win, *out;
    uint2 *stream;
    uint32_t *bm;
    cudaMalloc(&win, maxw); cudaMalloc(&out, 64); cudaMalloc(&stream, sbytes); cudaMalloc(&bm, maxw / 32);
    cudaMemset(win, 0x7f, maxw); cudaMemset(stream, 1, sbytes); cudaMemset(bm, 0, maxw / 32);
    const uint64_t ns = sbytes / 8;
    for (size_t mb : {24, 50, 100}) {
        const uint32_t nw = (uint32_t)((mb << 20) / 4);
        for (int occ : {4, 8}) {
            const int grid = sms * occ;
            const uint32_t it = 64 * 8 / occ;
            run<8, 0, false, false>("gather only", win, nw, stream, ns, out, grid, it, bm);
            run<8, 1, false, false>("+1/8 RED.MIN", win, nw, stream, ns, out, grid, it, bm);
            run<8, 3, false, false>("+3/8 RED.MIN", win, nw, stream, ns, out, grid, it, bm);
            run<8, 3, true, false>("+3/8 RED.MIN +OR", win, nw, stream, ns, out, grid, it, bm);
            run<8, 3, true, true>("+3/8 dep RED.MIN +OR", win, nw, stream, ns, out, grid, it, bm);
            run<8, 8, false, false>("+8/8 RED.MIN", win, nw, stream, ns, out, grid, it, bm);
        }
        run<16, 0, false, false>("gather only", win, nw, stream, ns, out, sms * 4, 64, bm);
        run<16, 3, true, false>("+3/8 RED.MIN +OR", win, nw, stream, ns, out, sms * 4, 64, bm);
    }
    return 0;
}
