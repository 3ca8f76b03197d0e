// Where does a dense SSSP round spend its time?  Synthetic rand-25M-shaped
// graph (n = 25M, out-degree 4, uniform targets), a fraction f of vertices
// active, finite random distances; one VERTEX round of the product kernel
// k_expand_warp in three modes (FK_PROBE): 0 = expansion chain only (bitmap ->
// items -> row offsets / own value -> arcs), 1 = + gather of the target value
// and compare, 2 = the real round (+ RED.MIN and bitmap RED.OR on success).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFK_PROBE -I include \
//      -o tools/expand_probe tools/expand_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1903_01665_b200/csrc/kernels.cuh"
using namespace fk;

__global__ void k_fill(uint32_t n, uint32_t m, uint32_t deg, uint32_t *row_off, uint2 *cw, int32_t *val,
                       uint32_t *bm, uint32_t nwords, uint32_t frac_pct, uint32_t seed) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
        uint64_t h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
        if (i < m) cw[i] = make_uint2((uint32_t)((h >> 8) % n), 1 + (uint32_t)(h % 100));
        if (i <= n) row_off[i] = (uint32_t)(i * deg);
        if (i < n) val[i] = (int32_t)((h >> 20) % 1000);
        if (i < nwords) {
            uint32_t w = 0;
            for (int b = 0; b < 32; b++) {
                uint64_t g = (i * 32 + b + 7) * 0xD6E8FEB86659FD93ull ^ seed;
                g ^= g >> 32;
                if (i * 32 + b < n && (g % 100) < frac_pct) w |= 1u << b;
            }
            bm[i] = w;
        }
    }
}

template <int U, int MINB>
float run(const Args &a, int grid, int mode, const int32_t *val0, int reps) {
    cudaMemcpyToSymbol(fk_probe_mode, &mode, sizeof mode);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaMemcpy(a.val, val0, (size_t)a.n * 4, cudaMemcpyDeviceToDevice);
        Ctrl h = {};
        h.iter = 2; h.cap = 1000;
        cudaMemcpy(a.ctrl, &h, sizeof h, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        k_expand_warp<SSSP, VERTEX, 256, U, MINB><<<grid, 256>>>(a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char **argv) {
    const uint32_t n = 25000000, deg = 4, m = n * deg;
    const uint32_t nwords = ((n + 31) / 32 + 3) & ~3u;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *row_off, *bm, *fr, *cnt32;
    uint2 *cw;
    int32_t *val, *val0;
    Ctrl *ctrl;
    unsigned long long *cnt;
    cudaMalloc(&row_off, (n + 1) * 4ull); cudaMalloc(&cw, m * 8ull); cudaMalloc(&val, n * 4ull);
    cudaMalloc(&val0, n * 4ull); cudaMalloc(&bm, 4ull * nwords * 4); cudaMalloc(&fr, 2 * (n + 1) * 4ull);
    cudaMalloc(&ctrl, sizeof(Ctrl)); cudaMalloc(&cnt, 3ull * 8 * sms * 8);
    Args a = {};
    a.n = n; a.m = m; a.nwords = nwords; a.row_off = row_off; a.cw = cw; a.rowb = row_off; a.cwb = cw; a.nblk = 1;
    a.val = val; a.bm0 = bm; a.bm1 = bm + nwords; a.bm2 = bm + 2 * nwords; a.vis = bm + 3 * nwords;
    a.fr0 = fr; a.fr1 = fr + n + 1; a.ctrl = ctrl; a.cnt = cnt; a.dense_div = 16; a.blk_div = 0;
    (void)cnt32;
    for (uint32_t frac : {10u, 30u, 60u, 100u}) {
        cudaMemset(bm, 0, 4ull * nwords * 4);
        k_fill<<<sms * 8, 256>>>(n, m, deg, row_off, cw, val0, a.bm1, nwords, frac, 12345u);   // bm[(iter-1)%3] = bm1
        cudaDeviceSynchronize();
        const double arcs = (double)m * frac / 100.0;
        for (int mode = 0; mode < 3; mode++) {
            float t43 = run<4, 3>(a, sms * 3, mode, val0, 3);
            float t24 = run<2, 4>(a, sms * 4, mode, val0, 3);
            float t82 = run<8, 2>(a, sms * 2, mode, val0, 3);
            printf("active %3u%%  mode %d  U4/3: %7.1f us (%6.1f G arcs/s)  U2/4: %7.1f us (%6.1f)  U8/2: %7.1f us (%6.1f)\n",
                   frac, mode, 1e3 * t43, arcs / t43 / 1e6, 1e3 * t24, arcs / t24 / 1e6, 1e3 * t82, arcs / t82 / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
