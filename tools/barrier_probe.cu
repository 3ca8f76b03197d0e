// Cost of a software grid barrier (atomic arrive + generation spin) vs
// cooperative_groups grid.sync(), for several grid sizes.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

struct Bar { unsigned arrive, gen, pad[30]; };

__device__ __forceinline__ unsigned ldv(const unsigned *p) { return *(const volatile unsigned *)p; }

__global__ void k_soft(Bar *b, int iters, int nsleep) {
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned gen = ldv(&b->gen);
            __threadfence();
            unsigned a = atomicAdd(&b->arrive, 1u);
            if (a == gridDim.x - 1) { b->arrive = 0; __threadfence(); atomicExch(&b->gen, gen + 1); }
            else { while (ldv(&b->gen) == gen) { if (nsleep) __nanosleep(nsleep); } }
            __threadfence();
        }
        __syncthreads();
    }
}
__global__ void k_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; i++) g.sync();
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    Bar *b; cudaMalloc(&b, sizeof(Bar)); cudaMemset(b, 0, sizeof(Bar));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2000;
    for (int per : {1, 2, 3, 4}) {
        int grid = sms * per;
        for (int ns : {0, 32, 100}) {
            void *args[] = {&b, (void *)&iters, &ns};
            cudaLaunchCooperativeKernel((void *)k_soft, grid, 256, args, 0, 0);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)k_soft, grid, 256, args, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("soft  grid=%4d nanosleep=%3d : %.2f us/barrier  (%s)\n", grid, ns, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
        }
        void *args2[] = {(void *)&iters};
        cudaLaunchCooperativeKernel((void *)k_cg, grid, 256, args2, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_cg, grid, 256, args2, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("cg    grid=%4d               : %.2f us/barrier  (%s)\n", grid, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
