// clock_check.cu -- does %clock64 tick at the SM clock on this B200?  One thread spins on a
// dependent integer chain between two (clock64, globaltimer) samples; the ratio of the deltas is
// clock64's rate.  Also times 36*256 back-to-back tcgen05.mma-free spins as a control.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/clock_check tools/clock_check.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long *out, int iters) {
    unsigned long long g0, g1;
    long long c0, c1;
    unsigned x = threadIdx.x + 1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
    for (int i = 0; i < iters; ++i) x = x * 1664525u + 1013904223u;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1) : "r"(x));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1) : "l"(c1));
    out[0] = c1 - c0; out[1] = (long long)(g1 - g0); out[2] = x;
}
int main() {
    long long *d, h[3];
    cudaMalloc(&d, 3 * sizeof(long long));
    for (int rep = 0; rep < 6; ++rep) {
        int iters = 1 << (20 + (rep & 1));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<1, 32>>>(d, iters);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("iters %d: clock64 %lld  globaltimer %lld ns  event %.1f us -> clock64 rate %.0f MHz\n", iters, h[0], h[1],
               ms * 1e3, h[0] * 1e3 / (double)h[1]);
    }
    return 0;
}
