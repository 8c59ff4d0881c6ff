// mbar_pingpong.cu -- round-trip latency of an mbarrier hand-off between two warps of one CTA
// (warp A arrives on bar0, warp B waits on it and arrives on bar1, warp A waits on bar1), with
// mbarrier.try_wait (default suspend), try_wait with a suspend-time hint, and test_wait polling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mbar_pingpong tools/mbar_pingpong.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ void wait_test(uint64_t *bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t ok = 0;
    do {
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns) {
    const uint32_t addr = smem_u32(bar);
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t@!P1 bra W_%=;\n}"
                 ::"r"(addr), "r"(parity), "r"(ns) : "memory");
}

template <int MODE>
__global__ void pingpong(long long *out, int iters, int warps) {
    __shared__ uint64_t bar[2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
    __syncthreads();
    auto wait = [&](uint64_t *b, uint32_t p) {
        if (MODE == 0) mbar_wait(b, p);
        else if (MODE == 1) wait_hint(b, p, 0x989680u);
        else wait_test(b, p);
    };
    const long long t0 = clock64();
    if (warp == 0) {
        for (int i = 0; i < iters; ++i) {
            if (lane == 0) mbar_arrive(&bar[0]);
            wait(&bar[1], i & 1);
        }
    } else if (warp == 1) {
        for (int i = 0; i < iters; ++i) {
            wait(&bar[0], i & 1);
            if (lane == 0) mbar_arrive(&bar[1]);
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    long long *out, h;
    cudaMalloc(&out, 64);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) pingpong<0><<<1, 256>>>(out, iters, 8);
            if (mode == 1) pingpong<1><<<1, 256>>>(out, iters, 8);
            if (mode == 2) pingpong<2><<<1, 256>>>(out, iters, 8);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %.1f cycles per round trip, err=%s\n", mode,
               mode == 0 ? "try_wait" : mode == 1 ? "try_wait + suspend hint" : "test_wait poll", (double)h / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
