// tmem_ld_bench.cu -- latency of tcgen05.ld (+ wait::ld) from an epilogue-like warp on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_ld_bench tools/tmem_ld_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

template <int NLD>
__global__ void __launch_bounds__(128, 1) bench(long long *out, int iters, float *sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = slot + ((uint32_t)(warp * 32) << 16);
    uint32_t v[16 * NLD];
    float acc = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < NLD; ++k)
            tmem_ld_32x32b_x16(base + (uint32_t)(k * 16 + (it & 7) * 64), *reinterpret_cast<uint32_t(*)[16]>(&v[16 * k]));
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16 * NLD; ++k) acc += __uint_as_float(v[k]);
    }
    const long long t1 = clock64();
    if (threadIdx.x % 32 == 0) out[blockIdx.x * 4 + warp] = t1 - t0;
    sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(slot);
}

int main() {
    long long *out;
    float *sink;
    cudaMalloc(&out, 8 * 148 * 4);
    cudaMalloc(&sink, 4 * 256);
    long long h[4];
    const int iters = 10000;
    bench<1><<<1, 128>>>(out, iters, sink);
    cudaDeviceSynchronize();
    bench<1><<<1, 128>>>(out, iters, sink);
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("1 x tcgen05.ld.x16 + wait + 16 FADD: %.1f cycles / iter (warp 0), err=%s\n", (double)h[0] / iters,
           cudaGetErrorString(cudaGetLastError()));
    bench<3><<<1, 128>>>(out, iters, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("3 x tcgen05.ld.x16 + wait + 48 FADD: %.1f cycles / iter (warp 0)\n", (double)h[0] / iters);
    bench<4><<<148, 128>>>(out, iters, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("4 x tcgen05.ld.x16 + wait + 64 FADD (148 CTAs): %.1f cycles / iter (warp 0)\n", (double)h[0] / iters);
    return 0;
}
