// mma_bench2.cu -- tcgen05.mma (kind::f16, M=128, cta_group::1) throughput on B200 vs N, operand
// data (zero / random bf16) and the SW128 A start row inside the 1024-byte atom (the fused
// kernel's tap offsets start A mid-atom).  One CTA per SM, one thread issues nmma MMAs
// back to back (k-step advance as in the kernel), then commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench2 tools/mma_bench2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__global__ void __launch_bounds__(128, 1) bench(int N, int nmma, int arow, int rnd, int m256, long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        // two bf16 in [-2, 2): sign, exponent 126..128, random mantissa
        uint32_t lo = ((h & 1) << 15) | ((126u + ((h >> 1) % 3)) << 7) | ((h >> 3) & 0x7F);
        uint32_t hi = (((h >> 10) & 1) << 15) | ((126u + ((h >> 11) % 3)) << 7) | ((h >> 14) & 0x7F);
        reinterpret_cast<uint32_t *>(smem)[i] = rnd ? (lo | (hi << 16)) : 0u;
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = make_idesc(false, 128, N);
    const uint32_t a0 = smem_u32(smem) + (uint32_t)arow * 128u, b0 = smem_u32(smem + 96 * 1024);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int m = 0; m < nmma; ++m) {
            const int k = m & 3;
            const uint64_t da = make_sdesc_k_sw128(a0 + k * 32);
            const uint64_t db = make_sdesc_k_sw128(b0 + k * 32);
            umma<false>(tmem + (uint32_t)((m >> 2) & 1) * (uint32_t)(m256 ? 0 : 256), da, db, idesc, 1);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int nmma = 4096;
    for (int rnd = 0; rnd < 2; ++rnd)
        for (int arow : {0, 1, 3})
            for (int N : {16, 32, 64, 128, 256}) {
                bench<<<148, 128, 200 * 1024>>>(N, nmma, arow, rnd, 1, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("data=%s arow=%d N=%3d : %6.1f cyc/mma  (math-bound %5.1f)\n", rnd ? "rand" : "zero", arow, N,
                       (double)mx / nmma, 128.0 * N * 16 * 2 / 8192.0);
            }
    return 0;
}
