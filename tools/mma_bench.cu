// mma_bench.cu -- microbenchmark: tcgen05.mma (kind::f16, M=128, cta_group::1) issue/execute
// rate for different smem operand layouts.  One CTA per SM; operands are left as whatever smem
// holds (zero-filled); D accumulates in TMEM.  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ uint64_t sdesc_interleave(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// mode 0: A sw128, B sw128 ; mode 1: A interleave (aligned), B sw128 ; mode 2: A interleave with
// row offset `off` (16 B units), B sw128 ; mode 3: A interleave, B interleave
// sync: 0 none; 1 every 4 MMAs: try_wait on a completed mbarrier + fence::after;
//       2 = 1 + tcgen05.commit to a second mbarrier every 4 MMAs; 3 = commit only
__global__ void __launch_bounds__(128, 1) bench(int mode, int N, int nmma, int off, int lbo, int sync, long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, done, sink;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); mbar_init(&sink, 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&done);   // phase 0 of `done` completes
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = make_idesc(false, 128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 96 * 1024);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int m = 0; m < nmma; ++m) {
            const int k = m & 3;
            uint64_t da, db;
            if (mode == 0) da = make_sdesc_k_sw128(a0 + k * 32);
            else da = sdesc_interleave(a0 + (uint32_t)(2 * k) * lbo + (mode == 2 ? off * 16 : 0), lbo, 128);
            if (mode == 3) db = sdesc_interleave(b0 + (uint32_t)(2 * k) * 4096, 4096, 128);
            else db = make_sdesc_k_sw128(b0 + k * 32);
            if ((sync == 1 || sync == 2) && k == 0) { mbar_wait(&done, 0); tc_fence_after(); }
            umma<false>(tmem, da, db, idesc, 1);
            if ((sync == 2 || sync == 3) && k == 3) umma_commit(&sink);
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
    const int nmma = 2048;
    const char *names[] = {"A sw128   B sw128", "A inter   B sw128", "A inter+off B sw128", "A inter   B inter"};
    for (int sync = 0; sync < 4; ++sync)
        for (int mode : {0, 2})
            for (int N : {64, 256}) {
                int grid = 148, off = 1, lbo = 9280;
                bench<<<grid, 128, 200 * 1024>>>(mode, N, nmma, off, lbo, sync, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                long long h[148];
                cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("sync=%d %-22s N=%3d : %6.1f cyc/mma (ideal %d)\n", sync, names[mode], N, (double)mx / nmma, N / 2);
            }
    return 0;
}
