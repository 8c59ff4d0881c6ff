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

__device__ __forceinline__ bool lane_is0() { return (threadIdx.x & 31) == 0; }
__global__ void __launch_bounds__(256, 1) bench(int N, int nmma, int arow, int rnd, int m256, long long *out,
                                               int taps, int stw, int xb = 16) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, done2, sink2;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        // two bf16 in [-2, 2): sign, exponent 126..128, random mantissa
        uint32_t lo = ((h & 1) << 15) | ((126u + ((h >> 1) % 3)) << 7) | ((h >> 3) & 0x7F);
        uint32_t hi = (((h >> 10) & 1) << 15) | ((126u + ((h >> 11) % 3)) << 7) | ((h >> 14) & 0x7F);
        reinterpret_cast<uint32_t *>(smem)[i] = rnd ? (lo | (hi << 16)) : 0u;
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done2, 1); mbar_init(&sink2, 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&done2);
    __syncthreads();
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = make_idesc(false, 128, N);
    const uint32_t a0 = smem_u32(smem) + (uint32_t)arow * 128u, b0 = smem_u32(smem + 48 * 1024);
    long long t0 = 0, t1 = 0;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (threadIdx.x == 0 && stw < 2) {
        t0 = clock64();
        for (int m = 0; m < nmma; ++m) {
            const int k = m & 3;
            // "taps": the A start row moves by 1 row per tap (mid-atom), B switches to another tile
            const int t = taps > 1 ? (m >> 2) % taps : 0;
            const uint64_t da = make_sdesc_k_sw128(a0 + (uint32_t)t * 128u + k * 32);
            const uint64_t db = make_sdesc_k_sw128(b0 + (uint32_t)t * (uint32_t)(N * 128) % (48u * 1024u) + k * 32);
            umma<false>(tmem + (uint32_t)((m >> 2) & 1) * (uint32_t)(m256 ? 0 : 256), da, db, idesc, 1);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        stop = 1;
        (void)t1;
    } else if (threadIdx.x >= 32 && threadIdx.x < 64 && stw >= 2) {
        // lean issuer (warp 1, converged): stw 2 = same A/B every MMA; 3 = conv-like taps (A row
        // offsets {0,1,2,16,17,18,32,33,34}, one 8 KB B tile per tap); 4 = 3 + a concurrent smem
        // writer warp (TMA-like traffic)
        __syncwarp();
        long long s0 = clock64();
        const uint64_t da0 = make_sdesc_k_sw128(a0), db0 = make_sdesc_k_sw128(b0);
        const uint32_t dcol = tmem;
        for (int m = 0; m < nmma; m += 36) {
            if (stw >= 5) {
                // per-step sync like the conv kernel: wait A, fence, wait B, fence
                mbar_wait_warp(&done2, 0);
                tc_fence_after();
                mbar_wait_warp(&done2, 0);
                tc_fence_after();
            }
            for (int t = 0; t < 9; ++t) {
                uint64_t da = da0, db = db0;
                if (stw >= 3) {
                    da += (uint64_t)(((t / 3) * xb + (t % 3)) * 8);
                    db += (uint64_t)(t * N * 8);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_elect<false>(dcol, da + 2 * k, db + 2 * k, idesc, 1);
            }
            if (stw >= 6) { umma_commit_elect(&sink2); umma_commit_elect(&sink2); }
        }
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        if (lane_is0()) out[blockIdx.x] = clock64() - s0;
        if (lane_is0()) stop = 1;
    } else if (threadIdx.x >= 64 && stw == 7) {
        // other warps block in mbarrier.try_wait (like the fused kernel's producer / epilogue warps)
        uint32_t ok = 0;
        while (!stop) {
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(smem_u32(&sink2)), "r"(0u) : "memory");
        }
    } else if (threadIdx.x >= 64 && threadIdx.x < 96 && stw >= 4 && stw < 7) {
        uint4 *dst = reinterpret_cast<uint4 *>(smem + 180 * 1024);
        int i = threadIdx.x - 64;
        while (!stop) {
#pragma unroll
            for (int r = 0; r < 8; ++r) dst[(i + r * 32) & 255] = make_uint4(r, i, 0, 0);
        }
    } else if (threadIdx.x >= 64 && stw == 1) {
        // concurrent smem writes (TMA-like traffic) into a region the MMAs do not read
        uint4 *dst = reinterpret_cast<uint4 *>(smem + 150 * 1024);
        int i = threadIdx.x - 64;
        while (!stop) {
            for (int r = 0; r < 16; ++r) dst[(i + r * 64) & 511] = make_uint4(r, i, 0, 0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main(int argc, char **argv) {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int nmma = 36 * 128;
    if (argc > 2) {   // blocked-waiter test: 128 vs 256 threads, other warps in try_wait
        for (int thr : {128, 256})
            for (int stw : {3, 7})
                for (int N : {16, 32, 64, 128}) {
                    bench<<<148, thr, 200 * 1024>>>(N, nmma, 0, 1, 1, d, 1, stw, 9);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                    long long h[148];
                    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                    long long mx = 0;
                    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
                    printf("threads=%d stw=%d N=%3d : %6.1f cyc/mma\n", thr, stw, N, (double)mx / nmma);
                }
        return 0;
    }
    if (argc > 1) {   // row-pitch sweep: conv tap offsets (t/3)*xb + t%3 (the fused kernel's patch width)
        for (int xb : {16, 8, 9, 10, 13, 18, 30})
            for (int N : {32, 64, 128}) {
                bench<<<148, 128, 200 * 1024>>>(N, nmma, 0, 1, 1, d, 1, 3, xb);
                cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("xb=%2d N=%3d : %6.1f cyc/mma\n", xb, N, (double)mx / nmma);
            }
        return 0;
    }

    for (int stw = 3; stw < 7; ++stw)
        for (int taps : {1})
            for (int N : {32, 64, 128}) {
                const int rnd = 1, arow = 0;
                bench<<<148, 128, 200 * 1024>>>(N, nmma, arow, rnd, 1, d, taps, stw);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("smem-writer=%d taps=%d N=%3d : %6.1f cyc/mma  (math-bound %5.1f)\n", stw, taps, N,
                       (double)mx / nmma, 128.0 * N * 16 * 2 / 8192.0);
            }
    return 0;
}
