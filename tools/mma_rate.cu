// mma_rate.cu -- issue and completion rate of back-to-back tcgen05.mma (kind::f16, M = 128, SS
// operands, K = 16 per MMA) by one elected thread, as a function of the swizzle mode / pixel-row
// width (32 / 64 / 128 B), N, and whether the A descriptor starts on a swizzle-atom boundary
// (row offset 0) or mid-atom (row offset 1..7, the row-streaming kernel's column shifts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_rate tools/mma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

struct P {
    int rowbytes, swz, N, shift, nmma, ksteps, vary_shift, nacc;
};

__global__ void __launch_bounds__(128, 1) mma_rate(P p, long long *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        const uint32_t idesc = make_idesc(false, 128, (uint32_t)p.N);
        const uint64_t dtpl = ((uint64_t)1 << 16) | ((uint64_t)((8u * (uint32_t)p.rowbytes) >> 4) << 32) |
                              ((uint64_t)1 << 46) | ((uint64_t)p.swz << 61);
        const uint32_t a16 = (smem_u32(sm) >> 4) + (uint32_t)(p.shift * p.rowbytes >> 4);
        const uint32_t b16 = smem_u32(sm + 64 * 1024) >> 4;
        const uint32_t row16 = (uint32_t)p.rowbytes >> 4;
        long long t0 = 0, t1 = 0, t2 = 0;
        if (elect_one()) {
            t0 = clock64();
#pragma unroll 4
            for (int i = 0; i < p.nmma; ++i) {
                const uint32_t k = (uint32_t)(i % p.ksteps);
                const uint32_t sh = p.vary_shift ? (uint32_t)(i % 9) * row16 : 0u;
                umma<false>(tmem + (uint32_t)((i & 3) * p.N), dtpl | (uint64_t)((a16 + sh + 2u * k) & 0x3FFF),
                            dtpl | (uint64_t)((b16 + 2u * k) & 0x3FFF), idesc, i >= 4 ? 1u : 0u);
            }
            t1 = clock64();
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        t2 = clock64();
        if (lane_id() == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// Converged-warp issue (uniform datapath): 16 MMAs per iteration, descriptors as (lo, hi) words,
// per-MMA offsets compile-time (shift j in 0..8 rows cycling, k-step 0..KS-1).
template <int KS>
__global__ void __launch_bounds__(128, 1) mma_rate_uniform(P p, long long *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        const uint32_t idesc = make_idesc(false, 128, (uint32_t)p.N);
        const uint32_t hi = (uint32_t)(((uint64_t)1 << 46 | (uint64_t)p.swz << 61 | ((uint64_t)((8u * (uint32_t)p.rowbytes) >> 4) << 32)) >> 32);
        const uint32_t lo_a = ((smem_u32(sm) >> 4) + (uint32_t)(p.shift * p.rowbytes >> 4)) | (1u << 16);
        const uint32_t lo_b = (smem_u32(sm + 64 * 1024) >> 4) | (1u << 16);
        const uint32_t row16 = (uint32_t)p.rowbytes >> 4;
        const long long t0 = clock64();
        for (int it = 0; it < p.nmma / 16; ++it) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const uint32_t j = (uint32_t)((m / KS) % 9), k = (uint32_t)(m % KS);
                umma_elect_lohi<false>(tmem + (uint32_t)((m % p.nacc) * p.N), lo_a + (p.vary_shift ? j * row16 : 0u) + 2u * k, hi,
                                       lo_b + 2u * k, hi, idesc, (it > 0 || m >= p.nacc) ? 1u : 0u);
            }
        }
        const long long t1 = clock64();
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if (lane_id() == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// Contention: the MMA warp (1) issues like mma_rate_uniform into columns [0, 4N) while warps 4..11
// either idle (mode 0), loop tcgen05.ld x16 + wait on columns [256, 512) (mode 1, an epilogue's
// TMEM reads), spin on mbarrier.try_wait of a barrier that completes only at the end (mode 2), or
// store to global memory (mode 3).
__global__ void __launch_bounds__(384, 1) mma_contend(P p, int mode, long long *out, float *sink) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, done;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); stop = 0; fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        const uint32_t idesc = make_idesc(false, 128, (uint32_t)p.N);
        const uint32_t hi = (uint32_t)(((uint64_t)1 << 46 | (uint64_t)p.swz << 61 | ((uint64_t)((8u * (uint32_t)p.rowbytes) >> 4) << 32)) >> 32);
        const uint32_t lo_a = (smem_u32(sm) >> 4) | (1u << 16);
        const uint32_t lo_b = (smem_u32(sm + 64 * 1024) >> 4) | (1u << 16);
        const uint32_t row16 = (uint32_t)p.rowbytes >> 4;
        const long long t0 = clock64();
        for (int it = 0; it < p.nmma / 16; ++it) {
#pragma unroll
            for (int m = 0; m < 16; ++m)
                umma_elect_lohi<false>(tmem + (uint32_t)((m & 1) * p.N), lo_a + (uint32_t)(m % 3) * row16, hi, lo_b, hi, idesc,
                                       (it > 0 || m >= 2) ? 1u : 0u);
        }
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if (lane_id() == 0) { stop = 1; mbar_arrive(&done); }
        if (lane_id() == 0 && blockIdx.x == 0) { out[0] = t2 - t0; }
    } else if (warp >= 4) {
        const int q = warp & 3;
        float acc = 0.f;
        if (mode == 1) {
            uint32_t v[16];
            while (!stop) {
                tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + 256u + (uint32_t)((warp >> 2) * 64), v);
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 16; ++k) acc += __uint_as_float(v[k]);
            }
        } else if (mode == 2) {
            mbar_wait(&done, 0);
        } else if (mode == 3) {
            int k = 0;
            while (!stop) { sink[(blockIdx.x * 384 + threadIdx.x + (k & 1023) * 384 * 148) & ((1 << 24) - 1)] = acc; ++k; }
        }
        if (acc == 12345.f) sink[threadIdx.x] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// Register reuse: 8 MMAs in one asm block, either re-using ONE descriptor register pair updated in
// place between MMAs (reuse = 1) or 8 distinct pairs computed up front (reuse = 0).
template <int kReuse>
__global__ void __launch_bounds__(128, 1) mma_reuse(P p, long long *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        const uint32_t idesc = make_idesc(false, 128, (uint32_t)p.N);
        const uint64_t hi = ((uint64_t)1 << 46 | (uint64_t)p.swz << 61 | ((uint64_t)((8u * (uint32_t)p.rowbytes) >> 4) << 32));
        const uint64_t da = hi | (smem_u32(sm) >> 4) | (1u << 16);
        const uint64_t db = hi | (smem_u32(sm + 64 * 1024) >> 4) | (1u << 16);
        const long long t0 = clock64();
        for (int it = 0; it < p.nmma / 8; ++it) {
            if constexpr (kReuse) {
                asm volatile(
                    "{\n\t.reg .pred e;\n\t.reg .b64 a;\n\tmov.b64 a, %1;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n\tadd.s64 a, a, 2;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, %2, %3, 1;\n}" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc));
            } else {
                asm volatile(
                    "{\n\t.reg .pred e;\n\t.reg .b64 a<8>;\n\t"
                    "add.s64 a0, %1, 0;\n\tadd.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
                    "add.s64 a4, %1, 8;\n\tadd.s64 a5, %1, 10;\n\tadd.s64 a6, %1, 12;\n\tadd.s64 a7, %1, 14;\n\t"
                    "elect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, %2, %3, 1;\n}" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc));
            }
        }
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if (lane_id() == 0 && blockIdx.x == 0) { out[0] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long *out, h[2];
    cudaMalloc(&out, 64);
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int nmma = 512;
    printf("%8s %4s %5s %5s %6s | %10s %10s  (cycles per MMA, grid 1 / grid 148)\n", "rowbytes", "N", "shift", "vary", "ksteps",
           "issue", "complete");
    for (int rb : {32, 64, 128})
        for (int N : {16, 48, 64, 128})
            for (int shift : {0, 1})
                for (int vary : {0, 1}) {
                    if (vary && shift) continue;
                    P p{rb, rb == 32 ? 6 : (rb == 64 ? 4 : 2), N, shift, nmma, rb / 32, vary, 4};
                    double r[2][2];
                    for (int gi = 0; gi < 2; ++gi) {
                        const int grid = gi ? 148 : 1;
                        for (int rep = 0; rep < 2; ++rep) mma_rate<<<grid, 128, 100 * 1024>>>(p, out);
                        cudaDeviceSynchronize();
                        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
                        r[gi][0] = (double)h[0] / nmma;
                        r[gi][1] = (double)h[1] / nmma;
                    }
                    printf("%8d %4d %5d %5d %6d | %5.1f/%5.1f %5.1f/%5.1f  %s\n", rb, N, shift, vary, p.ksteps, r[0][0], r[1][0],
                           r[0][1], r[1][1], cudaGetErrorString(cudaGetLastError()));
                }
    printf("converged-warp issue (umma_elect_lohi, 16 MMAs unrolled per iteration); column 'vary' = accumulators rotated:\n");
    cudaFuncSetAttribute(mma_rate_uniform<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(mma_rate_uniform<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(mma_rate_uniform<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int rb : {32, 128})
        for (int N : {16, 48, 64, 128})
            for (int vary : {1, 2, 4}) {     // here: number of accumulators the MMAs rotate over
                P p{rb, rb == 32 ? 6 : (rb == 64 ? 4 : 2), N, 0, nmma, rb / 32, 1, vary};
                double r[2][2];
                for (int gi = 0; gi < 2; ++gi) {
                    const int grid = gi ? 148 : 1;
                    for (int rep = 0; rep < 2; ++rep) {
                        if (rb == 32) mma_rate_uniform<1><<<grid, 128, 100 * 1024>>>(p, out);
                        if (rb == 64) mma_rate_uniform<2><<<grid, 128, 100 * 1024>>>(p, out);
                        if (rb == 128) mma_rate_uniform<4><<<grid, 128, 100 * 1024>>>(p, out);
                    }
                    cudaDeviceSynchronize();
                    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
                    r[gi][0] = (double)h[0] / nmma;
                    r[gi][1] = (double)h[1] / nmma;
                }
                printf("%8d %4d %5d %5d %6d | %5.1f/%5.1f %5.1f/%5.1f  %s\n", rb, N, 0, vary, p.ksteps, r[0][0], r[1][0],
                       r[0][1], r[1][1], cudaGetErrorString(cudaGetLastError()));
            }
    {
        float *sink;
        cudaMalloc(&sink, sizeof(float) << 24);
        cudaFuncSetAttribute(mma_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        printf("contention (MMA warp alone vs 8 other warps doing: 1 tcgen05.ld loops, 2 mbarrier wait, 3 global stores):\n");
        for (int N : {16, 48})
            for (int mode = 0; mode < 4; ++mode) {
                P p{32, 6, N, 0, nmma, 1, 1, 2};
                for (int rep = 0; rep < 2; ++rep) mma_contend<<<148, 384, 100 * 1024>>>(p, mode, out, sink);
                cudaDeviceSynchronize();
                cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
                printf("  N=%3d mode %d: %6.1f cycles per MMA  %s\n", N, mode, (double)h[0] / nmma,
                       cudaGetErrorString(cudaGetLastError()));
            }
    }
    cudaFuncSetAttribute(mma_reuse<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(mma_reuse<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    printf("descriptor register reuse (8 MMAs per asm block, one accumulator):\n");
    for (int N : {16, 48, 128})
        for (int reuse = 0; reuse < 2; ++reuse) {
            P p{32, 6, N, 0, nmma, 1, 0, 1};
            for (int rep = 0; rep < 2; ++rep) {
                if (reuse) mma_reuse<1><<<148, 128, 100 * 1024>>>(p, out);
                else mma_reuse<0><<<148, 128, 100 * 1024>>>(p, out);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
            printf("  N=%3d reuse %d: %6.1f cycles per MMA  %s\n", N, reuse, (double)h[0] / nmma, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
