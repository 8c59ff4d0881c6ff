// mma_issue_bench.cu -- how fast can one CTA issue tcgen05.mma (M=128, kind::f16)?
// Variants of the issue loop, each with a try_wait+fence on an already-complete mbarrier and
// a commit every 4 MMAs (the per-stage pattern of a pipelined kernel).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;


template <int V>
__global__ void __launch_bounds__(256, 1) bench(int N, int nstage, int spin, int nacc, const uint8_t *gsrc, long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, done, sink, never;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ (uint32_t)blockIdx.x * 40503u;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (nacc >= 100) {   // random bf16 values in [-1, 1): sign + exponent 0x3F.. + random mantissa
            uint32_t w[4];
            for (int q = 0; q < 4; ++q) {
                h = h * 1664525u + 1013904223u;
                uint32_t lo = 0x3F00u | ((h >> 8) & 0x7Fu) | ((h >> 16) & 0x8000u);
                h = h * 1664525u + 1013904223u;
                uint32_t hi = 0x3F00u | ((h >> 8) & 0x7Fu) | ((h >> 16) & 0x8000u);
                w[q] = lo | (hi << 16);
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        reinterpret_cast<uint4 *>(smem)[i] = v;
    }
    if (nacc >= 100) nacc -= 100;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); mbar_init(&sink, 1); mbar_init(&never, 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&done);
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = make_idesc(false, 128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 96 * 1024);
    const uint64_t da0 = make_sdesc_k_sw128(a0), db0 = make_sdesc_k_sw128(b0);
    long long t0 = clock64();
    if (V == 0) {                       // lane 0 branch, per-MMA descriptor build (current kernel style)
        if (threadIdx.x == 0) {
            for (int st = 0; st < nstage; ++st) {
                mbar_wait(&done, 0);
                tc_fence_after();
                for (int k = 0; k < 4; ++k)
                    umma<false>(tmem, make_sdesc_k_sw128(a0 + k * 32), make_sdesc_k_sw128(b0 + k * 32), idesc, 1);
                umma_commit(&sink);
            }
        }
    } else if (V == 1) {                // warp-converged, elect per stage, descriptors by 64-bit add
        if (threadIdx.x < 32) {
            for (int st = 0; st < nstage; ++st) {
                mbar_wait(&done, 0);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) umma<false>(tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idesc, 1);
                    umma_commit(&sink);
                }
                __syncwarp();
            }
        }
    } else if (V == 3) {                // exact replica of fused_conv's issue pattern (512x7 layer)
        if (threadIdx.x == 0) {
            const uint64_t adesc_t = ((uint64_t)((1296 >> 4) & 0x3FFF) << 16) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
            const uint64_t bdesc_t = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
            const uint32_t a16 = a0 >> 4, b16 = b0 >> 4, lbo16 = 1296 >> 4;
            for (int st = 0; st < nstage; ++st) {
                const int t = st % 9;
                const uint32_t off = (uint32_t)((t / 3) * 9 + t % 3) * (spin == 3 ? 1 : 0);
                mbar_wait(&done, 0);
                tc_fence_after();
                for (int k = 0; k < 4; ++k)
                    umma<false>(tmem, adesc_t | (uint64_t)((a16 + off + 2 * k * lbo16) & 0x3FFF),
                                bdesc_t | (uint64_t)((b16 + 2 * k) & 0x3FFF), idesc, (st | k) != 0);
                umma_commit(&sink);
            }
        }
    } else {                            // lane-0 branch but descriptors by 64-bit add, 16 MMAs per stage
        if (threadIdx.x == 0) {
            for (int st = 0; st < nstage / 4; ++st) {
                mbar_wait(&done, 0);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    umma<false>(tmem + (uint32_t)(((k >> 2) % nacc) * 64), da0 + (uint64_t)((k & 3) * 2),
                                db0 + (uint64_t)((k & 3) * 2), idesc, 1);
                umma_commit(&sink);
            }
        }
        if (spin == 1 && threadIdx.x >= 128 && (threadIdx.x & 31) == 0) mbar_wait(&never, 0);
        if (spin == 2 && threadIdx.x == 128) {
            // bulk-copy noise: 8 KB global -> smem (region after 160 KB) back to back until the MMAs end
            __shared__ uint64_t nb;
            mbar_init(&nb, 1);
            fence_barrier_init();
            uint32_t ph = 0;
            for (int it = 0; it < 4000; ++it) {
                mbar_arrive_expect_tx(&nb, 8192);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];"
                             :: "r"(smem_u32(smem + 160 * 1024)), "l"(gsrc + (size_t)((it * 148 + blockIdx.x) % 4096) * 8192),
                                "r"(smem_u32(&nb)) : "memory");
                mbar_wait(&nb, ph);
                ph ^= 1;
                if (*(volatile uint64_t *)&never != 0 && it > 100) {}
            }
        }
    }
    if (threadIdx.x == 0) {
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
        if (spin) mbar_arrive(&never);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int V>
void run(const char *name, long long *d, int spin = 0, int nacc = 1) {
    static uint8_t *g = nullptr;
    if (!g) { cudaMalloc(&g, (size_t)4096 * 8192); cudaMemset(g, 0, (size_t)4096 * 8192); }
    cudaFuncSetAttribute(bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int N : {64, 128, 256}) {
        const int nstage = 512;
        bench<V><<<148, 256, 200 * 1024>>>(N, nstage, spin, nacc, g, d);
        cudaDeviceSynchronize();
        long long h[148], mx = 0;
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-40s N=%3d : %6.1f cyc/mma (floor %d)\n", name, N, (double)mx / (nstage * 4), N <= 64 ? 50 : N / 2);
    }
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    run<0>("lane0, desc rebuilt, 4/stage", d);
    run<1>("warp+elect, desc add, 4/stage", d);
    run<2>("lane0, desc add, 16/stage", d);
    run<2>("  + 4 warps spinning on mbarrier", d, 1, 1);
    run<2>("  + 4 accumulators (no spin)", d, 0, 4);
    run<2>("  + 4 accumulators + spin", d, 1, 4);
    run<2>("  + bulk-copy noise 8KB chunks", d, 2, 4);
    run<3>("replica, no tap offsets", d, 0, 1);
    run<3>("replica, tap offsets", d, 3, 1);
    run<2>("16/stage, RANDOM data", d, 0, 101);
    run<3>("replica, tap offsets, RANDOM data", d, 3, 101);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
