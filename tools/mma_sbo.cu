// mma_sbo.cu -- tcgen05.mma (kind::f16, M=128) rate for the fused conv kernel's A-operand layouts:
// the 8-row-group stride SBO (1024 B = consecutive patch rows; Xb * 128 B = the grp8 lane layout),
// the tap row offsets of a patch of width xb ({0,1,2,xb,xb+1,...} rows), and MT accumulators.
// One CTA per SM, a converged issuer warp (one elected lane), 9 taps x 4 k-steps per accumulator
// per chunk, random bf16 data.  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_sbo tools/mma_sbo.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ void bulk1d_(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// stream > 0: warp 2 keeps 32 KB bulk copies (L2-resident source) landing in a 2-stage ring at smem
// offset 128 KB while the MMAs run (the fused kernel's loads next to its MMAs)
__global__ void __launch_bounds__(256, 1) bench(int N, int chunks, int sbo, int xb, int mt, int bpertap, long long *out,
                                               const uint8_t *gsrc = nullptr, int stream = 0, int spin = 0,
                                               const int *voff = nullptr, int sync = 0, int rot = 1, int gate = 0) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, sfull[2], done_bar, ready, sink[2], ring[8];
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    for (int i = threadIdx.x; i < 190 * 1024 / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        uint32_t lo = ((h & 1) << 15) | ((126u + ((h >> 1) % 3)) << 7) | ((h >> 3) & 0x7F);
        uint32_t hi = (((h >> 10) & 1) << 15) | ((126u + ((h >> 11) % 3)) << 7) | ((h >> 14) & 0x7F);
        reinterpret_cast<uint32_t *>(smem)[i] = lo | (hi << 16);
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&sfull[0], 1); mbar_init(&sfull[1], 1); mbar_init(&done_bar, 1); mbar_init(&ready, 1);
                            mbar_init(&sink[0], 1); mbar_init(&sink[1], 1);
                            for (int i = 0; i < 8; ++i) mbar_init(&ring[i], 1);
                            stop = 0; fence_barrier_init(); }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&ready);      // completes phase 0: waits on parity 0 pass at once
    __syncthreads();
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, tslot, 0);
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    if (warp == 1) {
        const uint32_t idesc = make_idesc(false, 128, (uint32_t)N);
        const uint64_t tpl = ((uint64_t)1 << 16) | ((uint64_t)((uint32_t)sbo >> 4) << 32) | ((uint64_t)1 << 46) |
                             ((uint64_t)2 << 61);
        const uint32_t a16 = smem_u32(smem) >> 4, b16 = smem_u32(smem + 48 * 1024) >> 4;
        const uint64_t da0 = tpl | a16, db0 = tpl | b16;
        const uint64_t dbn = (((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
                              ((uint64_t)2 << 61)) | b16;
        const uint32_t mstride16 = (uint32_t)(16 * xb) * 8u;    // stacked M-tiles: 16 rows of xb patch rows
        // voff: per-tap descriptor offsets read from global memory (vector registers: the operands then
        // reach the MMA through R2UR, as in the fused kernel's issue loop)
        int vo[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) vo[t] = voff ? __ldg(voff + t) : ((t / 3) * xb + (t % 3)) * 8;
        __syncwarp();
        const long long s0 = clock64();
        for (int c = 0; c < chunks; ++c) {
            if (gate > 0 && c >= gate) {   // chunk c may start once chunk c - gate's MMAs completed (a gate-deep ring)
                const int slot = c % gate;
                mbar_wait_warp(&ring[slot], (uint32_t)(((c - gate) / gate) & 1));
                tc_fence_after();
            }
            if (sync) {   // the fused kernel's per-step protocol: wait A, fence, wait B, fence ... commit, commit
                mbar_wait_warp(&ready, 0);
                tc_fence_after();
                mbar_wait_warp(&ready, 0);
                tc_fence_after();
            }
            if (elect_one()) {
                for (int m = 0; m < mt; ++m) {
                    const uint32_t dm = tmem + (uint32_t)(m * N);
#pragma unroll
                    for (int t = 0; t < 9; ++t) {
                        // rot > 1: the operands rotate over `rot` stage buffers chunk by chunk, as the fused
                        // kernel's rings do (A stages 24 KB apart, B stages 72 KB apart)
                        const uint32_t r = rot > 1 ? (uint32_t)(c % rot) : 0u;
                        const uint64_t da = da0 + (uint64_t)vo[t] + (uint64_t)(m * mstride16) + (uint64_t)(r * (24u * 1024u / 16u));
                        const uint64_t db = dbn + (uint64_t)(bpertap ? t * N * 8 : 0) + (uint64_t)(r * (72u * 1024u / 16u));
#pragma unroll
                        for (int k = 0; k < 4; ++k) umma<false>(dm, da + 2 * k, db + 2 * k, idesc, (c | t | k) ? 1u : 0u);
                    }
                }
            }
            __syncwarp();
            if (sync) {
                umma_commit_elect(&sink[0]);
                umma_commit_elect(&sink[1]);
                __syncwarp();
            }
            if (gate > 0) {
                umma_commit_elect(&ring[c % gate]);
                __syncwarp();
            }
        }
        (void)db0;
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        if ((threadIdx.x & 31) == 0) { out[blockIdx.x] = clock64() - s0; stop = 1; mbar_arrive(&done_bar); }
    } else if (spin && (warp == 0 || warp >= 4)) {
        // the fused kernel's waiting warps: every lane of warps 0 and 4-7 spins in try_wait
        mbar_wait(&done_bar, 0);
    } else if (warp == 2 && stream && (threadIdx.x & 31) == 0) {
        uint32_t ph[2] = {0, 0};
        long long n = 0;
        for (int s = 0; !stop; s ^= 1, ++n) {
            if (n >= 2) { mbar_wait(&sfull[s], ph[s]); ph[s] ^= 1; }
            mbar_arrive_expect_tx(&sfull[s], 32768);
            bulk1d_(smem + 128 * 1024 + s * 32768, gsrc + (size_t)blockIdx.x * 262144 + (size_t)(n & 7) * 32768, 32768, &sfull[s]);
        }
        for (int s = 0; s < 2; ++s) if (n > s) mbar_wait(&sfull[s], ph[s]);
        out[gridDim.x + blockIdx.x] = n;        // copies issued while the MMAs ran
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
    long long *d;
    cudaMalloc(&d, 2 * 148 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { int N, sbo, xb, mt, bpt; const char *what; };
    uint8_t *gsrc;
    cudaMalloc(&gsrc, (size_t)148 * 262144);
    cudaMemset(gsrc, 1, (size_t)148 * 262144);
    {
        int hv[9];
        for (int t = 0; t < 9; ++t) hv[t] = ((t / 3) * 10 + (t % 3)) * 8;
        int *dv;
        cudaMalloc(&dv, sizeof(hv));
        cudaMemcpy(dv, hv, sizeof(hv), cudaMemcpyHostToDevice);
        for (int gate : {1, 2, 3, 4}) {
            bench<<<148, 128, 200 * 1024>>>(64, 64, 1280, 10, 1, 1, d, gsrc, 0, 0, nullptr, 0, 1, gate);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("N= 64, chunk c gated on the MMA completion (commit) of chunk c-%d: %6.1f cyc/mma\n", gate, mx / (64 * 36.0));
        }
        for (int rot : {1, 2}) {
            bench<<<148, 128, 200 * 1024>>>(64, 64, 1280, 10, 1, 1, d, gsrc, 0, 0, nullptr, 1, rot);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("N= 64 grp8 Xb=10, per-step sync, operands rotating over %d stage buffer(s): %6.1f cyc/mma\n", rot,
                   mx / (64 * 36.0));
        }
        for (int sync : {0, 1}) {
            bench<<<148, 128, 200 * 1024>>>(64, 64, 1280, 10, 1, 1, d, gsrc, 0, 0, nullptr, sync);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("N= 64 grp8 Xb=10, %s: %6.1f cyc/mma\n", sync ? "per-36-MMA waits + fences + 2 commits    " : "no per-step synchronisation              ",
                   mx / (64 * 36.0));
        }
        for (int vec : {0, 1}) {
            bench<<<148, 128, 200 * 1024>>>(64, 64, 1280, 10, 1, 1, d, gsrc, 0, 0, vec ? dv : nullptr);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("N= 64 grp8 Xb=10, tap offsets %s: %6.1f cyc/mma\n", vec ? "from global memory (vector regs, R2UR)" : "compile-time (uniform)                 ",
                   mx / (64 * 36.0));
        }
    }
    for (int spin : {0, 1})
        for (int thr : {128, 256}) {
            if (spin && thr == 128) continue;
            bench<<<148, thr, 200 * 1024>>>(64, 64, 1280, 10, 1, 1, d, gsrc, 0, spin);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("N= 64 grp8 Xb=10, %d threads, %s: %6.1f cyc/mma\n", thr, spin ? "warps 0 and 4-7 spinning in try_wait" : "idle warps at the barrier",
                   mx / (64 * 36.0));
        }
    for (int stream : {0, 1})
        for (int N : {64, 128, 256}) {
            const int chunks = 64;
            bench<<<148, 128, 200 * 1024>>>(N, chunks, 1024, 16, 1, N == 256 ? 0 : 1, d, gsrc, stream);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            long long nc[148];
            cudaMemcpy(nc, d + 148, sizeof(nc), cudaMemcpyDeviceToHost);
            double mean_n = 0;
            for (int i = 0; i < 148; ++i) mean_n += nc[i] / 148.0;
            printf("N=%3d %s %6.1f cyc/mma", N, stream ? "with a concurrent 32 KB bulk-copy stream:" : "alone:                                   ",
                   mx / (chunks * 36.0));
            if (stream) printf("   copies meanwhile: %6.1f B/clk per SM", mean_n * 32768.0 / mx);
            printf("\n");
        }
    const Cfg cfgs[] = {
        {64, 1024, 16, 1, 1, "SBO 1024, patch width 16 (microbenchmark layout)"},
        {64, 1024, 10, 1, 1, "SBO 1024, patch width 10 (lanes over consecutive rows)"},
        {64, 1280, 10, 1, 1, "SBO 1280 = grp8 with Xb = 10"},
        {64, 1536, 12, 1, 1, "SBO 1536 = grp8 with Xb = 12 (CSRNet)"},
        {64, 1280, 10, 2, 1, "grp8 Xb = 10, MT = 2"},
        {64, 1024, 10, 2, 1, "SBO 1024, Xb = 10, MT = 2"},
        {64, 1280, 10, 1, 0, "grp8 Xb = 10, one B tile for all taps"},
        {128, 1024, 16, 1, 1, "N = 128, SBO 1024"},
        {128, 1280, 10, 1, 1, "N = 128, grp8 Xb = 10"},
        {256, 1280, 10, 1, 1, "N = 256, grp8 Xb = 10"},
        {32, 1024, 16, 1, 1, "N = 32, SBO 1024"},
        {32, 1280, 10, 1, 1, "N = 32, grp8 Xb = 10"},
    };
    for (const Cfg &c : cfgs) {
        const int chunks = 64;
        bench<<<148, 128, 200 * 1024>>>(c.N, chunks, c.sbo, c.xb, c.mt, c.bpt, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double nm = (double)chunks * c.mt * 36;
        printf("N=%3d %-55s %6.1f cyc/mma (math bound %5.1f)\n", c.N, c.what, mx / nm, 128.0 * c.N * 16 * 2 / 8192.0);
    }
    return 0;
}
