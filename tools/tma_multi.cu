// tma_multi.cu -- is a CTA's bulk-copy (TMA) stream serialised per CTA or per issuing warp?
// One CTA per SM streams L2-resident tiles (a private 256 KB window per CTA, read repeatedly) into
// smem rings with `nprod` producer warps, each with its own ring of `nst` stages and its own
// consumer warp that releases a stage as soon as it lands.  Prints bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_multi tools/tma_multi.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ void bulk1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int WIN = 256 * 1024;

__global__ void __launch_bounds__(512, 1) bench(const uint8_t *g, int tile, int ntiles, int nst, int nprod, int share,
                                                long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8][16], empty[8][16];
    __shared__ long long t_end[8];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int p = 0; p < nprod; ++p)
            for (int i = 0; i < nst; ++i) { mbar_init(&full[p][i], 1); mbar_init(&empty[p][i], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    // share: 0 private windows; 1 every CTA reads the same window in the same order; 2 groups of 32
    // CTAs share a window (the fused kernel's weight boxes: 4 f-slices over 128 CTAs)
    const uint8_t *base = g + (size_t)(share == 1 ? 0 : share == 2 ? blockIdx.x / 32 : blockIdx.x) * WIN;
    const int per = ntiles / nprod;
    const long long t0 = clock64();
    const int p = warp / 2;                       // producer p = warp 2p, its consumer = warp 2p + 1
    if (p < nprod && lane == 0) {
        uint8_t *ring = smem + (size_t)p * nst * tile;
        int s = 0;
        uint32_t ph = 0;
        if ((warp & 1) == 0) {
            for (int i = 0; i < per; ++i) {
                mbar_wait(&empty[p][s], ph ^ 1);
                mbar_arrive_expect_tx(&full[p][s], tile);
                const size_t off = ((size_t)(i * nprod + p) * tile) % WIN;
                bulk1d(ring + (size_t)s * tile, base + off, tile, &full[p][s]);
                if (++s == nst) { s = 0; ph ^= 1; }
            }
        } else {
            for (int i = 0; i < per; ++i) {
                mbar_wait(&full[p][s], ph);
                mbar_arrive(&empty[p][s]);
                if (++s == nst) { s = 0; ph ^= 1; }
            }
            t_end[p] = clock64();
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long mx = 0;
        for (int q = 0; q < nprod; ++q) mx = t_end[q] - t0 > mx ? t_end[q] - t0 : mx;
        out[blockIdx.x] = mx;
    }
}

int main() {
    const int grid = 148;
    uint8_t *g;
    cudaMalloc(&g, (size_t)grid * WIN);
    cudaMemset(g, 1, (size_t)grid * WIN);
    long long *d;
    cudaMalloc(&d, grid * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int share : {0, 1, 2})
    for (int tile : {8192, 16384, 32768, 65536})
        for (int nprod : {1, 2}) {
            if (tile == 65536 && nprod == 2) continue;
            const int nst = std::min(16, (192 * 1024 / nprod) / tile);
            if (nst < 2) continue;
            const int ntiles = 512;
            for (int rep = 0; rep < 2; ++rep) bench<<<grid, 512, 200 * 1024>>>(g, tile, ntiles, nst, nprod, share, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<long long> h(grid);
            cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("share %d tile %5d B, %d producer warp(s) x %2d stages: %6.1f B/clk/SM, %5.0f cyc/op\n", share, tile, nprod, nst,
                   (double)ntiles * tile / mx, (double)mx * nprod / ntiles);
        }
    return 0;
}
