// tma_bench.cu -- weight-tile streaming rate on B200: every CTA streams `ntiles` B tiles
// (box {64 bf16 = 128 B, FS rows, 1} of a 3-D {c, f, tap} tensor, SWIZZLE_128B) through an
// nst-deep smem ring (consumer releases immediately).  Variants:
//   share 0: every CTA reads the same tiles in the same order        (hot lines)
//   share 1: same tiles, per-CTA rotated order
//   share 2: each CTA reads its own copy of the weights              (no sharing)
//   mc = 2/4: clusters of mc CTAs; each CTA loads FS/mc rows and multicasts to the cluster
// Prints bytes delivered per SM per cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma3_mc(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                        uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
            smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void bulk1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 1-D bulk copies of `tile` contiguous bytes (pre-laid weight tiles), same ring protocol
__global__ void __launch_bounds__(64, 1) bench_bulk(const uint8_t *w, int tile, int ntiles_total, int ntiles, int nst,
                                                   int share, int copies, int pieces, long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[32], empty[32];
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int rot = share == 1 ? (blockIdx.x * 7) % ntiles_total : 0;
    const uint8_t *base = w + (size_t)(share == 2 ? blockIdx.x % copies : 0) * ntiles_total * tile;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < ntiles; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], tile);
            const int q = (i + rot) % ntiles_total;
            const int pc = tile / pieces;
            for (int p = 0; p < pieces; ++p)
                bulk1d(smem + s * tile + p * pc, base + (size_t)q * tile + p * pc, pc, &full[s]);
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < ntiles; ++i) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == nst) { s = 0; ph ^= 1; }
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

__global__ void __launch_bounds__(64, 1) bench(const __grid_constant__ CUtensorMap tm, int FS, int C, int taps,
                                              int ntiles, int nst, int share, int mc, int copies, long long *out,
                                              int tpo) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[32], empty[32];
    const int stage = FS * 128 * tpo;
    const uint32_t rank = mc > 1 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], mc > 1 ? mc : 1); }
        fence_barrier_init();
    }
    if (mc > 1) cluster_sync(); else __syncthreads();
    const int kch = C / 64;
    const int total = kch * (taps / tpo);
    const int cid = mc > 1 ? blockIdx.x / mc : blockIdx.x;
    const int rot = share == 1 ? (cid * 7) % total : 0;
    const int copy = share == 2 ? cid % copies : 0;
    long long t0 = clock64();
    if (threadIdx.x == 0) {            // producer
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < ntiles; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], stage);
            const int q = (i + rot) % total;
            const int kc = q / (taps / tpo), t = (q % (taps / tpo)) * tpo;
            if (mc > 1) {
                const int rows = FS / mc;
                tma3_mc(smem + s * stage + rank * rows * 128, &tm, &full[s], kc * 64, copy * FS + rank * rows, t,
                        (uint16_t)((1 << mc) - 1));
            } else {
                tma3(smem + s * stage, &tm, &full[s], kc * 64, copy * FS, t);
            }
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {    // consumer: release as soon as the tile landed
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < ntiles; ++i) {
            mbar_wait(&full[s], ph);
            if (mc > 1) {
                for (uint32_t r = 0; r < (uint32_t)mc; ++r) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), r));
            } else {
                mbar_arrive(&empty[s]);
            }
            if (++s == nst) { s = 0; ph ^= 1; }
        }
        out[blockIdx.x] = clock64() - t0;
    }
    if (mc > 1) {
        // drain: wait until the last releases from peers landed before leaving
        if (threadIdx.x == 0) {
            int s = ntiles % nst; uint32_t ph = (ntiles / nst) & 1;
            for (int i = 0; i < nst; ++i) { mbar_wait(&empty[s], ph ^ 1); if (++s == nst) { s = 0; ph ^= 1; } }
        }
        cluster_sync();
    }
}

int main() {
    const int C = 256, taps = 9, FS = 64;
    const int copies = 148;
    // W' as [copies * FS... ] : dims {c, f_total, taps}, f_total = copies * FS (share 2 uses its own rows)
    const size_t ftot = (size_t)copies * FS;
    void *w;
    cudaMalloc(&w, (size_t)C * ftot * taps * 2);
    cudaMemset(w, 0, (size_t)C * ftot * taps * 2);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)ftot, (cuuint64_t)taps};
    cuuint64_t strides[2] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * ftot};
    long long *d;
    cudaMalloc(&d, 4096 * sizeof(long long));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    {
        cudaFuncSetAttribute(bench_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int grid = 128, ntiles = 36 * 8, ntot = 36;
        for (int ctas : {1, 2, 4})
        for (int tile : {8192, 32768}) {
                    const int nst = std::min(8, (200 / ctas - 8) * 1024 / tile);
                    if (nst < 2) continue;
                    const int smem = nst * tile + 2048;
                    const int g = 148 * ctas;
                    bench_bulk<<<g, 64, smem>>>((const uint8_t *)w, tile, ntot, ntiles, nst, 0, 8, 1, d);
                    bench_bulk<<<g, 64, smem>>>((const uint8_t *)w, tile, ntot, ntiles, nst, 0, 8, 1, d);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                    std::vector<long long> h(g);
                    cudaMemcpy(h.data(), d, g * sizeof(long long), cudaMemcpyDeviceToHost);
                    long long mx = 0;
                    for (int i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
                    printf("bulk ctas/SM=%d tile=%5d nst=%2d : %6.1f B/clk/SM (all CTAs of the SM)\n", ctas, tile, nst,
                           (double)ntiles * tile * ctas / mx);
        }
    }
    for (int tpo : {1, 3, 9}) {
        const int rows = FS;
        cuuint32_t box[3] = {64, (cuuint32_t)rows, (cuuint32_t)tpo};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, dims, strides, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        const int stage = FS * 128 * tpo;
        const int nst = std::min(16, 190 * 1024 / stage);
        const int grid = 128, nops = 36 * 8 / tpo;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = nullptr; cfg.numAttrs = 0;
        for (int rep = 0; rep < 2; ++rep)
            cudaLaunchKernelEx(&cfg, bench, tm, FS, C, taps, nops, nst, 0, 1, copies, d, tpo);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("tensor box {64, %d, %d} = %6d B/op nst=%2d : %6.1f B/clk/SM, %5.0f cyc/op\n", FS, tpo, stage, nst,
               (double)nops * stage / mx, (double)mx / nops);
    }
    return 0;
}
