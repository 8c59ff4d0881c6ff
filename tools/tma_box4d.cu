// tma_box4d.cu -- per-CTA rate of the fused kernel's weight-box loads: a 4-D tensor box
// {64 ch, FS f, 3 j, 3 i} of W' viewed as {c, f, j, i} (128-byte rows at a C*2-byte stride, SWIZZLE_128B)
// against a 1-D bulk copy of the same byte count, 128 CTAs, 32 of them reading the same boxes (4 f-slices),
// a 2-deep ring, the consumer releasing a stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_box4d tools/tma_box4d.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__device__ __forceinline__ void tma4(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void bulk1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__global__ void __launch_bounds__(64, 1) bench(const __grid_constant__ CUtensorMap tm, const uint8_t *w, int mode, int FS,
                                              int nsteps, int nst, int kch, long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8], empty[8];
    const int box = 9 * FS * 128;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int fslice = blockIdx.x % 4;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < nsteps; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], box);
            const int kc = (i + blockIdx.x / 4) % kch;
            if (mode == 0) tma4(smem + s * box, &tm, &full[s], kc * 64, fslice * FS, 0, 0);
            else bulk1d(smem + s * box, w + ((size_t)(fslice * kch + kc) * box) % (8u << 20), box, &full[s]);
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < nsteps; ++i) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == nst) { s = 0; ph ^= 1; }
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    const int C = 256, F = 256, FS = 64, kch = C / 64;
    void *w;
    cudaMalloc(&w, (size_t)9 * F * C * 2 + (8u << 20));
    cudaMemset(w, 1, (size_t)9 * F * C * 2 + (8u << 20));
    long long *d;
    cudaMalloc(&d, 256 * sizeof(long long));
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)F, 3, 3};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * F, (cuuint64_t)C * 2 * F * 3};
    cuuint32_t boxd[4] = {64, (cuuint32_t)FS, 3, 3};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, w, dims, strides, boxd, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int box = 9 * FS * 128, nsteps = 64;
    for (int mode : {0, 1})
        for (int nst : {1, 2}) {
            for (int rep = 0; rep < 2; ++rep)
                bench<<<128, 64, 200 * 1024>>>(tm, (const uint8_t *)w, mode, FS, nsteps, nst, kch, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<long long> h(128);
            cudaMemcpy(h.data(), d, 128 * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            printf("%s, %d-deep ring: %6.1f B/clk per CTA, %5.0f cycles per %d KB box\n",
                   mode == 0 ? "4-D tensor box {64 ch, 64 f, 3, 3}" : "1-D bulk copy of the same bytes  ", nst,
                   (double)nsteps * box / mx, (double)mx / nsteps, box / 1024);
        }
    return 0;
}
