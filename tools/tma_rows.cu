// tma_rows.cu -- TMA streaming rate of image-row boxes (the row-streaming conv's loads) on B200.
// Every CTA streams its own contiguous run of rows of an NHWC bf16 tensor [rows][W][C] from HBM
// through an nst-deep smem ring (the consumer releases a slot as soon as it lands).  Prints the
// aggregate GB/s for box shapes {C_box, wbox, hbox} with C's swizzle, vs nst.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_rows tools/tma_rows.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2208_02025_b200/csrc/sm100_ptx.cuh"

using namespace ollie;

__global__ void __launch_bounds__(384, 1) stream_rows(const __grid_constant__ CUtensorMap tm, int rows_total, int W,
                                                    int wbox, int hbox, int nst, int box_bytes, long long *cyc, int park) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[32];
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {      // park = 1: the other threads wait at the final barrier (as in the conv kernels)
    const int r0 = (int)((long long)rows_total * blockIdx.x / gridDim.x);
    const int r1 = (int)((long long)rows_total * (blockIdx.x + 1) / gridDim.x);
    const int nb = W / wbox;
    const long long t0 = clock64();
    int issued = 0, done = 0;
    const int nops = ((r1 - r0) / hbox) * nb;
    auto issue = [&](int op) {
        const int s = op % nst;
        const int row = r0 + (op / nb) * hbox, b = op % nb;
        mbar_arrive_expect_tx(&full[s], box_bytes);
        tma_load_4d(smem + (size_t)s * box_bytes, &tm, &full[s], 0, b * wbox, row, 0);
    };
    for (; issued < nst && issued < nops; ++issued) issue(issued);
    for (; done < nops; ++done) {
        mbar_wait(&full[done % nst], (done / nst) & 1);
        if (issued < nops) issue(issued++);
    }
    cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
}

// producer (warp 0 lane 0) + consumer warp 1 (waits full, arrives empty), as in the row-streaming conv
__global__ void __launch_bounds__(256, 1) stream_rows_pc(const __grid_constant__ CUtensorMap tm, int rows_total, int W,
                                                        int wbox, int hbox, int nst, int box_bytes, long long *cyc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[32], empty[32];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int r0 = (int)((long long)rows_total * blockIdx.x / gridDim.x);
    const int r1 = (int)((long long)rows_total * (blockIdx.x + 1) / gridDim.x);
    const int nb = W / wbox;
    const int nops = ((r1 - r0) / hbox) * nb;
    const long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        for (int op = 0; op < nops; ++op) {
            const int s = op % nst;
            mbar_wait(&empty[s], ((op / nst) & 1) ^ 1);
            const int row = r0 + (op / nb) * hbox, b = op % nb;
            mbar_arrive_expect_tx(&full[s], box_bytes);
            tma_load_4d(smem + (size_t)s * box_bytes, &tm, &full[s], 0, b * wbox, row, 0);
        }
    } else if (warp == 1) {
        for (int op = 0; op < nops; ++op) {
            const int s = op % nst;
            mbar_wait_warp(&full[s], (op / nst) & 1);
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
}

// NPROD producer warps in one CTA (lane 0 of warps 0..NPROD-1), each streaming every NPROD-th op through
// its own share of the ring: is a CTA's TMA rate a per-warp or a per-CTA (per-SM) limit?
template <int NPROD>
__global__ void __launch_bounds__(128, 1) stream_rows_mp(const __grid_constant__ CUtensorMap tm, int rows_total, int W,
                                                        int wbox, int nst, int box_bytes, long long *cyc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[64];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NPROD * nst; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int r0 = (int)((long long)rows_total * blockIdx.x / gridDim.x);
    const int r1 = (int)((long long)rows_total * (blockIdx.x + 1) / gridDim.x);
    const int nb = W / wbox;
    const int nops = (r1 - r0) * nb;
    if (warp < NPROD && lane == 0) {
        uint64_t *fb = full + warp * nst;
        uint8_t *sm = smem + (size_t)warp * nst * box_bytes;
        int issued = 0, done = 0, mine = 0;
        for (int op = warp; op < nops; op += NPROD) ++mine;
        auto issue = [&](int j) {      // j-th op of this warp
            const int op = warp + j * NPROD, s = j % nst;
            const int row = r0 + op / nb, b = op % nb;
            mbar_arrive_expect_tx(&fb[s], box_bytes);
            tma_load_4d(sm + (size_t)s * box_bytes, &tm, &fb[s], 0, b * wbox, row, 0);
        };
        for (; issued < nst && issued < mine; ++issued) issue(issued);
        for (; done < mine; ++done) {
            mbar_wait(&fb[done % nst], (done / nst) & 1);
            if (issued < mine) issue(issued++);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = 0;
}

int main() {
    const int W = 256, H = 16384;   // 16384 rows of 256 pixels (FSRCNN: 64 images x 256 rows)
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(stream_rows_pc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    long long *cyc;
    cudaMalloc(&cyc, sizeof(long long) * 1024);
    struct Cfg { int C, cbox, wbox, hbox; };
    const Cfg cfgs[] = {{16, 16, 256, 1}};
    for (const Cfg &c : cfgs) {
        const size_t bytes = (size_t)H * W * c.C * 2;
        void *x;
        cudaMalloc(&x, bytes);
        {   // random bits: zero pages would be compressed by the L2 and overstate the streaming rate
            std::vector<uint16_t> hbuf(bytes / 2);
            uint32_t st = 12345u;
            for (auto &v : hbuf) { st = st * 1664525u + 1013904223u; v = (uint16_t)((st >> 16) & 0x3FFF) | 0x3000; }
            cudaMemcpy(x, hbuf.data(), bytes, cudaMemcpyHostToDevice);
        }
        CUtensorMap tm;
        cuuint64_t dims[4] = {(cuuint64_t)c.C, (cuuint64_t)W, (cuuint64_t)H, 1};
        cuuint64_t strides[3] = {(cuuint64_t)c.C * 2, (cuuint64_t)W * c.C * 2, (cuuint64_t)H * W * c.C * 2};
        cuuint32_t box[4] = {(cuuint32_t)c.cbox, (cuuint32_t)c.wbox, (cuuint32_t)c.hbox, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        const int rb = c.cbox * 2;
        const CUtensorMapSwizzle sw = rb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        for (int promo = 1; promo < 2; ++promo) {
            CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                                promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
            const int box_bytes = c.cbox * 2 * c.wbox * c.hbox;
            for (int park = 0; park < 2; ++park)
            for (int nst : {2, 4, 8, 16}) {
                if ((size_t)nst * box_bytes > 210 * 1024) continue;
                if (park) stream_rows_pc<<<sms, 256, nst * box_bytes + 1024>>>(tm, H, W, c.wbox, c.hbox, nst, box_bytes, cyc);
                else stream_rows<<<sms, 32, nst * box_bytes + 1024>>>(tm, H, W, c.wbox, c.hbox, nst, box_bytes, cyc, park);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                for (int it = 0; it < 3; ++it)
                    if (park) stream_rows_pc<<<sms, 256, nst * box_bytes + 1024>>>(tm, H, W, c.wbox, c.hbox, nst, box_bytes, cyc);
                    else stream_rows<<<sms, 32, nst * box_bytes + 1024>>>(tm, H, W, c.wbox, c.hbox, nst, box_bytes, cyc, park);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double moved = (double)H * W * c.cbox * 2;     // box bytes incl. OOB fill
                const double real = (double)bytes;
                printf("park=%d C=%2d box{%2d,%3d,%d} %5d B/op promo=%d nst=%2d: %7.1f us  %6.0f GB/s (HBM bytes)  %6.0f GB/s (box bytes)  err=%s\n",
                       park, c.C, c.cbox, c.wbox, c.hbox, box_bytes, promo, nst, ms * 1e3 / 3, real / (ms * 1e-3 / 3) / 1e9,
                       moved / (ms * 1e-3 / 3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(x);
    }
    {   // multi-producer test: C=16 box {16,256,1} (8 KB) and C=64 box {64,128,1} (16 KB)
        for (int C : {16, 64}) {
            const int W = 256, H = 16384, wbox = C == 16 ? 256 : 128;
            const size_t bytes = (size_t)H * W * C * 2;
            void *x; cudaMalloc(&x, bytes); cudaMemset(x, 1, bytes);
            CUtensorMap tm;
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, 1};
            cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
            cuuint32_t box[4] = {(cuuint32_t)C, (cuuint32_t)wbox, 1, 1};
            cuuint32_t estr[4] = {1, 1, 1, 1};
            cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   C == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int box_bytes = C * 2 * wbox;
            for (int np : {1, 2, 4}) {
                const int nst = 4;
                const size_t sm = (size_t)np * nst * box_bytes + 1024;
                auto run = [&]() {
                    if (np == 1) stream_rows_mp<1><<<sms, 128, sm>>>(tm, H, W, wbox, nst, box_bytes, cyc);
                    if (np == 2) stream_rows_mp<2><<<sms, 128, sm>>>(tm, H, W, wbox, nst, box_bytes, cyc);
                    if (np == 4) stream_rows_mp<4><<<sms, 128, sm>>>(tm, H, W, wbox, nst, box_bytes, cyc);
                };
                cudaFuncSetAttribute(stream_rows_mp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                cudaFuncSetAttribute(stream_rows_mp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                cudaFuncSetAttribute(stream_rows_mp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                run();
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                for (int it = 0; it < 3; ++it) run();
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                printf("multi-producer C=%d box %d B: %d producer warps x %d stages: %7.1f us  %6.0f GB/s  err=%s\n", C, box_bytes, np, nst,
                       ms * 1e3 / 3, bytes / (ms * 1e-3 / 3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
            cudaFree(x);
        }
    }
    return 0;
}
