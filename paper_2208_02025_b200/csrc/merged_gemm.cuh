// merged_gemm.cuh -- step a2 of the hot path: the merged Matmul of Ollie's derived
// convolution ("merges these matrix multiplications into a single one";
// operator matching t1,t2 -> m; r,s,f -> n; c -> k):
//
//     T[m][n] = sum_k A[m][k] * B[n][k]      A = X as [n*h*w, c] (layout-A is the identity on
//                                            NHWC), B = W' [(i*S+j)*F+f][c]
//
// sm_100a design: persistent, warp-specialised, one CTA per SM.
//   warp 0     TMA producer: A / B tiles (K-major, SWIZZLE_128B) into a STAGES-deep smem ring
//   warp 1     MMA issuer:   one thread issues tcgen05.mma (128 x BN x 16|8) into TMEM
//   warp 2     TMEM allocator (512 columns = two BN<=256 fp32 accumulators, double-buffered)
//   warps 4-7  epilogue:     tcgen05.ld -> registers -> 16-byte row stores (one row per thread)
// BN (the UMMA N) is a runtime parameter (multiple of 16, <= 256) chosen on the host to
// minimise N-tail waste.  M / N / K tails are handled by TMA zero fill and store guards.
#pragma once
#include "sm100_ptx.cuh"
#include "epilogue.cuh"

namespace ollie {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK_BYTES = 128;           // one SWIZZLE_128B row per operand row per stage
constexpr int GEMM_STAGES = 4;
constexpr int GEMM_MAX_BN = 256;
constexpr int GEMM_A_STAGE_BYTES = GEMM_BM * GEMM_BK_BYTES;          // 16 KB
constexpr int GEMM_B_STAGE_BYTES = GEMM_MAX_BN * GEMM_BK_BYTES;      // 32 KB (max)
constexpr int GEMM_STG_BYTES = 2 * 32 * 128;                         // per epilogue warp: 2 x (32 rows x 128 B)
constexpr int GEMM_THREADS = 256;
constexpr uint32_t GEMM_TMEM_COLS = 512;

constexpr size_t gemm_smem_bytes() {
    return 1024 /* alignment slack */ + (size_t)GEMM_STAGES * (GEMM_A_STAGE_BYTES + GEMM_B_STAGE_BYTES) +
           4 * GEMM_STG_BYTES + 256 /* barriers */;
}

// GEMM_RED plan: the epilogue performs the OffsetAdd (Conv2d) / selective addition (ConvT) itself
// as fp32 reductions into L2 -- T[m, (i,j,f)] is added to acc[output pixel of (m, i, j), f] with
// red.global.add.v4.f32 -- so T never reaches HBM ("the L2 reduction").
struct RedArgs {
    float *acc;          // [n][OH][OW][F] fp32, zeroed before the GEMM
    int32_t H, W, F, S, pad, stride, dil, OH, OW, transposed;
};

struct GemmArgs {
    int64_t M, N, K;
    int32_t BN;          // UMMA N of a tile
    void *out;           // fp32 or bf16, row-major with leading dimension ldo
    int64_t ldo;
    int32_t tma_out;     // 1: fp32 output tiles leave through smem staging + TMA stores (tmO)
    EpiArgs epi;         // element-wise epilogue (identity plan only: out is Y, column = channel)
    RedArgs red;         // GEMM_RED plan (kRed kernels only)
};

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <bool kTF32, bool kOutBF16, bool kRed = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
merged_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, GemmArgs args) {
    constexpr int ES = kTF32 ? 4 : 2;
    constexpr int BK = GEMM_BK_BYTES / ES;       // 64 bf16 / 32 tf32 elements
    constexpr int UMMA_K_BYTES = 32;             // 16 bf16 / 8 tf32 per tcgen05.mma
    constexpr int KSTEPS = GEMM_BK_BYTES / UMMA_K_BYTES;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = sA + GEMM_STAGES * GEMM_A_STAGE_BYTES;
    uint8_t *stg = sB + GEMM_STAGES * GEMM_B_STAGE_BYTES;         // 1024-aligned (SWIZZLE_128B staging)
    uint64_t *bars = reinterpret_cast<uint64_t *>(stg + 4 * GEMM_STG_BYTES);
    uint64_t *full = bars;                       // [STAGES]
    uint64_t *empty = bars + GEMM_STAGES;        // [STAGES]
    uint64_t *tfull = bars + 2 * GEMM_STAGES;    // [2]
    uint64_t *tempty = tfull + 2;                // [2]
    uint32_t *tmem_base_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    const int64_t M = args.M, N = args.N, K = args.K;
    const int BN = args.BN;
    const int num_m = (int)((M + GEMM_BM - 1) / GEMM_BM);
    const int num_n = (int)((N + BN - 1) / BN);
    const int num_tiles = num_m * num_n;
    const int num_k = (int)((K + BK - 1) / BK);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < GEMM_STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<GEMM_TMEM_COLS>(tmem_base_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;
    if (threadIdx.x == 0) pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            const uint32_t stage_bytes = GEMM_A_STAGE_BYTES + (uint32_t)BN * GEMM_BK_BYTES;
            int stage = 0;
            uint32_t phase = 0;
            if ((int)blockIdx.x < num_tiles) {   // read-only weights: warm L2 before waiting on the producer of A
                const int n_blk0 = blockIdx.x % num_n;
                // (one box: a CTA's TMA operations are serviced one at a time, ~0.3 us each from a cold L2,
                // so more prefetches delay the first A load)
                tma_prefetch_2d(&tmB, 0, n_blk0 * BN);
            }
            pdl_wait();
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m_blk = tile / num_n, n_blk = tile % num_n;
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], stage_bytes);
                    tma_load_2d(sA + stage * GEMM_A_STAGE_BYTES, &tmA, &full[stage], kb * BK, m_blk * GEMM_BM);
                    tma_load_2d(sB + stage * GEMM_B_STAGE_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
                    if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer (single thread) =====
            const uint32_t idesc = make_idesc(kTF32, GEMM_BM, (uint32_t)BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * GEMM_MAX_BN);
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * GEMM_A_STAGE_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * GEMM_B_STAGE_BYTES);
#pragma unroll
                    for (int k = 0; k < KSTEPS; ++k) {
                        umma<kTF32>(d_tmem, make_sdesc_k_sw128(a0 + k * UMMA_K_BYTES),
                                    make_sdesc_k_sw128(b0 + k * UMMA_K_BYTES), idesc, (kb | k) != 0);
                    }
                    umma_commit(&empty[stage]);
                    if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
                }
                umma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> global, one output row (pixel) per thread =====
        // Two 32-column TMEM loads in flight per wait; each thread writes its row's contiguous
        // columns with 16-byte stores (hardware bf16x2 packing for bf16 output).  Rows of
        // consecutive lanes are adjacent in memory, and each thread fills whole 32-byte sectors.
        const int ew = warp - 4;                 // == warp % 4: TMEM lane quadrant of this warp
        int acc = 0;
        uint32_t acc_phase = 0;
        const bool vec = kOutBF16 ? (args.ldo % 8 == 0) : (args.ldo % 4 == 0);
        pdl_wait();
        if (lane == 0 && !kRed && args.tma_out) tma_prefetch_desc(&tmO);
        uint32_t nst = 0;                        // TMA-store path: staging buffers used (buffer = nst & 1)
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int m_blk = tile / num_n, n_blk = tile % num_n;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if constexpr (!kRed) {
                if (args.tma_out) {
                    // tile -> 32-row x 128-byte SWIZZLE_128B smem blocks (32 fp32 / 64 bf16 columns, the
                    // NEXT-3 epilogue applied first) -> TMA stores: full 128-byte lines (thread-per-row
                    // 16-byte stores wrote half sectors and throttled the LSU)
                    constexpr int CW = kOutBF16 ? 64 : 32;   // output columns per staged 128-byte row
                    const uint32_t tb0 = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * GEMM_MAX_BN);
                    const int ncols = (int)min((int64_t)BN, N - (int64_t)n_blk * BN);
                    const int64_t row = (int64_t)m_blk * GEMM_BM + ew * 32 + lane;
                    for (int c0 = 0; c0 < ncols; c0 += CW) {
                        uint8_t *buf = stg + ew * GEMM_STG_BYTES + (nst & 1) * (32 * 128);
                        if (lane == 0) bulk_wait_read<1>();      // this buffer's previous store has read it
                        __syncwarp();
#pragma unroll
                        for (int h = 0; h < CW; h += 32) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(tb0 + (uint32_t)(c0 + h), v);
                            tmem_ld_wait();
                            if (c0 + h + 32 >= ncols) {          // accumulator drained: the MMA warp may reuse it
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&tempty[acc]);
                            }
                            const int64_t col = (int64_t)n_blk * BN + c0 + h;
                            if (args.epi.on && row < M && col < N)
                                epi_apply_bits<kOutBF16, 32>(args.epi, v, row * args.ldo + col, (int)col,
                                                             (int)min((int64_t)32, N - col));
                            if constexpr (kOutBF16) {
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    uint4 pk;
                                    pk.x = pack_bf16x2_rn(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1]));
                                    pk.y = pack_bf16x2_rn(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                                    pk.z = pack_bf16x2_rn(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                                    pk.w = pack_bf16x2_rn(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                                    const int jj = (h >> 3) + j;
                                    *reinterpret_cast<uint4 *>(buf + lane * 128 + ((jj ^ (lane & 7)) << 4)) = pk;
                                }
                            } else {
#pragma unroll
                                for (int c = 0; c < 8; ++c)
                                    *reinterpret_cast<uint4 *>(buf + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                                        make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                            }
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmO, buf, n_blk * BN + c0, m_blk * GEMM_BM + ew * 32);
                            bulk_commit();
                        }
                        ++nst;
                    }
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                    continue;
                }
            }
            const int64_t row = (int64_t)m_blk * GEMM_BM + ew * 32 + lane;
            const int64_t col_base = (int64_t)n_blk * BN;
            const int64_t col_end = col_base + BN < N ? col_base + BN : N;   // this tile's columns only
            const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * GEMM_MAX_BN);
            for (int c0 = 0; c0 < BN; c0 += 64) {
                if (col_base + c0 >= col_end) break;
                uint32_t v[64];
                tmem_ld_32x32b_x32(tbase + (uint32_t)c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                const bool two = c0 + 32 < BN && col_base + c0 + 32 < col_end;
                if (two) tmem_ld_32x32b_x32(tbase + (uint32_t)(c0 + 32), *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                tmem_ld_wait();
                if (row >= M) continue;
                const int nc = (int)min((int64_t)64, col_end - (col_base + c0));
                if constexpr (kRed) {
                    // column n = tap*F + f of input pixel `row`: add it at the tap's output pixel
                    const RedArgs &rd = args.red;
                    const int HW = rd.H * rd.W;
                    const int img = (int)(row / HW), rem = (int)(row - (int64_t)img * HW);
                    const int ih = rem / rd.W, iw = rem - (rem / rd.W) * rd.W;
                    int n = (int)(col_base + c0);
                    int tap = n / rd.F, f = n - tap * rd.F;
                    float *accb = rd.acc + (int64_t)img * rd.OH * rd.OW * rd.F;
#pragma unroll
                    for (int e = 0; e < 64; e += 4) {
                        if (e < nc) {
                            const int ti = tap / rd.S, tj = tap - (tap / rd.S) * rd.S;
                            int oh, ow;
                            bool ok;
                            if (rd.transposed) {           // selective addition: scatter form
                                oh = ih * rd.stride - rd.pad + ti * rd.dil;
                                ow = iw * rd.stride - rd.pad + tj * rd.dil;
                                ok = true;
                            } else {                       // OffsetAdd: ih = oh*st - pad + i*dil
                                const int a0 = ih + rd.pad - ti * rd.dil, b0 = iw + rd.pad - tj * rd.dil;
                                oh = a0 / rd.stride;
                                ow = b0 / rd.stride;
                                ok = a0 >= 0 && b0 >= 0 && oh * rd.stride == a0 && ow * rd.stride == b0;
                            }
                            if (ok && oh >= 0 && oh < rd.OH && ow >= 0 && ow < rd.OW)
                                red_add_v4(accb + ((int64_t)oh * rd.OW + ow) * rd.F + f, __uint_as_float(v[e]),
                                           __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                            f += 4;
                            if (f >= rd.F) { f -= rd.F; ++tap; }
                        }
                    }
                    continue;
                }
                if (args.epi.on)
                    epi_apply_bits<kOutBF16, 64>(args.epi, v, row * args.ldo + col_base + c0, (int)(col_base + c0), nc);
                if constexpr (kOutBF16) {
                    uint16_t *o = reinterpret_cast<uint16_t *>(args.out) + row * args.ldo + col_base + c0;
                    {
                        const int nv = vec ? (nc & ~7) : 0;      // whole 16-byte groups, then a scalar tail
#pragma unroll
                        for (int e = 0; e < 64; e += 8)
                            if (e < nv) {
                                uint4 pk;
                                pk.x = pack_bf16x2_rn(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
                                pk.y = pack_bf16x2_rn(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                                pk.z = pack_bf16x2_rn(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
                                pk.w = pack_bf16x2_rn(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
                                *reinterpret_cast<uint4 *>(o + e) = pk;
                            }
#pragma unroll
                        for (int e = 0; e < 64; ++e)
                            if (e >= nv && e < nc) o[e] = float_to_bf16_rne(__uint_as_float(v[e]));
                    }
                } else {
                    float *o = reinterpret_cast<float *>(args.out) + row * args.ldo + col_base + c0;
                    {
                        const int nv = vec ? (nc & ~3) : 0;      // whole 16-byte groups, then a scalar tail
#pragma unroll
                        for (int e = 0; e < 64; e += 4)
                            if (e < nv)
                                *reinterpret_cast<float4 *>(o + e) =
                                    make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                                __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
#pragma unroll
                        for (int e = 0; e < 64; ++e)
                            if (e >= nv && e < nc) o[e] = __uint_as_float(v[e]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }

    if (warp >= 4 && lane == 0) bulk_wait<0>();   // TMA stores complete before the CTA (and its smem) retire
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<GEMM_TMEM_COLS>(tmem_base);
    }
}

}  // namespace ollie
