// g2bmm.cuh -- NEXT-4: G2BMM, general-to-band matrix multiplication (iterator mapping table,
// P:1109-1118; LongFormer dilated attention), reading R4:
//     out[b][m][w] = sum_k A[b][m][k] * B[b][m + d*(w - W)][k],   w in [0, 2W]   (0 off the sequence)
//
// Derived form (the paper's dilated -> non-dilated rewrite): rows of residue r (m = r + d*u)
// only meet B rows of the same residue, so a tile is 128 rows u of ONE residue class and the band
// product is dense in u.  On sm_100a the rewrite costs no data movement: TMA loads the class's A
// rows and B rows straight from [b][L][K] with element stride d.  The direct (dilated) form uses
// the same kernel with contiguous rows (stride 1) and band columns d apart (cs = d).
//
// Tile: S[i][j] = A_tile[i] . B(j) for i < 128 and j < 256*nchunks, B(j) = mA0 + stride*j - d*W
// (j = i + cs*w is the band), computed by tcgen05.mma (M=128, N=256, K=64 bf16 / 32 tf32) into two
// 256-column TMEM buffers.  Epilogue (warps 4-7, rows 32q..32q+31): per block of 32 band columns
// w0..w0+31 a warp loads its own TMEM window [32q + cs*w0, +32(cs+1)) (tcgen05.ld addresses are per
// warp), writes each lane's 32 band values into a 32x32 smem tile with a skewed, bank-conflict-free
// store (pitch 32 words, lane stride 31 banks), and writes the tile back as rows of the output
// (coalesced).  HBM-bound (the output is (2W+1)/K times larger than the inputs).
#pragma once
#include "sm100_ptx.cuh"

namespace ollie {

// warps 0 TMA, 1 MMA, 2 TMEM alloc, 4.. epilogue: 12 epilogue warps for the derived form (cs = 1,
// 64-register windows), 8 for the direct form's wider windows
__host__ __device__ constexpr int g2_epi_warps(int cs) { return cs == 1 ? 12 : 8; }
__host__ __device__ constexpr int g2_threads(int cs) { return 128 + 32 * g2_epi_warps(cs); }
// per-warp staging tile: 32 rows x pitch floats (cs = 1: whole 64-column windows, pitch 68 keeps the
// 16-byte row writes conflict-free; otherwise a 32 x 32 band tile)
__host__ __device__ constexpr int g2_stage_pitch(int cs) { return cs == 1 ? 68 : 32; }
constexpr int G2_BN = 128;                 // B rows (S columns) per MMA chunk / TMEM buffer
constexpr int G2_NBUF = 4;                 // TMEM chunk buffers (4 x 128 = 512 columns) = B ring stages

struct G2Args {
    int32_t batch, L, W, d;
    int32_t stride;                        // tile row stride in the sequence: d (derived) or 1 (direct)
    int32_t cs;                            // band column stride in S: 1 (derived) or d (direct)
    int32_t nw;                            // 2W + 1
    int32_t nwb;                           // ceil(nw / 32) band-column blocks
    int32_t nchunks;                       // 256-column MMA chunks per tile
    int32_t rpb;                           // rows per TMA box (rpb * stride <= 256 traversed)
    int32_t tiles_r;                       // tiles per (batch, residue) (derived) or per batch (direct)
    int32_t nres;                          // residue classes per batch: d (derived) or 1
    int32_t num_items;
    int64_t ldo;                           // output row pitch (elements)
    void *out;
    int32_t dbg;                           // debug (0 in production): bit 0 skip stores, bit 1 skip staging
};

template <bool kTF32, int kCS>
__global__ void __launch_bounds__(g2_threads(kCS), 1)
g2bmm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
             const __grid_constant__ G2Args a) {
    constexpr int ES = kTF32 ? 4 : 2;
    constexpr int WIN = 32 * (kCS + 1);    // TMEM window per band block
    constexpr int EPI = g2_epi_warps(kCS);
    constexpr int PERQ = EPI / 4;          // epilogue warps per TMEM lane quadrant
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;                                   // 128 rows x 128 B
    uint8_t *sB = sA + 128 * 128;                         // G2_NBUF stages x G2_BN rows x 128 B
    constexpr int SP = g2_stage_pitch(kCS);
    float *sStage = reinterpret_cast<float *>(sB + G2_NBUF * G2_BN * 128);   // EPI warps x 32 x SP fp32
    uint64_t *bars = reinterpret_cast<uint64_t *>(sStage + EPI * 32 * SP);
    uint64_t *a_full = bars, *a_empty = bars + 1;
    uint64_t *b_full = bars + 2, *b_empty = b_full + G2_NBUF;
    uint64_t *tfull = b_empty + G2_NBUF, *tempty = tfull + G2_NBUF;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + G2_NBUF);

    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    const int lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_a);
        tma_prefetch_desc(&tm_b);
    }
    if (warp == 1 && lane == 0) {
        mbar_init(a_full, 1); mbar_init(a_empty, 1);
        for (int i = 0; i < G2_NBUF; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < G2_NBUF; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], EPI); }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) pdl_launch_dependents();

    // item -> (batch, first row mA0): derived items run over (batch, residue, tile)
    auto item_rows = [&](int item, int &bb, int &mA0) {
        const int t = item % a.tiles_r;
        const int br = item / a.tiles_r;
        const int r = br % a.nres;
        bb = br / a.nres;
        mA0 = r + a.stride * 128 * t;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer: A tile once per item, B band rows in 256-row chunks =====
            pdl_wait();
            uint32_t ap = 0;
            int bs = 0;
            uint32_t bp = 0;
            const int dW = a.d * a.W;
            for (int item = blockIdx.x; item < a.num_items; item += gridDim.x) {
                int bb, mA0;
                item_rows(item, bb, mA0);
                mbar_wait(a_empty, ap ^ 1);
                mbar_arrive_expect_tx(a_full, 128 * 128);
                for (int r0 = 0; r0 < 128; r0 += a.rpb)
                    tma_load_3d(sA + r0 * 128, &tm_a, a_full, 0, mA0 + a.stride * r0, bb);
                ap ^= 1;
                for (int c = 0; c < a.nchunks; ++c) {
                    mbar_wait(&b_empty[bs], bp ^ 1);
                    mbar_arrive_expect_tx(&b_full[bs], G2_BN * 128);
                    for (int r0 = 0; r0 < G2_BN; r0 += a.rpb)
                        tma_load_3d(sB + bs * (G2_BN * 128) + r0 * 128, &tm_b, &b_full[bs], 0,
                                    mA0 + a.stride * (c * G2_BN + r0) - dW, bb);
                    if (++bs == G2_NBUF) { bs = 0; bp ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (converged warp, elected lane issues): S chunk = A_tile . B_chunk^T =====
        const uint32_t idesc = make_idesc(kTF32, 128, G2_BN);
        const uint64_t desc_t = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        const uint64_t adesc = desc_t | (uint64_t)((smem_u32(sA) >> 4) & 0x3FFF);
        const uint32_t sB16 = smem_u32(sB) >> 4;
        uint32_t ap = 0;
        int bs = 0;
        uint32_t bp = 0;
        uint32_t cg = 0;                      // chunks produced by this CTA (TMEM buffer = cg & 1)
        for (int item = blockIdx.x; item < a.num_items; item += gridDim.x) {
            mbar_wait_warp(a_full, ap);
            tc_fence_after();
            for (int c = 0; c < a.nchunks; ++c, ++cg) {
                const uint32_t buf = cg % G2_NBUF;
                mbar_wait_warp(&tempty[buf], ((cg / G2_NBUF) & 1) ^ 1);
                mbar_wait_warp(&b_full[bs], bp);
                tc_fence_after();
                const uint64_t bdesc = desc_t | (uint64_t)((sB16 + (uint32_t)bs * (G2_BN * 128 / 16)) & 0x3FFF);
                const uint32_t d_tmem = tmem_base + buf * G2_BN;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)   // K = 128 bytes: 4 steps of 32 bytes
                    umma_elect<kTF32>(d_tmem, adesc + 2 * ks, bdesc + 2 * ks, idesc, ks > 0 ? 1u : 0u);
                umma_commit_elect(&b_empty[bs]);
                umma_commit_elect(&tfull[buf]);
                __syncwarp();
                if (++bs == G2_NBUF) { bs = 0; bp ^= 1; }
            }
            umma_commit_elect(a_empty);
            __syncwarp();
            ap ^= 1;
        }
    } else if (warp >= 4) {
        // ===== epilogue: band de-skew through a 32x32 smem tile per warp, coalesced row stores.
        // Two warps per TMEM lane quadrant (q = warp % 4) take alternate band blocks. =====
        const int e = warp - 4;
        const int q = warp & 3;
        const int half = e >> 2;                  // which of the quadrant's PERQ warps
        const int R0 = 32 * q;
        float *stg = sStage + e * (32 * SP);
        const uint32_t stg_addr = smem_u32(stg);
        pdl_wait();
        uint32_t cg0 = 0;
        for (int item = blockIdx.x; item < a.num_items; item += gridDim.x) {
            int bb, mA0;
            item_rows(item, bb, mA0);
            int c_ready = -1, c_freed = -1;
            for (int bi = half; bi < a.nwb; bi += PERQ) {
                const int w0 = 32 * bi;
                const int s = R0 + kCS * w0;                       // window start column in S
                const int need = (s + WIN - 1) / G2_BN;
                while (c_ready < need) {
                    ++c_ready;
                    const uint32_t cgc = cg0 + (uint32_t)c_ready;
                    mbar_wait(&tfull[cgc % G2_NBUF], (cgc / G2_NBUF) & 1);
                    tc_fence_after();
                }
                uint32_t v[WIN];
#pragma unroll
                for (int p = 0; p <= kCS; ++p) {
                    const int col = s + 32 * p;
                    const uint32_t cgc = cg0 + (uint32_t)(col / G2_BN);
                    const uint32_t taddr = tmem_base + ((uint32_t)R0 << 16) + (cgc % G2_NBUF) * G2_BN + (uint32_t)(col % G2_BN);
                    tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * p]));
                }
                tmem_ld_wait();
                if constexpr (kCS == 1 && !kTF32) {
                    if ((a.ldo & 7) == 0) {
                        // whole windows into smem (16-byte stores, pitch 68: conflict-free), the skew is
                        // taken on the read side: lane (r, x0) gathers stg[r][r + x0 .. r + x0 + 7]
                        // (bank 5r + x0 + k: all 32 distinct)
                        if (!(a.dbg & 2)) {
#pragma unroll
                            for (int t4 = 0; t4 < 16; ++t4)
                                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                                 stg_addr + (uint32_t)((lane * SP + 4 * t4) * 4)),
                                             "f"(__uint_as_float(v[4 * t4])), "f"(__uint_as_float(v[4 * t4 + 1])),
                                             "f"(__uint_as_float(v[4 * t4 + 2])), "f"(__uint_as_float(v[4 * t4 + 3])));
                        }
                        __syncwarp();
                        const int x = 8 * (lane & 3);
                        float g8[4][8];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int r = 8 * i + (lane >> 2);
#pragma unroll
                            for (int k = 0; k < 8; ++k) g8[i][k] = stg[r * SP + r + x + k];
                        }
                        const int w = w0 + x;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int m = mA0 + a.stride * (R0 + 8 * i + (lane >> 2));
                            if (m >= a.L || w >= a.nw || (a.dbg & 1)) continue;
                            uint16_t *o = reinterpret_cast<uint16_t *>(a.out) + (((int64_t)bb * a.L + m) * a.ldo + w);
                            if (w + 8 <= a.nw) {
                                uint4 pk;
                                pk.x = pack_bf16x2_rn(g8[i][0], g8[i][1]);
                                pk.y = pack_bf16x2_rn(g8[i][2], g8[i][3]);
                                pk.z = pack_bf16x2_rn(g8[i][4], g8[i][5]);
                                pk.w = pack_bf16x2_rn(g8[i][6], g8[i][7]);
                                *reinterpret_cast<uint4 *>(o) = pk;
                            } else {
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    if (w + k < a.nw) o[k] = float_to_bf16_rne(g8[i][k]);
                            }
                        }
                        __syncwarp();
                        goto block_done;
                    }
                }
                // lane l's band value x (w = w0 + x) sits at window column l + kCS*x
                if (!(a.dbg & 2))
#pragma unroll
                for (int t = 0; t < WIN; ++t) {
                    const int e = t - lane;
                    if (e >= 0 && e < 32 * kCS && (kCS == 1 || e % kCS == 0))
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(stg_addr + (uint32_t)((lane * SP + e / kCS) * 4)),
                                     "f"(__uint_as_float(v[t])));
                }
                __syncwarp();
                // rows -> output: pairs of band columns per lane, two rows per instruction (bf16); all
                // smem reads first (independent), then the stores
                if constexpr (kTF32) {
                    float f[32];
#pragma unroll
                    for (int rl = 0; rl < 32; ++rl) f[rl] = stg[rl * SP + lane];
#pragma unroll
                    for (int rl = 0; rl < 32; ++rl) {
                        const int m = mA0 + a.stride * (R0 + rl), w = w0 + lane;
                        if (m < a.L && w < a.nw && !(a.dbg & 1))
                            reinterpret_cast<float *>(a.out)[((int64_t)bb * a.L + m) * a.ldo + w] = f[rl];
                    }
                } else if ((a.ldo & 7) == 0) {
                    // 16-byte aligned rows (ldo % 8 == 0): 8 band columns per lane, 8 rows per instruction
                    const int x = 8 * (lane & 3);
                    float4 f[8];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float *src = &stg[(8 * i + (lane >> 2)) * SP + x];
                        f[2 * i] = *reinterpret_cast<const float4 *>(src);
                        f[2 * i + 1] = *reinterpret_cast<const float4 *>(src + 4);
                    }
                    const int w = w0 + x;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int m = mA0 + a.stride * (R0 + 8 * i + (lane >> 2));
                        if (m >= a.L || w >= a.nw || (a.dbg & 1)) continue;
                        uint16_t *o = reinterpret_cast<uint16_t *>(a.out) + (((int64_t)bb * a.L + m) * a.ldo + w);
                        const float4 lo = f[2 * i], hi = f[2 * i + 1];
                        if (w + 8 <= a.nw) {
                            uint4 pk;
                            pk.x = pack_bf16x2_rn(lo.x, lo.y);
                            pk.y = pack_bf16x2_rn(lo.z, lo.w);
                            pk.z = pack_bf16x2_rn(hi.x, hi.y);
                            pk.w = pack_bf16x2_rn(hi.z, hi.w);
                            *reinterpret_cast<uint4 *>(o) = pk;
                        } else {
                            const float v8[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                if (w + k < a.nw) o[k] = float_to_bf16_rne(v8[k]);
                        }
                    }
                } else {
                    const int x = 2 * (lane & 15);
                    float2 f[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = *reinterpret_cast<const float2 *>(&stg[(2 * i + (lane >> 4)) * SP + x]);
                    const int w = w0 + x;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int m = mA0 + a.stride * (R0 + 2 * i + (lane >> 4));
                        if (m >= a.L || w >= a.nw || (a.dbg & 1)) continue;
                        const int64_t off = ((int64_t)bb * a.L + m) * a.ldo + w;
                        uint16_t *o = reinterpret_cast<uint16_t *>(a.out) + off;
                        if (w + 1 < a.nw) {
                            if ((off & 1) == 0) {
                                *reinterpret_cast<uint32_t *>(o) = pack_bf16x2_rn(f[i].x, f[i].y);
                            } else {
                                o[0] = float_to_bf16_rne(f[i].x);
                                o[1] = float_to_bf16_rne(f[i].y);
                            }
                        } else {
                            o[0] = float_to_bf16_rne(f[i].x);
                        }
                    }
                }
                __syncwarp();
            block_done:
                // chunks below the next window are no longer needed by this warp
                const int fmin = (bi + PERQ < a.nwb) ? (s + 32 * PERQ * kCS) / G2_BN : a.nchunks;
                while (c_freed + 1 < fmin) {
                    ++c_freed;
                    while (c_ready < c_freed) {   // never release a chunk before it was produced
                        ++c_ready;
                        const uint32_t cgc = cg0 + (uint32_t)c_ready;
                        mbar_wait(&tfull[cgc % G2_NBUF], (cgc / G2_NBUF) & 1);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[(cg0 + (uint32_t)c_freed) % G2_NBUF]);
                }
            }
            // warps whose first band block is past nwb (small W: nwb < PERQ) read no window, but the
            // tempty barriers count every epilogue warp: release each remaining chunk once it exists
            while (c_freed + 1 < a.nchunks) {
                ++c_freed;
                while (c_ready < c_freed) {
                    ++c_ready;
                    const uint32_t cgc = cg0 + (uint32_t)c_ready;
                    mbar_wait(&tfull[cgc % G2_NBUF], (cgc / G2_NBUF) & 1);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[(cg0 + (uint32_t)c_freed) % G2_NBUF]);
            }
            cg0 += (uint32_t)a.nchunks;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace ollie
