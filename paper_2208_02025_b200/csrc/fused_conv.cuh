// fused_conv.cuh -- a8: the merged GEMM with the OffsetAdd fused in, T never materialised.
//
// Derivation: OffsetAdd o Matmul (E7 o E6, P:1049-1051,
// P:1342-1352) is fused by the chain rule (expression fusion) and the inner
// scope is then removed by traversal merging with
// Phi(m, (i,j)) = (m + Delta_ij, (i,j,f)):
//     Y[m, f] = Sum_{i,j} T[m + Delta_ij, (i,j,f)] = Sum_{i,j} Sum_c X[m + Delta_ij, c] W'[(i,j,f), c]
// i.e. each (i,j) column block of the merged GEMM is accumulated straight into the output
// accumulator at its OffsetAdd offset.  On sm_100a the offset Delta_ij becomes a row
// offset into a haloed input patch held in shared memory in the K-major "interleaved"
// (no-swizzle) UMMA layout, where rows are 16 bytes apart, so ONE TMA load of the patch
// per channel chunk feeds all r*s taps: tap (i,j) is the same smem tile read from row
// i*dil*Xb + j*dil.  Zero padding is TMA out-of-bounds fill.
//
// Tile: 128 TMEM lanes = output pixels (y, x) of a Yb x XB block, lane = y*Xb + x where
// Xb = XB + (S-1)*dil is the patch width; N = FS output channels (<= 256); the fp32
// accumulator lives in TMEM (two buffers), the epilogue converts and stores Y directly.
// Persistent, warp-specialised (TMA producer / single-thread MMA issuer / TMEM allocator /
// 4 epilogue warps), stride 1 only.
#pragma once
#include "../../include/ollie.h"
#include "sm100_ptx.cuh"

namespace ollie {

constexpr int FC_THREADS = 256;
constexpr uint32_t FC_TMEM_COLS = 512;
constexpr int FC_SMEM_BUDGET = 225 * 1024;

struct FusedArgs {
    int32_t n, H, W, C, F, R, S, pad, dil;
    int32_t OH, OW;
    int32_t XB, Yb, Xb, Yp;        // output cols / rows per tile, patch width / rows
    int32_t tiles_x, tiles_y, f_slices, FS, num_tiles;
    int32_t kchunks, BK;           // channel chunks of BK elements
    int32_t a_box_bytes;           // bytes TMA writes per patch load
    int32_t a_stage_bytes;         // patch stage stride in smem (box + slack, 1024-aligned)
    int32_t lbo;                   // planar chunk stride (bytes) = Yp*Xb*16
    int32_t b_stage_bytes;         // FS * 128
    int32_t na, nb;                // ring depths
    void *y;
};

// K-major, no-swizzle ("interleaved") UMMA smem descriptor: core matrices of 8 rows x 16 B,
// rows 16 B apart (SBO = 128 B between 8-row groups), K-chunks of 16 B `lbo` bytes apart.
__device__ __forceinline__ uint64_t make_sdesc_k_interleave(uint32_t smem_addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(128 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;  // layout type 0 = SWIZZLE_NONE
}

__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *m, uint64_t *bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int32_t c0, int32_t c1,
                                            int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

struct TileCoord {
    int img, y0, x0, f0;
};
__device__ __forceinline__ TileCoord fc_tile(const FusedArgs &a, int tile) {
    TileCoord t;
    const int fs = tile % a.f_slices;
    int q = tile / a.f_slices;
    const int tx = q % a.tiles_x;
    q /= a.tiles_x;
    const int ty = q % a.tiles_y;
    t.img = q / a.tiles_y;
    t.y0 = ty * a.Yb;
    t.x0 = tx * a.XB;
    t.f0 = fs * a.FS;
    return t;
}

template <bool kTF32>
__global__ void __launch_bounds__(FC_THREADS, 1)
fused_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, FusedArgs a) {
    constexpr int ES = kTF32 ? 4 : 2;
    constexpr int CI = 16 / ES;                  // elements per 16-byte planar chunk
    constexpr int KI = 32 / ES;                  // K per tcgen05.mma (16 bf16 / 8 tf32)

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = sA + a.na * a.a_stage_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + a.nb * a.b_stage_bytes);
    uint64_t *a_full = bars;
    uint64_t *a_empty = a_full + a.na;
    uint64_t *b_full = a_empty + a.na;
    uint64_t *b_empty = b_full + a.nb;
    uint64_t *tfull = b_empty + a.nb;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    const int taps = a.R * a.S;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < a.na; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
        for (int i = 0; i < a.nb; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<FC_TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer: per tile, per channel chunk: 1 patch + r*s weight tiles =====
            int as = 0, bs = 0;
            uint32_t ap = 0, bp = 0;
            for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
                const TileCoord tc = fc_tile(a, tile);
                for (int kc = 0; kc < a.kchunks; ++kc) {
                    mbar_wait(&a_empty[as], ap ^ 1);
                    mbar_arrive_expect_tx(&a_full[as], (uint32_t)a.a_box_bytes);
                    tma_load_5d(sA + as * a.a_stage_bytes, &tmX, &a_full[as], 0, tc.x0 - a.pad, tc.y0 - a.pad, tc.img,
                                kc * (a.BK / CI));
                    if (++as == a.na) { as = 0; ap ^= 1; }
                    for (int t = 0; t < taps; ++t) {
                        mbar_wait(&b_empty[bs], bp ^ 1);
                        mbar_arrive_expect_tx(&b_full[bs], (uint32_t)a.b_stage_bytes);
                        tma_load_3d(sB + bs * a.b_stage_bytes, &tmW, &b_full[bs], kc * (128 / ES), tc.f0, t);
                        if (++bs == a.nb) { bs = 0; bp ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer: D[lane, f] += Patch[lane + off(i,j), c] * W'[(i,j), f, c] =====
            const uint32_t idesc = make_idesc(kTF32, 128, (uint32_t)a.FS);
            int as = 0, bs = 0;
            uint32_t ap = 0, bp = 0;
            int acc = 0;
            uint32_t accp = 0;
            for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
                mbar_wait(&tempty[acc], accp ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 256);
                for (int kc = 0; kc < a.kchunks; ++kc) {
                    const int kvalid = min(a.BK, a.C - kc * a.BK);
                    const int ksteps = (kvalid + KI - 1) / KI;
                    mbar_wait(&a_full[as], ap);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + as * a.a_stage_bytes);
                    for (int t = 0; t < taps; ++t) {
                        const int i = t / a.S, j = t - i * a.S;
                        const uint32_t off = (uint32_t)((i * a.Xb + j) * a.dil) * 16u;
                        mbar_wait(&b_full[bs], bp);
                        tc_fence_after();
                        const uint32_t b_base = smem_u32(sB + bs * a.b_stage_bytes);
                        for (int k = 0; k < ksteps; ++k) {
                            umma<kTF32>(d_tmem, make_sdesc_k_interleave(a_base + (uint32_t)(2 * k) * a.lbo + off, a.lbo),
                                        make_sdesc_k_sw128(b_base + k * 32), idesc, (kc | t | k) != 0);
                        }
                        umma_commit(&b_empty[bs]);
                        if (++bs == a.nb) { bs = 0; bp ^= 1; }
                    }
                    umma_commit(&a_empty[as]);
                    if (++as == a.na) { as = 0; ap ^= 1; }
                }
                umma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) accp ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> Y (bf16 RNE or fp32), one output pixel per thread =====
        const int q = warp - 4;
        const int L = q * 32 + lane;
        const int ly = L / a.Xb, lx = L - (L / a.Xb) * a.Xb;
        int acc = 0;
        uint32_t accp = 0;
        const bool vec = (a.F % (kTF32 ? 4 : 8)) == 0;
        for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
            const TileCoord tc = fc_tile(a, tile);
            mbar_wait(&tfull[acc], accp);
            tc_fence_after();
            const int oy = tc.y0 + ly, ox = tc.x0 + lx;
            const bool valid = ly < a.Yb && lx < a.XB && oy < a.OH && ox < a.OW;
            const int64_t pix = ((int64_t)tc.img * a.OH + oy) * a.OW + ox;
            for (int c = 0; c < a.FS; c += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256 + c), v);
                tmem_ld_wait();
                const int f = tc.f0 + c;
                if (valid && f < a.F) {
                    const int nf = min(min(32, a.FS - c), a.F - f);
                    if constexpr (kTF32) {
                        float *yp = reinterpret_cast<float *>(a.y) + pix * a.F + f;
                        if (vec && nf == 32) {
#pragma unroll
                            for (int e = 0; e < 32; e += 4)
                                *reinterpret_cast<float4 *>(yp + e) =
                                    make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                                __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e < nf) yp[e] = __uint_as_float(v[e]);
                        }
                    } else {
                        uint16_t *yp = reinterpret_cast<uint16_t *>(a.y) + pix * a.F + f;
                        if (vec && nf == 32) {
#pragma unroll
                            for (int e = 0; e < 32; e += 8) {
                                uint4 pk;
                                pk.x = (uint32_t)float_to_bf16_rne(__uint_as_float(v[e])) |
                                       ((uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 1])) << 16);
                                pk.y = (uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 2])) |
                                       ((uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 3])) << 16);
                                pk.z = (uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 4])) |
                                       ((uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 5])) << 16);
                                pk.w = (uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 6])) |
                                       ((uint32_t)float_to_bf16_rne(__uint_as_float(v[e + 7])) << 16);
                                *reinterpret_cast<uint4 *>(yp + e) = pk;
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e < nf) yp[e] = float_to_bf16_rne(__uint_as_float(v[e]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) accp ^= 1;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<FC_TMEM_COLS>(tmem_base);
    }
}

}  // namespace ollie
