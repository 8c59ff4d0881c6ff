// fused_conv.cuh -- a8: the merged GEMM with the OffsetAdd (Conv2d) or the selective addition
// (ConvTranspose2d) fused in; the intermediate T is never materialised.
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
// per channel chunk feeds every tap: tap (i,j) is the same smem tile read from another row.
// Zero padding is TMA out-of-bounds fill.  When a channel chunk is a full 128 bytes
// the patch is instead loaded as 128-byte pixel rows with SWIZZLE_128B (one TMA row per pixel,
// 8x fewer than 16-byte planar rows); a tap's row shift then starts the descriptor inside a
// 1024-byte swizzle atom, which is consistent because both TMA and the tensor core apply the
// swizzle to absolute shared-memory address bits (base offset 0).
//
// ConvTranspose2d: the selective addition is split by output residue class
// (oh mod st, ow mod st) -- expression splitting, P:927-934 -- and every class is a stride-1
// tap accumulation over the UNPADDED input with the class's tap subset (each output sums
// only the Matmul outputs that land on it, no work on inserted zeros); the epilogue writes
// the class interleaved into NHWC Y (the fused "selective add o interleave DLT" pair of
// SURVEY 8(a) a5).
//
// Tile: 128 TMEM lanes = output pixels (y, x) of a Yb x XB block of one class grid, lane =
// y*Xb + x (Xb = patch width); N = FS output channels (<= 256); MT blocks stacked vertically
// share one patch and every weight tile; fp32 accumulators in TMEM (two buffers when they
// fit), epilogue converts and stores Y directly.  Persistent, warp-specialised: warp 0 TMA
// producer, warp 1 MMA issuer (one elected thread), warp 2 TMEM allocator, warps 4-7 epilogue.
#pragma once
#include "../../include/ollie.h"
#include "sm100_ptx.cuh"
#include "epilogue.cuh"

namespace ollie {

// Debug switches (FusedArgs::dbg, env OLLIE_FC_DBG) exist only in builds with -DOLLIE_FC_DEBUG=1:
// production code is compiled without them.
#ifndef OLLIE_FC_DEBUG
#define OLLIE_FC_DEBUG 0
#endif

constexpr int FC_THREADS = 256;
constexpr uint32_t FC_TMEM_COLS = 512;
constexpr int FC_SMEM_BUDGET = 225 * 1024;
constexpr int FC_MAX_CLASSES = 9;            // table entries: ConvT output classes x strided-conv input phases
constexpr int FC_MAX_TAPS = 32;
constexpr int FC_YSTAGE_BYTES = 128 * 128;   // Y staging: <= 128 output pixels x one 128-byte channel chunk
// split-K receive buffer: (ks - 1) senders x (128 / ks) owned rows x FS fp32 (host sizes it)
__host__ __device__ constexpr int fc_red_bytes(int ks, int FS) { return ks > 1 ? (ks - 1) * (128 / ks) * FS * 4 : 0; }

struct FusedClass {                   // one (output class, input phase) table entry
    int32_t ntaps;
    int32_t oy0, ox0;                 // output residue (ConvT) -- 0 for Conv2d
    int32_t py, px;                   // patch origin: input pixel ist * (tile origin) + (py, px)
    int32_t wi0, wj0;                 // first kernel row / col of the entry's taps (weight box origin)
    int32_t ngroups;                  // weight boxes per step: kernel-row groups of grb rows
    int32_t bres;                     // resident layout: tile offset of the entry's boxes in a channel chunk
    // The entry's taps form a grid (k, l) < (nr, ns): kernel row wi0 + westr*k, col wj0 + westr*l.
    // Tap (k, l) reads patch row a_base + k*a_dk + l*a_dl and weight tile k*nsb + l of the box grid
    // (affine, so the MMA issue loop needs no per-tap table lookups).
    int32_t nr, ns;
    int32_t a_base, a_dk, a_dl;
};

struct FusedArgs {
    int32_t n, H, W, C, F, R, S, pad, dil;
    int32_t OH, OW;
    int32_t ost;                      // output stride: 1 (Conv2d) or st (ConvTranspose2d classes)
    int32_t nclass, max_taps;
    int32_t nph;                      // input phases per class (strided Conv2d: nonempty residues of i*dil-pad mod st)
    int32_t ist;                      // input stride of the patch (TMA element stride): st for Conv2d, 1 for ConvT
    int32_t XB, Yb, Xb, Yp;           // output cols / rows per tile, patch width / rows
    int32_t tma_y;                    // 1: Y tiles leave through a SWIZZLE_128B smem stage + TMA stores
    int32_t ipt, Xr, ngrp;            // images per tile (interleaved patch rows [y][image][x]),
                                      // patch row pitch Xr = ipt * Xb, image groups ceil(n / ipt)
    int32_t grp8;                     // lane layout: 0 = 128 consecutive patch rows (lane = y*Xr + k*Xb + x);
                                      // 1 = 16 groups of 8 lanes, group g = y*ipt + k starting at patch row
                                      // g*Xb (XB <= 8): the A descriptor's 8-row stride SBO = Xb rows, so
                                      // no lane maps to a halo column
    int32_t lane_lp, lane_ip;         // lane decode: ly = L / lane_lp, image (L % lane_lp) / lane_ip, lx = L % lane_ip
    int32_t a_sbo;                    // A descriptor stride between 8-row groups, bytes
    int32_t tiles_x, tiles_y, f_slices, FS, num_tiles;
    int32_t kchunks, BK;              // channel chunks of BK elements
    int32_t a_box_bytes;              // bytes TMA writes per patch load
    int32_t a_stage_bytes;            // patch stage stride in smem (box + slack, 1024-aligned)
    int32_t lbo;                      // planar chunk stride (bytes) = Yp*Xb*16
    int32_t b_tile_bytes;             // one tap's weight tile: FS (pair: FS / 2) rows x 128 B
    int32_t b_stage_bytes;            // one weight box = box_tiles tiles
    int32_t nsb, grb, westr;          // weight box: nsb kernel cols x grb kernel rows, element stride westr
    int32_t box_tiles;                // nsb * grb
    int32_t kc_tiles;                 // resident tiles per channel chunk (all entries' boxes)
    int32_t na, nb;                   // ring depths
    int32_t MT;                       // M-tiles stacked vertically per work item
    int32_t resident;                 // 1: the CTA's whole weight slice stays in smem (loaded once)
    int32_t nbuf;                     // TMEM accumulator sets (2 = epilogue overlaps the next item)
    int32_t acc_cols;                 // TMEM columns per M-tile accumulator (FS rounded up to 32)
    int32_t sw128;                    // 1: patch rows are 128-byte pixel rows, SWIZZLE_128B (BK*es == 128)
    int32_t tmem_cols;                // 512 (1 CTA / SM) or 256 (2 CTAs / SM share the SM's TMEM)
    int32_t pair;                     // 1: CTA pairs (cluster of 2) issue cta_group::2 MMAs with M = 256
    int32_t ksplit;                   // > 1: split-K over a cluster of ksplit CTAs (DSMEM reduction), MT == 1
    int32_t num_items;                // work items: num_tiles (single) or ceil(spatial / 2) * f_slices (pair)
    int32_t spatial;                  // spatial tiles = nclass * n * tiles_y * tiles_x
    void *y;
    EpiArgs epi;                      // NEXT-3 element-wise epilogue (bias / residual / ReLU / PReLU)
    long long *trace;                 // debug only (nullptr in production): per-CTA timestamps
    int32_t dbg;                      // debug only (0 in production): 1 skip MMAs, 2 tap offsets 0, 4 skip Y stores, 8 B tile 0,
                                      // 128 no weight loads, 256 no patch loads
    int32_t split_prod;               // 1: patches issued by warp 0, weight boxes by warp 3
    FusedClass cls[FC_MAX_CLASSES];
};

// Debug timeline: slot k of CTA b at trace[b * 32 + k] = %globaltimer (ns) when the point was
// reached; slot 30 = CTA entry, 31 = CTA exit.  (clock64 deltas proved unreliable for this.)
__device__ __forceinline__ long long fc_gtimer() {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    return (long long)gt;
}
#define FC_TRACE(k)                                                              \
    do {                                                                         \
        if (a.trace) a.trace[blockIdx.x * 32 + (k)] = fc_gtimer();               \
    } while (0)

struct TileCoord {
    int cls, img, y0, x0, f0;   // y0 / x0: first output row / col of the tile in class-grid units
    bool valid;                 // false: the odd CTA of a pair past the last spatial tile (no stores)
};
// tile = (((cls * n + img) * tiles_y + ty) * tiles_x + tx) * f_slices + fs
__device__ __forceinline__ TileCoord fc_tile(const FusedArgs &a, int tile) {
    TileCoord t;
    const int fs = tile % a.f_slices;
    int q = tile / a.f_slices;
    const int tx = q % a.tiles_x;
    q /= a.tiles_x;
    const int ty = q % a.tiles_y;
    q /= a.tiles_y;
    t.img = (q % a.ngrp) * a.ipt;     // first image of the tile's group
    t.cls = q / a.ngrp;
    t.y0 = ty * a.Yb * a.MT;
    t.x0 = tx * a.XB;
    t.f0 = fs * a.FS;
    t.valid = true;
    return t;
}
// Pair mode: item = (cls * ppc + pp) * f_slices + fs; CTA `rank` of the pair takes tile 2 * pp + rank
// of class cls.  Both CTAs share the f-slice (the two halves of B serve both CTAs' MMAs) and the
// class (the leader issues the MMAs with ITS class's tap table for both).
__device__ __forceinline__ TileCoord fc_tile_pair(const FusedArgs &a, int item, int rank) {
    const int fs = item % a.f_slices;
    const int per_cls = a.spatial / a.nclass, ppc = (per_cls + 1) / 2;
    const int q = item / a.f_slices;
    const int cls = q / ppc;
    int s = 2 * (q - cls * ppc) + rank;
    const bool valid = s < per_cls;
    if (!valid) s -= 1;
    TileCoord t = fc_tile(a, (cls * per_cls + s) * a.f_slices + fs);
    t.valid = valid;
    return t;
}
template <bool kPair>
__device__ __forceinline__ TileCoord fc_work(const FusedArgs &a, int item, int rank) {
    if constexpr (kPair) return fc_tile_pair(a, item, rank);
    else return fc_tile(a, item);
}

// Producer-side barrier wait; debug builds with FusedArgs::dbg bit 512 poll with a nanosleep back-off
// instead of spinning in try_wait (ablation: do spinning warps slow the MMA warp?)
__device__ __forceinline__ void fc_pwait(uint64_t *bar, uint32_t parity, int dbg) {
    if (OLLIE_FC_DEBUG && (dbg & 512)) {
        uint32_t ok = 0;
        while (true) {
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
            if (ok) break;
            __nanosleep(200);
        }
    } else {
        mbar_wait(bar, parity);
    }
}

template <bool kTF32, bool kPair, bool kOneEntry, bool kSplit>
__global__ void __launch_bounds__(FC_THREADS, 2)
fused_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmY, const __grid_constant__ FusedArgs a) {
    constexpr int ES = kTF32 ? 4 : 2;
    constexpr int CI = 16 / ES;                  // elements per 16-byte planar chunk
    constexpr int KI = 32 / ES;                  // K per tcgen05.mma (16 bf16 / 8 tf32)

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // B region: nb streamed boxes, or (resident) kchunks x kc_tiles weight tiles loaded once
    const int b_region = a.resident ? a.kchunks * a.kc_tiles * a.b_tile_bytes : a.nb * a.b_stage_bytes;
    uint8_t *sA = smem;
    uint8_t *sB = sA + a.na * a.a_stage_bytes;
    // split-K receive buffer: [sender slot][FS/4 float4 column groups][owned rows]
    float4 *sRed = reinterpret_cast<float4 *>(sB + b_region);
    // Y staging (tma_y plans, never split-K): 1024-aligned since stages and tiles are
    uint8_t *sY = sB + b_region + (kSplit ? fc_red_bytes(a.ksplit, a.FS) : 0);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sY + (a.tma_y ? FC_YSTAGE_BYTES : 0));
    uint64_t *a_full = bars;
    uint64_t *a_empty = a_full + a.na;
    uint64_t *b_full = a_empty + a.na;      // [nb]   (resident: b_full[0] = "all weights loaded")
    uint64_t *b_empty = b_full + a.nb;
    uint64_t *tfull = b_empty + a.nb;
    uint64_t *tempty = tfull + 2;
    uint64_t *recv_full = tempty + 2;       // split-K: every peer pushed its partial of my rows
    uint64_t *peer_done = recv_full + 1;    // split-K: every peer consumed what I pushed to it
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(peer_done + 1);

    // warp index via a lane-0 broadcast: ptxas then knows the role branches are warp-uniform and
    // keeps the MMA issuer on the uniform datapath (plain tid/32 made every issue operand go
    // through R2UR: ~90 instead of ~48 cycles per N=64 MMA)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    const int lane = threadIdx.x & 31;
    // pair mode: cid = the pair's index, rank 0 = the MMA leader; work is strided over pairs
    // split-K: a cluster of ks CTAs shares every item; CTA `krank` takes steps [q_lo, q_lo + q_cnt)
    const int ks = kSplit ? a.ksplit : 1;    // compile-time 1 unless this is the split-K variant
    const int krank = ks > 1 ? (int)cluster_ctarank() : 0;
    const int rank = kPair ? (int)cluster_ctarank() : 0;
    const int cid = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x / ks;
    const int ncl = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x / ks;
    const bool leader = rank == 0;
    const int nq_all = a.kchunks * a.nph;
    const int q_lo = ks > 1 ? krank * nq_all / ks : 0;
    const int q_cnt = ks > 1 ? (krank + 1) * nq_all / ks - q_lo : nq_all;
    const int fhalf = kPair ? a.FS / 2 : 0;        // B rows this CTA loads start at f0 + rank * fhalf
    if (threadIdx.x == 0) FC_TRACE(30);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < a.na; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
        for (int i = 0; i < a.nb; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], kPair ? 8 : 4); }
        if (ks > 1) {   // arrivals per item: one per (peer CTA, thread of the relevant rows), each a release
            mbar_init(recv_full, (ks - 1) * (128 / ks));
            mbar_init(peer_done, (ks - 1) * (128 / ks));
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        if constexpr (kPair) {
            if (a.tmem_cols == 256) tmem_alloc_pair<256>(tmem_slot);
            else tmem_alloc_pair<FC_TMEM_COLS>(tmem_slot);
        } else {
            if (a.tmem_cols == 256) tmem_alloc<256>(tmem_slot);
            else tmem_alloc<FC_TMEM_COLS>(tmem_slot);
        }
    }
    tc_fence_before();
    if (kPair || ks > 1) cluster_sync();   // the peers' barriers exist before any TMA / arrive targets them
    else __syncthreads();
    tc_fence_after();
    // lane-0 broadcast: ptxas then treats the TMEM base as warp-uniform, so the MMA issuer's
    // accumulator address stays in uniform registers (a plain smem load left it in a vector
    // register and cost an R2UR per tcgen05.mma, ~110 cycles each at N <= 64)
    const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    if (threadIdx.x == 0) FC_TRACE(0);
    if (threadIdx.x == 0) pdl_launch_dependents();   // the next layer may start its prologue

    if (warp == 0 || (warp == 3 && a.split_prod)) {
        if (lane == 0) {
            // ===== TMA producer: per work item, per channel chunk: 1 patch + the class's weight tiles =====
            // split_prod: warp 0 issues the patches, warp 3 the weight boxes (a CTA's TMA issues block
            // behind earlier loads in flight; two issuing warps keep both rings fed)
            const bool doA = warp == 0, doB = !a.split_prod || warp == 3;
            int as = 0, bs = 0;
            uint32_t ap = 0, bp = 0;
            // pair mode: both CTAs' loads complete on the LEADER's full barriers, which the leader
            // arms with the bytes of both; each CTA waits on its own empty barriers (the leader's
            // MMA commit multicasts to both)
            const uint32_t xmul = kPair ? 2u : 1u;
            // Weights are read-only for the whole stream (the weight DLT never triggers its dependents
            // early, ollie.h), so their smem loads go out BEFORE griddepcontrol.wait and overlap the
            // previous kernel's tail: the resident slice, or the first step's weight boxes.
            if (doB && a.resident && cid < a.num_items) {
                // the CTA's f-slice is fixed (pair count is a multiple of f_slices): load it once
                const TileCoord tc0 = fc_work<kPair>(a, cid, rank);
                if (leader) mbar_arrive_expect_tx(&b_full[0], xmul * (uint32_t)b_region);
                // one TMA box per (chunk, entry, kernel-row group): few, large copies (a CTA's TMA
                // ops are ~serialised at ~275 cycles each, tools/tma_bench.cu)
                for (int kc = 0; kc < a.kchunks; ++kc)
                    for (int e = 0; e < a.nclass * a.nph; ++e) {
                        const FusedClass &en = a.cls[e];
                        for (int g = 0; g < en.ngroups; ++g) {
                            uint8_t *dst = sB + (kc * a.kc_tiles + en.bres + g * a.box_tiles) * a.b_tile_bytes;
                            const int wi = en.wi0 + g * a.grb * a.westr;
                            if constexpr (kPair)
                                tma_load_4d_pair(dst, &tmW, &b_full[0], kc * (128 / ES), tc0.f0 + rank * fhalf, en.wj0, wi);
                            else
                                tma_load_4d(dst, &tmW, &b_full[0], kc * (128 / ES), tc0.f0, en.wj0, wi);
                        }
                    }
            }
            int pre_b = 0;                   // weight boxes of the first step already issued
            if (doB && !a.resident && cid < a.num_items) {
                const TileCoord tc = fc_work<kPair>(a, cid, rank);
                const int q = ks > 1 ? q_lo : (cid / a.max_taps) % nq_all;
                const int kc = q / a.nph;
                const FusedClass &cl = a.cls[tc.cls * a.nph + (q - kc * a.nph)];
                for (int g = 0; g < cl.ngroups && g < a.nb; ++g) {
                    fc_pwait(&b_empty[bs], bp ^ 1, a.dbg);
                    if (g == 0) FC_TRACE(26);                        // step 0's weights issued (debug trace)
                    if (OLLIE_FC_DEBUG && (a.dbg & 128)) {           // debug: no weight loads (stale smem)
                        mbar_arrive(&b_full[bs]);
                        if (++bs == a.nb) { bs = 0; bp ^= 1; }
                        ++pre_b;
                        continue;
                    }
                    if (leader) mbar_arrive_expect_tx(&b_full[bs], xmul * (uint32_t)a.b_stage_bytes);
                    uint8_t *dstB = sB + bs * a.b_stage_bytes;
                    const int wi = cl.wi0 + g * a.grb * a.westr;
                    if constexpr (kPair)
                        tma_load_4d_pair(dstB, &tmW, &b_full[bs], kc * (128 / ES), tc.f0 + rank * fhalf, cl.wj0, wi);
                    else
                        tma_load_4d(dstB, &tmW, &b_full[bs], kc * (128 / ES), tc.f0, cl.wj0, wi);
                    if (++bs == a.nb) { bs = 0; bp ^= 1; }
                    ++pre_b;
                }
            }
            if (doA) {                       // X may be written by the previous kernel (weights are not)
                pdl_wait();
                FC_TRACE(2);
            }
            for (int item = cid; item < a.num_items; item += ncl) {
                const TileCoord tc = fc_work<kPair>(a, item, rank);
                // steps (kc, ph): channel chunk kc of input phase ph -- one patch, that phase's taps.
                // A per-CTA rotation of the step and tap order spreads identical weight requests in time.
                const int nq = nq_all;
                int q = ks > 1 ? q_lo : (cid / a.max_taps) % nq;
                for (int qi = 0; qi < q_cnt; ++qi) {
                    const int kc = q / a.nph;
                    const FusedClass &cl = a.cls[tc.cls * a.nph + (q - kc * a.nph)];
                    const int xin = a.ist * tc.x0 + cl.px, yin = a.ist * tc.y0 + cl.py;
                    if (doA && OLLIE_FC_DEBUG && (a.dbg & 256)) {   // debug: no patch loads (stale smem)
                        fc_pwait(&a_empty[as], ap ^ 1, a.dbg);
                        mbar_arrive(&a_full[as]);
                        if (++as == a.na) { as = 0; ap ^= 1; }
                    } else if (doA) {
                    fc_pwait(&a_empty[as], ap ^ 1, a.dbg);
                    if (leader) mbar_arrive_expect_tx(&a_full[as], xmul * (uint32_t)a.a_box_bytes);
                    uint8_t *dstA = sA + as * a.a_stage_bytes;
                    if (a.sw128) {
                        if constexpr (kPair) tma_load_4d_pair(dstA, &tmX, &a_full[as], kc * a.BK, xin, tc.img, yin);
                        else tma_load_4d(dstA, &tmX, &a_full[as], kc * a.BK, xin, tc.img, yin);
                    } else {
                        if constexpr (kPair)
                            tma_load_5d_pair(dstA, &tmX, &a_full[as], 0, xin, tc.img, yin, kc * (a.BK / CI));
                        else
                            tma_load_5d(dstA, &tmX, &a_full[as], 0, xin, tc.img, yin, kc * (a.BK / CI));
                    }
                    if (++as == a.na) { as = 0; ap ^= 1; }
                    }
                    if (doB && !a.resident) {
                        for (int g = (item == cid && qi == 0) ? pre_b : 0; g < cl.ngroups; ++g) {
                            fc_pwait(&b_empty[bs], bp ^ 1, a.dbg);
                            if (item == cid && qi == 1 && g == 0) FC_TRACE(27);   // step 1's weights issued (debug trace)
                            if (OLLIE_FC_DEBUG && (a.dbg & 128)) {   // debug: no weight loads (stale smem)
                                mbar_arrive(&b_full[bs]);
                                if (++bs == a.nb) { bs = 0; bp ^= 1; }
                                continue;
                            }
                            if (leader) mbar_arrive_expect_tx(&b_full[bs], xmul * (uint32_t)a.b_stage_bytes);
                            uint8_t *dstB = sB + bs * a.b_stage_bytes;
                            const int wi = cl.wi0 + g * a.grb * a.westr;
                            if constexpr (kPair)
                                tma_load_4d_pair(dstB, &tmW, &b_full[bs], kc * (128 / ES), tc.f0 + rank * fhalf, cl.wj0, wi);
                            else
                                tma_load_4d(dstB, &tmW, &b_full[bs], kc * (128 / ES), tc.f0, cl.wj0, wi);
                            if (++bs == a.nb) { bs = 0; bp ^= 1; }
                        }
                    }
                    if (++q == nq) q = 0;
                }
            }
            if constexpr (kPair) {
                // producer tail: every stage's last release (a multicast commit from the leader)
                // has landed before this CTA may exit
                for (int i = 0; i < (doA ? a.na : 0); ++i) {
                    fc_pwait(&a_empty[as], ap ^ 1, a.dbg);
                    if (++as == a.na) { as = 0; ap ^= 1; }
                }
                if (doB && !a.resident)
                    for (int i = 0; i < a.nb; ++i) {
                        fc_pwait(&b_empty[bs], bp ^ 1, a.dbg);
                        if (++bs == a.nb) { bs = 0; bp ^= 1; }
                    }
            }
        }
    } else if (warp == 1 && leader) {
        // ===== MMA issuer: D[lane, f] += Patch[lane + off(tap), c] * W'[tap, f, c] =====
        // The whole warp walks the schedule (warp-uniform values live in uniform registers); one
        // elected thread issues a whole channel chunk: taps x MT x ksteps tcgen05.mma, with
        // descriptors built as templates + 16-byte-unit address adds.
        const uint32_t idesc = make_idesc(kTF32, kPair ? 256 : 128, (uint32_t)a.FS);
        const bool sw = a.sw128 != 0;
        // A: interleaved (LBO = planar chunk stride, SBO = 128 B) or SWIZZLE_128B (SBO = 1024 B)
        // (grp8 lanes: SBO = Xb patch rows, so group g starts at patch row g*Xb; SWIZZLE_128B still
        // works since the tensor core swizzles absolute smem address bits, as TMA wrote them)
        const uint64_t sbo_f = (uint64_t)(((uint32_t)a.a_sbo >> 4) & 0x3FFF) << 32;
        const uint64_t adesc_t = sw ? (((uint64_t)1 << 16) | sbo_f | ((uint64_t)1 << 46) | ((uint64_t)2 << 61))
                                    : (((uint64_t)((a.lbo >> 4) & 0x3FFF) << 16) | sbo_f | ((uint64_t)1 << 46));
        const uint32_t rowb16 = sw ? 8u : 1u;                           // one patch row, 16-byte units
        const uint64_t bdesc_t = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
                                 ((uint64_t)2 << 61);
        const uint32_t lbo16 = (uint32_t)a.lbo >> 4;
        const uint32_t mstride16 = (uint32_t)(a.Yb * a.Xr) * rowb16;    // stacked M-tiles, 16-byte units
        const uint32_t kstep16 = sw ? 2u : 2u * lbo16;                  // one K=16|8 step, 16-byte units
        const uint32_t sA16 = smem_u32(sA) >> 4, sB16 = smem_u32(sB) >> 4;
        const uint32_t astage16 = (uint32_t)a.a_stage_bytes >> 4, bstage16 = (uint32_t)a.b_stage_bytes >> 4;
        const uint32_t btile16 = (uint32_t)a.b_tile_bytes >> 4;
        const int box_tiles = a.box_tiles, kc_tiles = a.kc_tiles, nsb = a.nsb, grb = a.grb;
        const int MT = a.MT, nb = a.nb, na = a.na, kchunks = a.kchunks, nbuf = a.nbuf, BK = a.BK, C = a.C;
        const uint32_t acc_cols = (uint32_t)a.acc_cols;
        const bool resident = a.resident != 0;
        const int dbg = OLLIE_FC_DEBUG ? a.dbg : 0;
        int as = 0, bs = 0;
        uint32_t ap = 0, bp = 0;
        int acc = 0;
        uint32_t accp = 0;
        if (resident && cid < a.num_items) {
            mbar_wait_warp(&b_full[0], 0);
            tc_fence_after();
        }
        for (int item = cid; item < a.num_items; item += ncl) {
            const TileCoord tc = fc_work<kPair>(a, item, 0);
            mbar_wait_warp(&tempty[acc], accp ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + (uint32_t)acc * (uint32_t)MT * acc_cols;
            const int nph = a.nph, nq = nq_all;
            int q = ks > 1 ? q_lo : (cid / a.max_taps) % nq;
            for (int qi = 0; qi < q_cnt; ++qi) {
                const int kc = q / nph;
                // single-entry layers (stride-1 Conv2d) read entry 0 with a constant index: the
                // table fields then load as uniform constants and the issue loop stays uniform
                const FusedClass &cl = kOneEntry ? a.cls[0] : a.cls[tc.cls * nph + (q - kc * nph)];
                const int kvalid = min(BK, C - kc * BK);
                const int ksteps = (kvalid + KI - 1) / KI;
                mbar_wait_warp(&a_full[as], ap);
                tc_fence_after();
                if (item == cid && qi == 0 && lane == 0) FC_TRACE(1);
                if (item == cid && qi < 6 && lane == 0) FC_TRACE(8 + 3 * qi);     // A landed
                const uint32_t a16 = sA16 + (uint32_t)as * astage16;
                {
                    // the whole (converged) warp walks the tap grid with warp-uniform values; only the
                    // tcgen05.mma / commit instructions are issued by one elected lane.  Taps come in
                    // weight boxes (kernel-row groups): one wait / commit per box.
                    const bool full_k = ksteps == 4;
                    const int nr = cl.nr, ns = cl.ns;
                    const int a_dk = cl.a_dk * (int)rowb16, a_dl = cl.a_dl * (int)rowb16;
                    const uint64_t adesc_s = adesc_t | (uint64_t)((a16 + (uint32_t)cl.a_base * rowb16) & 0x3FFF);
                    for (int g = 0; g < cl.ngroups; ++g) {
                        uint32_t gb16;
                        if (resident) {
                            gb16 = sB16 + (uint32_t)(kc * kc_tiles + cl.bres + g * box_tiles) * btile16;
                        } else {
                            mbar_wait_warp(&b_full[bs], bp);
                            tc_fence_after();
                            if (item == cid && qi < 6 && g == 0 && lane == 0) FC_TRACE(9 + 3 * qi);   // B landed
                            gb16 = sB16 + (uint32_t)bs * bstage16;
                        }
                        const uint64_t bdesc_g = bdesc_t | (uint64_t)(gb16 & 0x3FFF);
                        const int k_lo = g * grb, k_hi = min(k_lo + grb, nr);
                        // One elected thread walks the whole box (a single divergent region per box):
                        // per-MMA elect / reconvergence inside the tap loop cost ~2x in MMA issue rate.
                        if (elect_one()) {
                          if (full_k && ns <= 3 && !(dbg & 32)) {
                            // Kernel rows of <= 3 taps: the (tap, k-step) walk of a row is unrolled (12 MMAs
                            // with distinct descriptor registers).  Rewriting the registers an in-flight
                            // tcgen05.mma still has to read stalls the issue (WAR on its uniform operands):
                            // a rolled 4-MMA loop ran at ~100 cycles per MMA, the unrolled row at the
                            // tensor pipe's own rate.
                            for (int rep = 0; rep < ((dbg & 16) ? 8 : 1); ++rep)
                            for (int m = 0; m < ((dbg & 1) ? 0 : MT); ++m) {
                                const uint32_t dm = d_tmem + (uint32_t)m * acc_cols;
                                const uint64_t atm = adesc_s + (uint64_t)((uint32_t)m * mstride16);
                                for (int k = k_lo; k < k_hi; ++k) {
                                    const uint64_t ak = atm + (uint64_t)(int64_t)(k * a_dk);
                                    const uint64_t bk = bdesc_g + (uint64_t)((uint32_t)((k - k_lo) * nsb) * btile16);
                                    const uint32_t first = (uint32_t)(qi == 0 && k == 0);
#pragma unroll
                                    for (int l = 0; l < 3; ++l) {
                                        if (l < ns) {
                                            const uint64_t al = ak + (uint64_t)(int64_t)(l * a_dl);
                                            const uint64_t bl = bk + (uint64_t)((uint32_t)l * btile16);
#pragma unroll
                                            for (int ks = 0; ks < 4; ++ks) {
                                                const uint32_t accum = (first && l == 0 && ks == 0) ? 0u : 1u;
                                                if constexpr (kPair)
                                                    umma_pair<kTF32>(dm, al + (uint64_t)((uint32_t)ks * kstep16),
                                                                     bl + (uint64_t)(2 * ks), idesc, accum);
                                                else
                                                    umma<kTF32>(dm, al + (uint64_t)((uint32_t)ks * kstep16),
                                                                bl + (uint64_t)(2 * ks), idesc, accum);
                                            }
                                        }
                                    }
                                }
                            }
                          } else
                            for (int rep = 0; rep < ((dbg & 16) ? 8 : 1); ++rep)
                            for (int k = k_lo; k < k_hi; ++k) {
                                for (int l = 0; l < ns; ++l) {
                                    // descriptor address fields are 16-byte units; offsets stay inside the
                                    // 14-bit field (smem < 256 KB), so plain 64-bit adds are exact
                                    const uint64_t bd = bdesc_g + ((dbg & 8) ? 0ull : (uint64_t)((uint32_t)((k - k_lo) * nsb + l) * btile16));
                                    const uint64_t at = adesc_s + ((dbg & 2) ? 0ull : (uint64_t)(int64_t)(k * a_dk + l * a_dl));
                                    const uint32_t first = (uint32_t)(qi == 0 && k == 0 && l == 0);
                                    for (int m = 0; m < ((dbg & 1) ? 0 : MT); ++m) {
                                        // SWIZZLE_128B rows may start anywhere inside a 1024-byte atom: the
                                        // tensor core XORs with absolute smem address bits, exactly as TMA
                                        // wrote them, so the descriptor's base-offset field stays 0
                                        const uint64_t adm = at + (uint64_t)((uint32_t)m * mstride16);
                                        const uint32_t dm = d_tmem + (uint32_t)m * acc_cols;
                                        if (full_k) {
#pragma unroll
                                            for (int ks = 0; ks < 4; ++ks) {
                                                const uint32_t accum = (first && ks == 0) ? 0u : 1u;
                                                if constexpr (kPair)
                                                    umma_pair<kTF32>(dm, adm + (uint64_t)((uint32_t)ks * kstep16),
                                                                     bd + (uint64_t)(2 * ks), idesc, accum);
                                                else
                                                    umma<kTF32>(dm, adm + (uint64_t)((uint32_t)ks * kstep16),
                                                                bd + (uint64_t)(2 * ks), idesc, accum);
                                            }
                                        } else {
                                            for (int ks = 0; ks < ksteps; ++ks) {
                                                const uint32_t accum = (first && ks == 0) ? 0u : 1u;
                                                if constexpr (kPair)
                                                    umma_pair<kTF32>(dm, adm + (uint64_t)((uint32_t)ks * kstep16),
                                                                     bd + (uint64_t)(2 * ks), idesc, accum);
                                                else
                                                    umma<kTF32>(dm, adm + (uint64_t)((uint32_t)ks * kstep16),
                                                                bd + (uint64_t)(2 * ks), idesc, accum);
                                            }
                                        }
                                    }
                                }
                            }
                        }
                        __syncwarp();
                        if (!resident) {
                            if constexpr (kPair) umma_commit_pair_elect(&b_empty[bs], 3);
                            else umma_commit_elect(&b_empty[bs]);
                            if (++bs == nb) { bs = 0; bp ^= 1; }
                        }
                    }
                    if constexpr (kPair) umma_commit_pair_elect(&a_empty[as], 3);
                    else umma_commit_elect(&a_empty[as]);
                }
                __syncwarp();
                if (item == cid && qi < 6 && lane == 0) FC_TRACE(10 + 3 * qi);    // step issued
                if (++as == na) { as = 0; ap ^= 1; }
                if (++q == nq) q = 0;
            }
            if constexpr (kPair) umma_commit_pair_elect(&tfull[acc], 3);
            else umma_commit_elect(&tfull[acc]);
            __syncwarp();
            if (item == cid && lane == 0) FC_TRACE(3);
            if (++acc == nbuf) { acc = 0; accp ^= 1; }
        }
        if (lane == 0) FC_TRACE(4);
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> Y (bf16 RNE or fp32), one output pixel per thread =====
        const int q = warp - 4;
        const int L = q * 32 + lane;
        // lane L = ly * Xr + k * Xb + lx (grp8: ly * 8 * ipt + k * 8 + lx): output row ly, image k of the
        // tile's group, column lx
        const int ly = L / a.lane_lp, lrem = L - ly * a.lane_lp, limg = lrem / a.lane_ip, lx = lrem - limg * a.lane_ip;
        int acc = 0;
        uint32_t accp = 0;
        const bool vec = (a.F % (kTF32 ? 4 : 8)) == 0;
        pdl_wait();   // Y may still be read by the previous kernel: order our stores after it
        // pair mode: the follower's warps release the LEADER's accumulator barrier (count 8)
        const uint32_t tempty_leader0 = kPair ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        uint32_t rc = 0;                         // split-K: reduction chunks processed (buffer = rc & 1)
        for (int item = cid; item < a.num_items; item += ncl) {
            const TileCoord tc = fc_work<kPair>(a, item, rank);
            const FusedClass &cl = a.cls[tc.cls * a.nph];
            if (kSplit) {
                // ===== split-K (push): rows [o*rpc, (o+1)*rpc) of the tile belong to CTA o.  A warp whose
                // rows another CTA owns pushes its fp32 partial into that CTA's receive buffer with
                // fire-and-forget distributed-shared-memory stores; owner warps add the pushed
                // partials to their own and run the normal epilogue.  One arrive per warp per item.
                const int rpc = 128 / ks;
                const int owner = L / rpc;
                const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * a.acc_cols);
                mbar_wait(&tfull[acc], accp);
                tc_fence_after();
                if (owner != krank) {
                    if (rc > 0) mbar_wait_cluster(peer_done, (rc - 1) & 1);   // owner consumed the last push
                    const int slot = krank < owner ? krank : krank - 1;
                    const uint32_t dst0 = mapa_shared(smem_u32(sRed), (uint32_t)owner) +
                                          (uint32_t)((slot * (a.FS / 4) * rpc + (L - owner * rpc)) * 16);
                    for (int c0 = 0; c0 < a.FS; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(tbase + (uint32_t)c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int g = 0; g < 8; ++g)
                            if (c0 + 4 * g < a.FS)
                                st_dsmem_f4(dst0 + (uint32_t)(((c0 / 4 + g) * rpc) * 16),
                                            make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                                        __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3])));
                    }
                    tc_fence_before();
                    // every pushing thread publishes its own stores (release.cluster arrive)
                    mbar_arrive_cluster(mapa_shared(smem_u32(recv_full), (uint32_t)owner));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                } else {
                    mbar_wait_cluster(recv_full, rc & 1);
                    const int lr = L - krank * rpc;
                    const int oy = (tc.y0 + ly) * a.ost + cl.oy0, ox = (tc.x0 + lx) * a.ost + cl.ox0;
                    const int img = tc.img + limg;
                    const bool valid = tc.valid && ly < a.Yb && lx < a.XB && img < a.n && oy < a.OH && ox < a.OW;
                    const int64_t pix = ((int64_t)img * a.OH + oy) * a.OW + ox;
                    for (int c0 = 0; c0 < a.FS; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(tbase + (uint32_t)c0, v);
                        tmem_ld_wait();
                        for (int sl = 0; sl < ks - 1; ++sl) {
#pragma unroll
                            for (int g = 0; g < 8; ++g)
                                if (c0 + 4 * g < a.FS) {
                                    const float4 p4 = sRed[(sl * (a.FS / 4) + c0 / 4 + g) * rpc + lr];
                                    v[4 * g] = __float_as_uint(__uint_as_float(v[4 * g]) + p4.x);
                                    v[4 * g + 1] = __float_as_uint(__uint_as_float(v[4 * g + 1]) + p4.y);
                                    v[4 * g + 2] = __float_as_uint(__uint_as_float(v[4 * g + 2]) + p4.z);
                                    v[4 * g + 3] = __float_as_uint(__uint_as_float(v[4 * g + 3]) + p4.w);
                                }
                        }
                        const int f = tc.f0 + c0;
                        if (!valid || f >= a.F) continue;
                        const int nf = min(min(32, a.FS - c0), a.F - f);
                        if (a.epi.on) epi_apply_bits<!kTF32, 32>(a.epi, v, pix * a.F + f, f, nf);
                        if constexpr (kTF32) {
                            float *yp = reinterpret_cast<float *>(a.y) + pix * a.F + f;
                            const int nv = vec ? (nf & ~3) : 0;
#pragma unroll
                            for (int e = 0; e < 32; e += 4)
                                if (e < nv)
                                    *reinterpret_cast<float4 *>(yp + e) =
                                        make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                                    __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e >= nv && e < nf) yp[e] = __uint_as_float(v[e]);
                        } else {
                            uint16_t *yp = reinterpret_cast<uint16_t *>(a.y) + pix * a.F + f;
                            const int nv = vec ? (nf & ~7) : 0;
#pragma unroll
                            for (int e = 0; e < 32; e += 8)
                                if (e < nv) {
                                    uint4 pk;
                                    pk.x = pack_bf16x2_rn(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
                                    pk.y = pack_bf16x2_rn(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                                    pk.z = pack_bf16x2_rn(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
                                    pk.w = pack_bf16x2_rn(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
                                    *reinterpret_cast<uint4 *>(yp + e) = pk;
                                }
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e >= nv && e < nf) yp[e] = float_to_bf16_rne(__uint_as_float(v[e]));
                        }
                    }
                    tc_fence_before();
                    // my receive buffer is free again: every owner thread tells every peer (its reads
                    // are ordered before the peers' next pushes by its own release)
                    for (int k = 0; k < ks; ++k)
                        if (k != krank) mbar_arrive_cluster(mapa_shared(smem_u32(peer_done), (uint32_t)k));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
                ++rc;
                if (threadIdx.x == 128 && item == cid) FC_TRACE(5);
                if (++acc == a.nbuf) { acc = 0; accp ^= 1; }
                continue;
            }
            if (OLLIE_FC_DEBUG && (a.dbg & 64)) {   // debug: poll with back-off instead of a blocking try_wait
                uint32_t ok = 0;
                while (true) {
                    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(smem_u32(&tfull[acc])), "r"(accp) : "memory");
                    if (ok) break;
                    __nanosleep(500);
                }
            } else
                mbar_wait(&tfull[acc], accp);
            tc_fence_after();
            for (int m = 0; m < a.MT; ++m) {
                const int oy = (tc.y0 + m * a.Yb + ly) * a.ost + cl.oy0, ox = (tc.x0 + lx) * a.ost + cl.ox0;
                const int img = tc.img + limg;
                const bool valid = tc.valid && ly < a.Yb && lx < a.XB && img < a.n && oy < a.OH && ox < a.OW;
                const int64_t pix = ((int64_t)img * a.OH + oy) * a.OW + ox;
                const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((acc * a.MT + m) * a.acc_cols);
                if (a.tma_y) {
                    // One 128-byte channel chunk at a time: every lane of the tile writes its pixel's chunk
                    // into the SWIZZLE_128B stage (row = (y * ipt + image) * XB + x, the TMA box order
                    // {c, x, image, y}), then one thread stores the whole Yb x ipt x XB box; rows / images /
                    // channels past the tensor are clipped by TMA.  Full-line writes instead of
                    // thread-per-pixel 16-byte stores (which cost 1-2 us per layer, OLLIE_FC_DBG=4).
                    constexpr int CB = kTF32 ? 32 : 64;          // channels per 128-byte row
                    const bool in_tile = ly < a.Yb && lx < a.XB;
                    const int srow = (ly * a.ipt + limg) * a.XB + lx;
                    for (int c0 = 0; c0 < a.FS; c0 += CB) {
                        if (threadIdx.x == 128) bulk_wait_read<0>();   // the stage's previous store has read it
                        named_bar_sync(1, 128);
                        // 32 columns at a time (bf16: two halves of the 128-byte row) keeps the epilogue
                        // within the register budget of the 2-CTA/SM variants
#pragma unroll 1
                        for (int h = 0; h < CB; h += 32) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(tbase + (uint32_t)(c0 + h), v);
                            tmem_ld_wait();
                            const int f = tc.f0 + c0 + h;
                            if (a.epi.on && valid && f < a.F)
                                epi_apply_bits<!kTF32, 32>(a.epi, v, pix * a.F + f, f, min(min(32, a.FS - c0 - h), a.F - f));
                            if (in_tile) {
                                uint8_t *row = sY + srow * 128;
                                if constexpr (kTF32) {
#pragma unroll
                                    for (int j = 0; j < 8; ++j)
                                        *reinterpret_cast<uint4 *>(row + ((j ^ (srow & 7)) << 4)) =
                                            make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                                } else {
#pragma unroll
                                    for (int j = 0; j < 4; ++j) {
                                        uint4 pk;
                                        pk.x = pack_bf16x2_rn(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1]));
                                        pk.y = pack_bf16x2_rn(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                                        pk.z = pack_bf16x2_rn(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                                        pk.w = pack_bf16x2_rn(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                                        const int jj = (h >> 3) + j;          // 16-byte chunk of the row
                                        *reinterpret_cast<uint4 *>(row + ((jj ^ (srow & 7)) << 4)) = pk;
                                    }
                                }
                            }
                        }
                        fence_proxy_async_smem();
                        named_bar_sync(1, 128);
                        if (threadIdx.x == 128 && tc.valid) {   // (the odd CTA of a last pair stores nothing)
                            tma_store_4d(&tmY, sY, tc.f0 + c0, tc.x0 * a.ost + cl.ox0, tc.img,
                                         (tc.y0 + m * a.Yb) * a.ost + cl.oy0);
                            bulk_commit();
                        }
                    }
                    continue;
                }
                // up to 64 columns per round: both TMEM loads in flight before one wait
                for (int c0 = 0; c0 < a.FS; c0 += 64) {
                    uint32_t v[64];
                    tmem_ld_32x32b_x32(tbase + (uint32_t)c0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    const bool two = c0 + 32 < a.FS;
                    if (two) tmem_ld_32x32b_x32(tbase + (uint32_t)(c0 + 32), *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    tmem_ld_wait();
                    const int f = tc.f0 + c0;
                    if (!valid || f >= a.F || (OLLIE_FC_DEBUG && (a.dbg & 4))) continue;
                    const int nf = min(min(64, a.FS - c0), a.F - f);
                    if (a.epi.on) epi_apply_bits<!kTF32, 64>(a.epi, v, pix * a.F + f, f, nf);
                    if constexpr (kTF32) {
                        float *yp = reinterpret_cast<float *>(a.y) + pix * a.F + f;
                        const int nv = vec ? (nf & ~3) : 0;      // whole 16-byte groups, then a scalar tail
#pragma unroll
                        for (int e = 0; e < 64; e += 4)
                            if (e < nv)
                                *reinterpret_cast<float4 *>(yp + e) =
                                    make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                                __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
#pragma unroll
                        for (int e = 0; e < 64; ++e)
                            if (e >= nv && e < nf) yp[e] = __uint_as_float(v[e]);
                    } else {
                        uint16_t *yp = reinterpret_cast<uint16_t *>(a.y) + pix * a.F + f;
                        const int nv = vec ? (nf & ~7) : 0;      // whole 16-byte groups, then a scalar tail
                        {
#pragma unroll
                            for (int e = 0; e < 64; e += 8)
                                if (e < nv) {
                                    uint4 pk;
                                    pk.x = pack_bf16x2_rn(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
                                    pk.y = pack_bf16x2_rn(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                                    pk.z = pack_bf16x2_rn(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
                                    pk.w = pack_bf16x2_rn(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
                                    *reinterpret_cast<uint4 *>(yp + e) = pk;
                                }
#pragma unroll
                            for (int e = 0; e < 64; ++e)
                                if (e >= nv && e < nf) yp[e] = float_to_bf16_rne(__uint_as_float(v[e]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (kPair) mbar_arrive_cluster(tempty_leader0 + (uint32_t)acc * 8u);
                else mbar_arrive(&tempty[acc]);
            }
            if (threadIdx.x == 128 && item == cid) FC_TRACE(5);
            if (++acc == a.nbuf) { acc = 0; accp ^= 1; }
        }
        if (a.tma_y && threadIdx.x == 128) bulk_wait<0>();   // Y stores complete before the stage retires
        if (ks > 1 && rc > 0 && (L / (128 / ks)) != krank) {
            // pusher warps: the owners' last "consumed" arrives must land before this CTA may leave
            mbar_wait_cluster(peer_done, (rc - 1) & 1);
        }
        if (threadIdx.x == 128) FC_TRACE(6);
        if (a.trace && threadIdx.x == 128) *reinterpret_cast<volatile uint32_t *>(tmem_slot + 1) = 0xD0E;
    }

    tc_fence_before();
    if (kPair || ks > 1) cluster_sync();   // no CTA leaves while a peer's MMAs / arrives / reads may target it
    else __syncthreads();
    if (threadIdx.x == 0) FC_TRACE(31);
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 32 + 28] = *reinterpret_cast<volatile uint32_t *>(tmem_slot + 1);
    if (a.trace && threadIdx.x == 128) FC_TRACE(29);
    if (warp == 2) {
        tc_fence_after();
        if constexpr (kPair) {
            if (a.tmem_cols == 256) tmem_dealloc_pair<256>(tmem_base);
            else tmem_dealloc_pair<FC_TMEM_COLS>(tmem_base);
        } else {
            if (a.tmem_cols == 256) tmem_dealloc<256>(tmem_base);
            else tmem_dealloc<FC_TMEM_COLS>(tmem_base);
        }
    }
}

}  // namespace ollie
