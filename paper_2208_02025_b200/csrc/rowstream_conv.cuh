// rowstream_conv.cuh -- a8 for NARROW outputs (FSRCNN's 12/16-channel layers, its 56 -> 1 9x9
// deconvolution, DCGAN's 64 -> 3 ConvT): the merged GEMM + OffsetAdd with the r*s taps split
// between the two halves of the derived program instead of being carried by one.
//
// Derivation.  The merged Matmul (E6) computes T[m, (i, j, f)] with N = r*s*f, and
// OffsetAdd (E7) sums T over the r*s shifted regions.  Summation splitting
// applied to the two tap dimensions separately gives
//     Y[y, x, f] = Sum_i D_{y - p + i}[x, (i, f)],   D_r[x, (i, f)] = Sum_j Sum_c X[r, x - p + j, c] W'[(i, j, f), c]
// i.e. for every INPUT row r one merged GEMM whose N is (i, f) -- the kernel ROWS and the output
// channels, r*f wide -- accumulated over the kernel COLUMNS j by shifting the A operand by j pixels
// (the OffsetAdd of the column offsets done by the tensor core into TMEM), and an OffsetAdd over
// the row offsets i only, done in the epilogue by adding column group i of the TMEM accumulators
// of consecutive input rows (same TMEM lanes: no data crosses lanes).  For narrow f this keeps
// N = r*f >= 16 useful columns per MMA instead of f, each A row is read s (not r*s) times, and an
// input row is needed in shared memory only while its own MMAs run.  Zero padding: the
// pixels left / right of the image are zero rows kept in every ring slot; rows above / below the
// image have no D (their OffsetAdd terms are 0).
//
// ConvTranspose2d is first rewritten by expression splitting over the output residue
// classes (cy, cx) -- class (cy, cx) of output row sigma*q + cy reads input rows q + d
// with kernel row i = cy + p - sigma*d -- and the classes are then put on N as well ("sub-pixel"
// form): a stride-1 program over the union of the classes' input offsets d in [dmin, dmax], with
// sigma^2 * f columns per kernel row, whose epilogue writes each class interleaved into NHWC Y
// (the fused "selective add o interleave DLT" pair).  Its weight tiles are the
// prepared W' re-indexed by (d, cy, cx, f) -- built in shared memory by the CTA, zero where a class
// has no tap.
//
// Schedule: a persistent CTA owns a contiguous run of output rows (n * OH rows in total, split
// evenly) and streams the input rows they read through a ring of shared-memory slots, one TMA box
// per row (<= 256 pixels, 32/64/128-byte swizzled pixel rows), each input row loaded ONCE per run.
// Measured on B200: a CTA's TMA boxes are serviced one after another with microseconds of latency
// from HBM, so the ring only ever holds rows in flight or under MMA (never the r-row window).
// Input row r, M-tile h (pixels 128h .. 128h + 127): s shifts x ksteps tcgen05.mma 128 x NP x 16 into
// TMEM row slot r % NT.  Warp 0: TMA producer; warp 1: MMA issuer; warp 2: TMEM allocator; warps
// 4-7: epilogue (r TMEM loads per M-tile, the row OffsetAdd, NEXT-3 element-wise ops, RNE, stores).
#pragma once
#include "../../include/ollie.h"
#include "sm100_ptx.cuh"
#include "epilogue.cuh"

#include <type_traits>

namespace ollie {

constexpr int RS_THREADS = 384;       // warps 0-3: TMA, MMA, TMEM, idle; 4-11: two epilogue groups
constexpr int RS_MAX_NP = 64;          // columns per input row the epilogue reads (r * f')
constexpr int RS_MAX_S = 9;            // kernel columns of the stride-1 program (A-row shifts)
constexpr int RS_ZR = 8;               // zero pixel rows before / after the image row in a slot (one swizzle atom)

struct RsArgs {
    int32_t n, H, W, C;                // input NHWC, C channels in memory
    int32_t F, R0, S0, pad0;           // the layer: output channels, kernel, padding (weight re-indexing)
    int32_t R, S, pad_y, pad_x;        // the stride-1 program: output row y reads input rows y - pad_y + i
    int32_t sub;                       // sigma of a ConvTranspose2d in sub-pixel form (1 for Conv2d)
    int32_t tr;                        // 1: ConvTranspose2d (weights re-indexed by class), 0: Conv2d
    int32_t direct;                    // 1: direct form (N = f, every tap an A shift, one accumulator per OUTPUT row)
    int32_t OHc, OWc;                  // output grid of the stride-1 program (class grid for sub > 1)
    int32_t OH, OW;                    // the layer's output (clipping of the interleaved classes)
    int32_t Fp, N, NP, acc_cols;       // Fp = sub^2 * F columns per kernel row; N = R * Fp -> NP (mult. of 16)
    int32_t nt, row_cols;              // TMEM row slots (D of one input row = mtr accumulators) and their width
    int32_t mtr;                       // M-tiles (128 pixels) per image row
    int32_t rowbytes, swz, ksteps;     // pixel row in smem (32/64/128 B), UMMA layout code, K steps per row
    int32_t ring, slot_bytes, wbox, nbox;
    int32_t tmem_cols;                 // 512 (1 CTA / SM)
    int64_t rows_total;                // n * OHc
    const void *wprep;                 // W' [(i * S0 + j) * F + f][C]
    void *y;
    EpiArgs epi;
    long long *trace;                  // debug only (nullptr in production): CTA 0 timeline, %globaltimer ns
    int32_t dbg;                       // debug only (0 in production; reserved for ablations)
};

// shared-memory carve-up (host and device agree): ring | B tiles (one per kernel column) | barriers
__host__ __device__ inline int rs_b_bytes(const RsArgs &a) { return (a.direct ? a.R * a.S : a.S) * a.NP * a.rowbytes; }
__host__ __device__ inline int rs_bar_bytes(const RsArgs &a) { return 8 * (2 * a.ring + 2 * a.nt) + 16; }
__host__ __device__ inline size_t rs_smem_bytes(const RsArgs &a) {
    return 1024 + (size_t)a.ring * a.slot_bytes + rs_b_bytes(a) + rs_bar_bytes(a);
}

// One contiguous run of output rows of one image inside [g, g1).
struct RsSeg {
    int img, ylo, yhi, rlo, rhi;       // output rows [ylo, yhi); input rows [rlo, rhi) they read
};
__device__ __forceinline__ RsSeg rs_seg(const RsArgs &a, int64_t g, int64_t g1) {
    RsSeg s;
    s.img = (int)(g / a.OHc);
    s.ylo = (int)(g - (int64_t)s.img * a.OHc);
    { const int64_t e = (int64_t)s.ylo + (g1 - g); s.yhi = (int)(e < (int64_t)a.OHc ? e : (int64_t)a.OHc); }
    s.rlo = max(0, s.ylo - a.pad_y);
    s.rhi = min(a.H, s.yhi - a.pad_y + a.R - 1);
    if (s.rhi < s.rlo) s.rhi = s.rlo;
    return s;
}

__device__ __forceinline__ long long rs_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
}

// bf16 / fp32 store of one element (Y's dtype)
template <bool kTF32>
__device__ __forceinline__ void rs_store1(void *y, int64_t e, float v) {
    if constexpr (kTF32) reinterpret_cast<float *>(y)[e] = v;
    else reinterpret_cast<uint16_t *>(y)[e] = float_to_bf16_rne(v);
}

// Y[e0 .. e0 + kN) = v[0 .. kN) for one pixel (kN compile-time, the pixel's kN * ES bytes are
// aligned to their size's largest power-of-two divisor): the widest vector stores that alignment
// allows (16 / 8 / 4 bytes) -- a 12-channel bf16 pixel leaves as three 8-byte stores, not twelve
// 2-byte ones (the LSU cost of the narrow-f epilogues is per store instruction).
template <bool kTF32, int kN>
__device__ __forceinline__ void rs_store_pixel(void *y, int64_t e0, const float *v) {
    constexpr int ES = kTF32 ? 4 : 2, B = kN * ES;
    constexpr int VB = (B % 16 == 0) ? 16 : (B % 8 == 0) ? 8 : (B % 4 == 0) ? 4 : ES;
    constexpr int VE = VB / ES;                          // elements per store
    uint8_t *base = reinterpret_cast<uint8_t *>(y) + e0 * ES;
#pragma unroll
    for (int f = 0; f < kN; f += VE) {
        uint32_t w[4];
        if constexpr (kTF32) {
#pragma unroll
            for (int u = 0; u < VE; ++u) w[u] = __float_as_uint(v[f + u]);
        } else {
#pragma unroll
            for (int u = 0; u < VE / 2; ++u) w[u] = pack_bf16x2_rn(v[f + 2 * u], v[f + 2 * u + 1]);
        }
        if constexpr (VB == 16) *reinterpret_cast<uint4 *>(base + f * ES) = make_uint4(w[0], w[1], w[2], w[3]);
        else if constexpr (VB == 8) *reinterpret_cast<uint2 *>(base + f * ES) = make_uint2(w[0], w[1]);
        else if constexpr (VB == 4) *reinterpret_cast<uint32_t *>(base + f * ES) = w[0];
        else rs_store1<kTF32>(y, e0 + f, v[f]);
    }
}

// tcgen05.ld of kFp consecutive fp32 columns (kFp in {4, 8, 12, 16}) into v[0, kFp)
template <int kFp>
__device__ __forceinline__ void rs_tmem_ld(uint32_t taddr, uint32_t *v) {
    if constexpr (kFp == 16) {
        tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(v));
    } else {
        if constexpr (kFp >= 8)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(taddr));
        if constexpr (kFp % 8 == 4)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[kFp - 4]), "=r"(v[kFp - 3]), "=r"(v[kFp - 2]), "=r"(v[kFp - 1])
                         : "r"(taddr + (uint32_t)(kFp - 4)));
    }
}

// MMAs of one M-tile of one input row: kS column shifts x kKS k-steps, D (+)= shift_j(A) W'_j.
// Called by the converged MMA warp; one elected lane issues each MMA (umma_elect_lohi) with the
// warp-uniform descriptor words plus compile-time offsets.  The shift / k-step counts are template
// parameters: the same walk with runtime bounds (the _rt fallback) puts a data-dependent branch
// before every MMA, and ptxas then re-converges the warp around each one -- measured on B200 at
// ~205 cycles per MMA against ~25-65 for the straight-line form (tools/mma_rate.cu: the tensor
// core itself takes ~40 cycles per 128 x 16 x 16 MMA, its (128 + N) x 32-byte SMEM operand read).
template <bool kTF32, int kS, int kKS>
__device__ __forceinline__ void rs_issue_shifts(uint32_t d, uint32_t alo, uint32_t blo, uint32_t hi, uint32_t a_step,
                                                uint32_t b_step, uint32_t idesc, uint32_t acc0) {
#pragma unroll
    for (int j = 0; j < kS; ++j)
#pragma unroll
        for (int k = 0; k < kKS; ++k)
            umma_elect_lohi<kTF32>(d, alo + (uint32_t)j * a_step + 2u * k, hi, blo + (uint32_t)j * b_step + 2u * k, hi, idesc,
                                   (j == 0 && k == 0) ? acc0 : 1u);
}
template <bool kTF32>
__device__ __forceinline__ void rs_issue_shifts_rt(uint32_t d, uint32_t alo, uint32_t blo, uint32_t hi, uint32_t a_step,
                                                   uint32_t b_step, uint32_t idesc, uint32_t acc0, int S, int ksteps) {
#pragma unroll
    for (int j = 0; j < RS_MAX_S; ++j) {
        if (j < S) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < ksteps)
                    umma_elect_lohi<kTF32>(d, alo + (uint32_t)j * a_step + 2u * k, hi, blo + (uint32_t)j * b_step + 2u * k,
                                           hi, idesc, (j == 0 && k == 0) ? acc0 : 1u);
        }
    }
}
template <bool kTF32, int kS, int kKS>
__device__ __forceinline__ void rs_issue(uint32_t d, uint32_t alo, uint32_t blo, uint32_t hi, uint32_t a_step,
                                         uint32_t b_step, uint32_t idesc, uint32_t acc0, int S, int ksteps) {
    if constexpr (kS > 0) rs_issue_shifts<kTF32, kS, kKS>(d, alo, blo, hi, a_step, b_step, idesc, acc0);
    else rs_issue_shifts_rt<kTF32>(d, alo, blo, hi, a_step, b_step, idesc, acc0, S, ksteps);
}
template <int v>
using rs_ic = std::integral_constant<int, v>;
// Runs body(rs_ic<S>, rs_ic<ksteps>) for the (S, ksteps) pairs the planner produces most (1x1, 3x3,
// 5x5 programs; 1-4 channel chunks), else body(rs_ic<0>, rs_ic<0>) (runtime bounds).
template <typename Body>
__device__ __forceinline__ void rs_dispatch_shifts(int S, int ksteps, Body &&body) {
    switch (S * 8 + ksteps) {
        case 1 * 8 + 1: body(rs_ic<1>{}, rs_ic<1>{}); break;
        case 1 * 8 + 2: body(rs_ic<1>{}, rs_ic<2>{}); break;
        case 1 * 8 + 3: body(rs_ic<1>{}, rs_ic<3>{}); break;
        case 1 * 8 + 4: body(rs_ic<1>{}, rs_ic<4>{}); break;
        case 3 * 8 + 1: body(rs_ic<3>{}, rs_ic<1>{}); break;
        case 3 * 8 + 2: body(rs_ic<3>{}, rs_ic<2>{}); break;
        case 3 * 8 + 4: body(rs_ic<3>{}, rs_ic<4>{}); break;
        case 5 * 8 + 1: body(rs_ic<5>{}, rs_ic<1>{}); break;
        case 5 * 8 + 2: body(rs_ic<5>{}, rs_ic<2>{}); break;
        case 5 * 8 + 4: body(rs_ic<5>{}, rs_ic<4>{}); break;
        default: body(rs_ic<0>{}, rs_ic<0>{}); break;
    }
}

template <bool kTF32, int kFp, bool kDirect>
__global__ void __launch_bounds__(RS_THREADS, 1)
rowstream_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ RsArgs a) {
    constexpr int ES = kTF32 ? 4 : 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sRing = smem;
    uint8_t *sB = sRing + (size_t)a.ring * a.slot_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + rs_b_bytes(a));
    uint64_t *full = bars;                    // [ring]  input row landed
    uint64_t *empty = full + a.ring;          // [ring]  MMAs reading the slot retired
    uint64_t *afull = empty + a.ring;         // [nt]    D of the slot's input row complete
    uint64_t *aempty = afull + a.nt;          // [nt]    every output row reading it is done
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(aempty + a.nt);

    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    const int lane = threadIdx.x & 31;
    const int64_t g0 = a.rows_total * (int64_t)blockIdx.x / gridDim.x;
    const int64_t g1 = a.rows_total * (int64_t)(blockIdx.x + 1) / gridDim.x;

    if (warp == 0 && lane == 0) tma_prefetch_desc(&tmX);
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < a.ring; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < a.nt; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], kDirect ? 4 : 8); }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    {
        // B tile j (kernel column j of the stride-1 program): NP rows (i, [cy, cx,] f) x C channels,
        // K-major in the swizzled layout the MMA descriptor names (weights are read-only for the
        // stream, so this overlaps the previous kernel under PDL)
        const int cpr = a.rowbytes / 16, CI = 16 / ES;
        const uint32_t swmask = (uint32_t)cpr - 1;
        const int total = (kDirect ? a.R * a.S : a.S) * a.NP * cpr;
        for (int t = threadIdx.x; t < total; t += RS_THREADS) {
            const int chunk = t % cpr, nrow = (t / cpr) % a.NP, j = t / (cpr * a.NP);
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if constexpr (kDirect) {             // tile i*S + j of tap (i, j): rows f < F
                const int ti = j / a.S, tj = j - ti * a.S, c0 = chunk * CI;
                if (nrow < a.F && c0 < a.C)
                    v = __ldg(reinterpret_cast<const uint4 *>(reinterpret_cast<const uint8_t *>(a.wprep) +
                                                              ((((int64_t)ti * a.S0 + tj) * a.F + nrow) * a.C + c0) * ES));
            } else if (nrow < a.N) {
                const int i = nrow / a.Fp, rem = nrow - i * a.Fp;
                int ki, kj, f;
                if (!a.tr) {
                    ki = i; kj = j; f = rem;
                } else {   // tap of class (cy, cx) at union offset (i - pad_y, j - pad_x): k = cy + p - sigma*d
                    const int cls = rem / a.F;
                    f = rem - cls * a.F;
                    const int cy = cls / a.sub, cx = cls - cy * a.sub;
                    ki = cy + a.pad0 - a.sub * (i - a.pad_y);
                    kj = cx + a.pad0 - a.sub * (j - a.pad_x);
                }
                const int c0 = chunk * CI;
                if (ki >= 0 && ki < a.R0 && kj >= 0 && kj < a.S0 && c0 < a.C)
                    v = __ldg(reinterpret_cast<const uint4 *>(reinterpret_cast<const uint8_t *>(a.wprep) +
                                                              ((((int64_t)ki * a.S0 + kj) * a.F + f) * a.C + c0) * ES));
            }
            const uint32_t off = (uint32_t)(j * a.NP + nrow) * (uint32_t)a.rowbytes + (uint32_t)chunk * 16u;
            *reinterpret_cast<uint4 *>(sB + (off ^ (((off >> 7) & swmask) << 4))) = v;
        }
        // the zero pixel rows of every ring slot (left of the image, and right of what TMA writes)
        const int slot_rows = a.slot_bytes / a.rowbytes, tma_rows = a.nbox * a.wbox;
        const int zrows = slot_rows - tma_rows, z16 = zrows * cpr;
        for (int t = threadIdx.x; t < a.ring * z16; t += RS_THREADS) {
            const int sl = t / z16, u = t - sl * z16, row = u / cpr, chunk = u - row * cpr;
            const int prow = row < RS_ZR ? row : row + tma_rows;
            *reinterpret_cast<uint4 *>(sRing + (size_t)sl * a.slot_bytes + (size_t)prow * a.rowbytes + chunk * 16) =
                make_uint4(0u, 0u, 0u, 0u);
        }
        fence_proxy_async_smem();   // generic-proxy writes -> visible to TMA / the tensor core (async proxy)
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    if (threadIdx.x == 0) pdl_launch_dependents();

    // Ring slots and TMEM row slots are walked with counters (slot index + phase bit): these loops run
    // once per image row on one warp per SM sub-partition, where a runtime division's dependent
    // latency is not hidden by other warps.
    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer: every input row of the CTA's runs, once, in order =====
            pdl_wait();                                  // X is produced by the previous kernel
            const uint32_t row_tx = (uint32_t)(a.nbox * a.wbox * a.rowbytes);
            const int ring = a.ring, nbox = a.nbox, wbox = a.wbox;
            const size_t slot_bytes = (size_t)a.slot_bytes, box_bytes = (size_t)wbox * a.rowbytes;
            uint8_t *const ring0 = sRing + (size_t)RS_ZR * a.rowbytes;
            int slot = 0;
            uint32_t ph = 0, seq = 0;
            for (int64_t g = g0; g < g1;) {
                const RsSeg s = rs_seg(a, g, g1);
                for (int r = s.rlo; r < s.rhi; ++r, ++seq) {
                    mbar_wait(&empty[slot], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[slot], row_tx);
                    if (a.trace && blockIdx.x == 0 && seq < 64) a.trace[seq] = rs_gtimer();
                    uint8_t *dst = ring0 + (size_t)slot * slot_bytes;
                    for (int b = 0; b < nbox; ++b)
                        tma_load_4d(dst + (size_t)b * box_bytes, &tmX, &full[slot], 0, b * wbox, r, s.img);
                    if (++slot == ring) { slot = 0; ph ^= 1u; }
                }
                g += s.yhi - s.ylo;
            }
        }
    } else if (kDirect && warp == 1) {
        // ===== direct form, MMA issuer: accumulator of OUTPUT row y = Sum_{i,j} shift_j(X_{y-p+i}) W'_{i,j} =====
        const uint32_t idesc = make_idesc(kTF32, 128, (uint32_t)a.NP);
        const uint64_t dtpl = ((uint64_t)1 << 16) | ((uint64_t)((8u * (uint32_t)a.rowbytes) >> 4) << 32) |
                              ((uint64_t)1 << 46) | ((uint64_t)a.swz << 61);
        const uint32_t row16 = (uint32_t)a.rowbytes >> 4, slot16 = (uint32_t)a.slot_bytes >> 4;
        const uint32_t b16 = smem_u32(sB) >> 4, bt16 = (uint32_t)(a.NP * a.rowbytes) >> 4;
        const uint32_t lo0 = (uint32_t)dtpl, hi = (uint32_t)(dtpl >> 32), blo = lo0 + b16;
        const uint32_t ring_a16 = (smem_u32(sRing) >> 4) + (uint32_t)(RS_ZR - a.pad_x) * row16;
        const uint32_t mt16 = 128u * row16, acc_cols = (uint32_t)a.acc_cols, row_cols = (uint32_t)a.row_cols;
        const int ring = a.ring, nt = a.nt, ksteps = a.ksteps, S = a.S, R = a.R, mtr = a.mtr, pad_y = a.pad_y;
        int t = 0;                                      // TMEM slot of the output row
        uint32_t tph = 0;
        int next_slot = 0;                              // ring slot of the next loaded row
        int wslot = 0;                                  // full-wait cursor: next loaded row to wait for
        uint32_t wph = 0, wseq = 0, seq0 = 0;
        int rslot = 0;                                  // release cursor: next loaded row to hand back
        uint32_t rseq = 0;
        auto wait_upto = [&](uint32_t sq) {
            while (wseq <= sq) {
                mbar_wait_warp(&full[wslot], wph);
                if (++wslot == ring) { wslot = 0; wph ^= 1u; }
                ++wseq;
            }
        };
        auto release_upto = [&](uint32_t sq_end) {     // rows with sequence < sq_end
            while (rseq < sq_end) {
                wait_upto(rseq);
                umma_commit_elect(&empty[rslot]);       // retires with the MMAs that read the row
                __syncwarp();
                if (++rslot == ring) rslot = 0;
                ++rseq;
            }
        };
        rs_dispatch_shifts(S, ksteps, [&](auto Sc, auto KSc) {
          constexpr int kS = decltype(Sc)::value, kKS = decltype(KSc)::value;
          for (int64_t g = g0; g < g1;) {
            const RsSeg s = rs_seg(a, g, g1);
            const int slot0 = next_slot;
            for (int y = s.ylo; y < s.yhi; ++y) {
                const int rb = y - pad_y;
                const int i_lo = max(0, s.rlo - rb), i_hi = min(R, s.rhi - rb);
                if (i_hi > i_lo) wait_upto(seq0 + (uint32_t)(rb + i_hi - 1 - s.rlo));
                mbar_wait_warp(&aempty[t], tph ^ 1u);
                tc_fence_after();
                const uint32_t d0 = tmem_base + (uint32_t)t * row_cols;
                const int64_t kr = (int64_t)(y - s.ylo) + (g - g0);
                if ((a.dbg & 8) && a.trace && blockIdx.x == 0 && kr == 5 && lane == 0) a.trace[319] = clock64();
                if (a.trace && blockIdx.x == 0 && kr < 64 && lane == 0) a.trace[64 + kr] = rs_gtimer();
                int sl = slot0 + (rb + i_lo - s.rlo);            // ring slot of input row rb + i_lo
                while (sl >= ring) sl -= ring;
                for (int i = i_lo; i < i_hi; ++i) {
                    const uint32_t a0 = lo0 + ring_a16 + (uint32_t)sl * slot16;
                    const uint32_t bi = blo + (uint32_t)(i * S) * bt16;
                    for (int h = 0; h < mtr; ++h) {
                        rs_issue<kTF32, kS, kKS>(d0 + (uint32_t)h * acc_cols, a0 + (uint32_t)h * mt16, bi, hi, row16, bt16,
                                                 idesc, i == i_lo ? 0u : 1u, S, ksteps);
                        if ((a.dbg & 8) && a.trace && blockIdx.x == 0 && kr == 5 && lane == 0)
                            a.trace[320 + (i - i_lo) * mtr + h] = clock64();
                    }
                    if (++sl == ring) sl = 0;
                }
                __syncwarp();
                umma_commit_elect(&afull[t]);           // (no valid tap: arrives at once; the epilogue writes 0)
                __syncwarp();
                if (a.trace && blockIdx.x == 0 && kr < 64 && lane == 0) a.trace[128 + kr] = rs_gtimer();
                if (++t == nt) { t = 0; tph ^= 1u; }
                // no later output row reads rb (rows below the image, rb >= rhi, were never loaded)
                if (rb >= s.rlo) release_upto(seq0 + (uint32_t)min(rb - s.rlo + 1, s.rhi - s.rlo));
            }
            release_upto(seq0 + (uint32_t)(s.rhi - s.rlo));
            seq0 += (uint32_t)(s.rhi - s.rlo);
            next_slot = slot0 + (s.rhi - s.rlo);
            while (next_slot >= ring) next_slot -= ring;
            g += s.yhi - s.ylo;
          }
        });
    } else if (kDirect && warp >= 4) {
        // ===== direct form, epilogue: two groups on alternate output rows; one TMEM slot per output row =====
        const int q = warp & 3;
        const int gi = (warp - 4) >> 2;
        pdl_wait();
        const int nt = a.nt, R = a.R, mtr = a.mtr, pad_y = a.pad_y, OWc = a.OWc, F = a.F, NP = a.NP;
        const uint32_t row_cols = (uint32_t)a.row_cols, acc_cols = (uint32_t)a.acc_cols;
        const uint32_t lane0 = tmem_base + ((uint32_t)(q * 32) << 16);
        const int xq = 32 * q + lane;
        int t = 0;
        uint32_t tph = 0, krow = 0;
        uint32_t v[RS_MAX_NP];
        for (int64_t g = g0; g < g1;) {
            const RsSeg s = rs_seg(a, g, g1);
            const int64_t img_el = (int64_t)s.img * a.OH;
            for (int y = s.ylo; y < s.yhi; ++y, ++krow) {
                const int tt = t;
                const uint32_t ph = tph;
                if (++t == nt) { t = 0; tph ^= 1u; }
                if ((int)(krow & 1u) != gi) continue;
                const int rb = y - pad_y;
                const bool any = min(R, s.rhi - rb) > max(0, s.rlo - rb);
                mbar_wait(&afull[tt], ph);
                tc_fence_after();
                if (a.dbg & 1) {                         // ablation: no TMEM reads, no stores
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aempty[tt]);
                    continue;
                }
                for (int h = 0; h < mtr; ++h) {
                    const uint32_t tb = lane0 + (uint32_t)tt * row_cols + (uint32_t)h * acc_cols;
#pragma unroll
                    for (int c = 0; c < RS_MAX_NP; c += 16)
                        if (c < NP) tmem_ld_32x32b_x16(tb + (uint32_t)c, *reinterpret_cast<uint32_t(*)[16]>(&v[c]));
                    tmem_ld_wait();
                    if (h == mtr - 1) {                  // the row's accumulator is read: hand the slot back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aempty[tt]);
                    }
                    const int x = 128 * h + xq;
                    if (x >= OWc) continue;
                    if (!any) {
#pragma unroll
                        for (int f = 0; f < RS_MAX_NP; ++f) v[f] = 0u;
                    }
                    float *out = reinterpret_cast<float *>(v);   // the accumulator values, in place
                    const int64_t e0 = ((img_el + y) * a.OW + x) * F;
                    if (a.epi.on) epi_apply<!kTF32, RS_MAX_NP>(a.epi, out, e0, 0, F);
                    if (((F * ES) % 16) == 0) {               // groups of 16 bytes
                        constexpr int G = 16 / ES;
#pragma unroll
                        for (int f = 0; f < RS_MAX_NP; f += G)
                            if (f < F) rs_store_pixel<kTF32, G>(a.y, e0 + f, out + f);
                    } else if (((F * ES) % 8) == 0) {
                        constexpr int G = 8 / ES;
#pragma unroll
                        for (int f = 0; f < RS_MAX_NP; f += G)
                            if (f < F) rs_store_pixel<kTF32, G>(a.y, e0 + f, out + f);
                    } else if (((F * ES) % 4) == 0) {
                        constexpr int G = 4 / ES;
#pragma unroll
                        for (int f = 0; f < RS_MAX_NP; f += G)
                            if (f < F) rs_store_pixel<kTF32, G>(a.y, e0 + f, out + f);
                    } else {
#pragma unroll
                        for (int f = 0; f < RS_MAX_NP; ++f)
                            if (f < F) rs_store1<kTF32>(a.y, e0 + f, out[f]);
                    }
                }
                if (a.trace && blockIdx.x == 0 && lane == 0 && q == 0) {
                    const int64_t kr = (int64_t)(y - s.ylo) + (g - g0);
                    if (kr < 64) a.trace[192 + kr] = rs_gtimer();
                }
            }
            g += s.yhi - s.ylo;
        }
    } else if (!kDirect && warp == 1) {
        // ===== MMA issuer (converged warp, one elected lane issues): D_r = Sum_j shift_j(X_r) W'_j =====
        const uint32_t idesc = make_idesc(kTF32, 128, (uint32_t)a.NP);
        const uint64_t dtpl = ((uint64_t)1 << 16) | ((uint64_t)((8u * (uint32_t)a.rowbytes) >> 4) << 32) |
                              ((uint64_t)1 << 46) | ((uint64_t)a.swz << 61);
        const uint32_t row16 = (uint32_t)a.rowbytes >> 4, slot16 = (uint32_t)a.slot_bytes >> 4;
        const uint32_t b16 = smem_u32(sB) >> 4, bj16 = (uint32_t)(a.NP * a.rowbytes) >> 4;
        // descriptor words: lo = start address >> 4 (14 bits, smem < 256 KB) | LBO; hi = SBO, version, swizzle
        const uint32_t lo0 = (uint32_t)dtpl, hi = (uint32_t)(dtpl >> 32), blo = lo0 + b16;
        const uint32_t ring_a16 = (smem_u32(sRing) >> 4) + (uint32_t)(RS_ZR - a.pad_x) * row16;
        const uint32_t mt16 = 128u * row16, acc_cols = (uint32_t)a.acc_cols, row_cols = (uint32_t)a.row_cols;
        const int ring = a.ring, nt = a.nt, ksteps = a.ksteps, S = a.S, mtr = a.mtr;
        int slot = 0, t = 0;
        uint32_t ph = 0, tph = 0, seq = 0;
        rs_dispatch_shifts(S, ksteps, [&](auto Sc, auto KSc) {
          constexpr int kS = decltype(Sc)::value, kKS = decltype(KSc)::value;
          for (int64_t g = g0; g < g1;) {
            const RsSeg s = rs_seg(a, g, g1);
            for (int r = s.rlo; r < s.rhi; ++r, ++seq) {
                mbar_wait_warp(&full[slot], ph);
                if (a.trace && blockIdx.x == 0 && seq < 64 && lane == 0) a.trace[64 + seq] = rs_gtimer();
                mbar_wait_warp(&aempty[t], tph ^ 1u);
                tc_fence_after();
                const uint32_t d0 = tmem_base + (uint32_t)t * row_cols;
                const uint32_t a0 = lo0 + ring_a16 + (uint32_t)slot * slot16;
                // the converged warp walks the row's (M-tile, shift, k-step) MMAs (rs_issue_shifts)
                for (int h = 0; h < mtr; ++h)
                    rs_issue<kTF32, kS, kKS>(d0 + (uint32_t)h * acc_cols, a0 + (uint32_t)h * mt16, blo, hi, row16, bj16,
                                             idesc, 0u, S, ksteps);
                __syncwarp();
                umma_commit_elect(&afull[t]);
                umma_commit_elect(&empty[slot]);         // the slot returns to the producer when they retire
                __syncwarp();
                if (a.trace && blockIdx.x == 0 && seq < 64 && lane == 0) a.trace[128 + seq] = rs_gtimer();
                if (++slot == ring) { slot = 0; ph ^= 1u; }
                if (++t == nt) { t = 0; tph ^= 1u; }
            }
            g += s.yhi - s.ylo;
          }
        });
    } else if (!kDirect && warp >= 4) {
        // ===== epilogue: Y[y] = Sum_i column group i of D_{y - pad_y + i}; element-wise ops; stores =====
        // Two groups of 4 warps: group gi takes the CTA's output rows k with k % 2 == gi (one warp per SM
        // sub-partition runs this loop at dependent-instruction latency: two rows in flight per
        // sub-partition double the rate).  Each group hands every input row's TMEM slot back once
        // (aempty counts 8 arrivals): after its last output row reading it, or at the run's end.
        const int q = warp & 3;                          // TMEM lane quadrant of this warp
        const int gi = (warp - 4) >> 2;
        pdl_wait();                                      // Y may still be read by the previous kernel
        const int nt = a.nt, R = a.R, mtr = a.mtr, pad_y = a.pad_y, OWc = a.OWc, sub = a.sub, F = a.F;
        const uint32_t row_cols = (uint32_t)a.row_cols, acc_cols = (uint32_t)a.acc_cols;
        const uint32_t lane0 = tmem_base + ((uint32_t)(q * 32) << 16);
        const int xq = 32 * q + lane;
        const int64_t OWF = (int64_t)a.OW * F;
        // The kernel-row count is a compile-time constant for the common programs (r' = 1, 3, 5):
        // the R TMEM loads and the row sum are then straight-line code with the image-edge rows
        // masked by a select, not branched around (a tcgen05.ld is warp-collective: a branch around
        // it makes ptxas re-converge the warp per load -- measured ~480 cycles to issue one row's loads).
        auto epilogue = [&](auto Rc) {
        constexpr int kR = decltype(Rc)::value;          // 0: runtime R (generic shapes)
        constexpr int kRI = kR > 0 ? kR : RS_MAX_NP / kFp;
        uint32_t v[kRI * kFp];
        int tb = 0;                                      // TMEM slot of the run's first loaded row (rlo)
        uint32_t seq0 = 0;                               // sequence number of the run's first loaded row
        uint32_t n_c = 0, ph_c = 0;                      // cursor: newest row waited for (seq, slot, phase)
        int t_c = 0;
        uint32_t krow = 0;                               // output row index in the CTA's sequence
        for (int64_t g = g0; g < g1;) {
            const RsSeg s = rs_seg(a, g, g1);
            int rel = s.rlo;                             // next input row whose TMEM slot is handed back
            int t_rel = tb;
            auto release_upto = [&](int rmax) {          // rows <= rmax: no later output row reads them
                if (rel > rmax || rel >= s.rhi) return;
                tc_fence_before();
                __syncwarp();
                for (; rel <= rmax && rel < s.rhi; ++rel) {
                    if (lane == 0) mbar_arrive(&aempty[t_rel]);
                    if (++t_rel == nt) t_rel = 0;
                }
            };
            const int64_t img_el = (int64_t)s.img * a.OH;
            // TMEM slot of input row rb = y - pad_y: (tb + rb - rlo) mod nt, reduced once per run and then
            // advanced by one per output row (a per-row reduction loop of ~(rb - rlo) / nt iterations ran
            // at branch-resolve latency and was the largest item of the epilogue's row time)
            int t0y = tb + (s.ylo - pad_y - s.rlo);
            while (t0y < 0) t0y += nt;
            while (t0y >= nt) t0y -= nt;
            for (int y = s.ylo; y < s.yhi; ++y, ++krow, t0y = (t0y + 1 == nt) ? 0 : t0y + 1) {
                if ((int)(krow & 1u) != gi) continue;
                // debug-only phase timeline of CTA 0, warp 4, output row 4 (OLLIE_RS_DBG bit 2)
                const bool ptr = (a.dbg & 4) && a.trace && blockIdx.x == 0 && warp == 4 && lane == 0 && krow == 4;
                if (ptr) a.trace[256] = clock64();
                const int rb = y - pad_y;                // input row of kernel row 0
                const int rtop = min(rb + R - 1, s.rhi - 1);
                if (rtop >= s.rlo) {                     // D of every row up to rtop is complete (in-order commits)
                    const uint32_t target = seq0 + (uint32_t)(rtop - s.rlo);
                    while (n_c < target) {
                        ++n_c;
                        if (++t_c == nt) { t_c = 0; ph_c ^= 1u; }
                    }
                    mbar_wait(&afull[t_c], ph_c);
                    tc_fence_after();
                }
                if (ptr) a.trace[257] = clock64();
                // TMEM slot of row rb + i: (tb + rb - rlo + i) mod nt (rb - rlo in [-pad_y, ...])
                const int t0 = t0y;
                uint32_t vmask = 0;                      // kernel rows i whose input row rb + i exists
#pragma unroll
                for (int i = 0; i < kRI; ++i)
                    if ((kR > 0 || i < R) && rb + i >= s.rlo && rb + i < s.rhi) vmask |= 1u << i;
                for (int h = 0; h < mtr; ++h) {
                    const uint32_t lanebase = lane0 + (uint32_t)h * acc_cols;
#pragma unroll
                    for (int i = 0; i < kRI; ++i) {
                        int ti = t0 + i;                     // TMEM slot of row rb + i (i < R < nt)
                        if (ti >= nt) ti -= nt;
                        if constexpr (kR > 0) {
                            rs_tmem_ld<kFp>(lanebase + (uint32_t)ti * row_cols + (uint32_t)(i * kFp), &v[i * kFp]);
                        } else {
                            if (i < R && ((vmask >> i) & 1u))
                                rs_tmem_ld<kFp>(lanebase + (uint32_t)ti * row_cols + (uint32_t)(i * kFp), &v[i * kFp]);
                        }
                    }
                    if (ptr) a.trace[260 + 4 * h] = clock64();
                    tmem_ld_wait();
                    if (ptr) a.trace[261 + 4 * h] = clock64();
                    // the row's last TMEM reads are done: hand the slots back before the stores (this
                    // group's next row, y + 2, reads rows >= rb + 2), shortening the MMA <-> epilogue chain
                    if (h == mtr - 1) release_upto(rb + 1);
                    float out[kFp];
#pragma unroll
                    for (int f = 0; f < kFp; ++f) out[f] = 0.f;
#pragma unroll
                    for (int i = 0; i < kRI; ++i) {
                        const bool ok = (vmask >> i) & 1u;   // edge rows: garbage / stale TMEM, selected out
#pragma unroll
                        for (int f = 0; f < kFp; ++f) out[f] += ok ? __uint_as_float(v[i * kFp + f]) : 0.f;
                    }
                    if (ptr) a.trace[262 + 4 * h] = clock64();
                    const int x = 128 * h + xq;              // output column of this lane
                    if (x >= OWc) continue;
                    if (sub == 1) {
                        const int64_t e0 = ((img_el + y) * a.OW + x) * F;
                        if (a.epi.on) epi_apply<!kTF32, kFp>(a.epi, out, e0, 0, F);
                        if (F == kFp) {
                            rs_store_pixel<kTF32, kFp>(a.y, e0, out);
                            if (ptr) a.trace[263 + 4 * h] = clock64();
                        } else {
#pragma unroll
                            for (int f = 0; f < kFp; ++f)
                                if (f < F) rs_store1<kTF32>(a.y, e0 + f, out[f]);
                        }
                    } else {
                        // class (cy, cx) of column x -> output pixel (sigma*y + cy, sigma*x + cx); columns are
                        // ordered (cy, cx, f): walk them with counters (no divisions); neighbouring elements of
                        // one output row that are adjacent in memory leave as one bf16x2 store
                        int cy = 0, cx = 0, f = 0;
                        int64_t rowel = ((img_el + (int64_t)sub * y) * a.OW + (int64_t)sub * x) * F;
                        bool pend = false;                 // element e-1 held back for pairing
                        float pv = 0.f;
                        int64_t pel = 0;
#pragma unroll
                        for (int e = 0; e < kFp; ++e) {
                            const int oy = sub * y + cy, ox = sub * x + cx;
                            const bool okp = oy < a.OH && ox < a.OW;
                            const int64_t el = rowel + (int64_t)cx * F + f;
                            float vv = out[e];
                            if (okp && a.epi.on) epi_apply<!kTF32, 1>(a.epi, &vv, el, f, 1);
                            if constexpr (!kTF32) {
                                if (pend && el == pel + 1 && okp) {
                                    *reinterpret_cast<uint32_t *>(reinterpret_cast<uint16_t *>(a.y) + pel) = pack_bf16x2_rn(pv, vv);
                                    pend = false;
                                } else {
                                    if (pend) rs_store1<false>(a.y, pel, pv);
                                    pend = okp && (el & 1) == 0;
                                    if (pend) { pv = vv; pel = el; }
                                    else if (okp) rs_store1<false>(a.y, el, vv);
                                }
                            } else {
                                if (okp) rs_store1<true>(a.y, el, vv);
                            }
                            if (++f == F) {
                                f = 0;
                                if (++cx == sub) { cx = 0; ++cy; rowel += OWF; }
                            }
                        }
                        if constexpr (!kTF32) {
                            if (pend) rs_store1<false>(a.y, pel, pv);
                        }
                    }
                }
                if (a.trace && blockIdx.x == 0 && lane == 0 && q == 0) {
                    const int64_t kr = (int64_t)(y - s.ylo) + (g - g0);
                    if (kr < 64) a.trace[192 + kr] = rs_gtimer();
                }
            }
            release_upto(s.rhi - 1);
            seq0 += (uint32_t)(s.rhi - s.rlo);
            tb += s.rhi - s.rlo;
            while (tb >= nt) tb -= nt;
            g += s.yhi - s.ylo;
        }
        };
        switch (R) {
            case 1: epilogue(rs_ic<1>{}); break;
            case 3:
                if constexpr (3 * kFp <= RS_MAX_NP) epilogue(rs_ic<3>{});
                else epilogue(rs_ic<0>{});
                break;
            case 5:
                if constexpr (5 * kFp <= RS_MAX_NP) epilogue(rs_ic<5>{});
                else epilogue(rs_ic<0>{});
                break;
            default: epilogue(rs_ic<0>{}); break;
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
