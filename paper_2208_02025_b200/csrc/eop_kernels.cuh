// eop_kernels.cuh -- the memory-bound eOperators of the derived convolution.
//
//  a3  OffsetAdd (E7):
//        Y[b,oh,ow,f] = sum_{i<R,j<S} T[b, oh*st-p+i*d, ow*st-p+j*d, (i*S+j)*F+f]
//      taps whose spatial index leaves [0,H)x[0,W) contribute 0, tested per dimension
//      (reading Q5 -- never on the flattened m = t1*W+t2).
//  a4  ConvTranspose selective addition, dilation 1:
//        Y[b,oh,ow,f] = sum over i = (oh+p) mod st + st*k  (likewise j) of
//                       T[b, (oh+p-i)/st, (ow+p-j)/st, (i*S+j)*F+f]   (in-range rows only)
//  a0  weight DLT (Eq. layout-K) as a tiled smem transpose.
//
// Roofline: HBM.  No data reuse (each T element feeds at most one output),
// so the kernels only need coalescing, 128-bit vectors and enough loads in flight: one
// thread owns VEC consecutive f of one output pixel and issues all its r*s tap loads
// before summing.  Tap order (i, j) is fixed, so results are deterministic.
#pragma once
#include <type_traits>
#include "sm100_ptx.cuh"
#include "epilogue.cuh"

namespace ollie {

struct OffsetAddArgs {
    const float *T;
    int64_t ldT;               // row stride of T (elements)
    void *y;
    int64_t n, h, w, f, r, s;
    int64_t oh, ow;
    int32_t pad, stride, dil;
    int64_t items;             // n*oh*ow*(f/VEC)
    EpiArgs epi;               // NEXT-3 element-wise epilogue
};

__device__ __forceinline__ float4 ld_stream_f4(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream_f1(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

template <int VEC, bool kOutBF16>
__device__ __forceinline__ void store_y(void *y, int64_t off, const float (&acc)[VEC]) {
    if constexpr (kOutBF16) {
        uint16_t *yp = reinterpret_cast<uint16_t *>(y) + off;
        if constexpr (VEC == 4) {
            uint2 pk;
            pk.x = (uint32_t)float_to_bf16_rne(acc[0]) | ((uint32_t)float_to_bf16_rne(acc[1]) << 16);
            pk.y = (uint32_t)float_to_bf16_rne(acc[2]) | ((uint32_t)float_to_bf16_rne(acc[3]) << 16);
            *reinterpret_cast<uint2 *>(yp) = pk;
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) yp[v] = float_to_bf16_rne(acc[v]);
        }
    } else {
        float *yp = reinterpret_cast<float *>(y) + off;
        if constexpr (VEC == 4)
            *reinterpret_cast<float4 *>(yp) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) yp[v] = acc[v];
        }
    }
}

template <int VEC>
__device__ __forceinline__ void accum_tap(float (&acc)[VEC], const float *src) {
    if constexpr (VEC == 4) {
        float4 t = ld_stream_f4(src);
        acc[0] += t.x; acc[1] += t.y; acc[2] += t.z; acc[3] += t.w;
    } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] += ld_stream_f1(src + v);
    }
}

// a3: OffsetAdd.  Taps are issued in (i, j) order; out-of-image taps are skipped.  Index
// decoding is 32-bit (IDX = int32_t) whenever the host proves every index fits.
template <int VEC, bool kOutBF16, typename IDX>
__global__ void __launch_bounds__(256) offset_add_kernel(OffsetAddArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const IDX fv_per_px = (IDX)(a.f / VEC);
    const IDX OW = (IDX)a.ow, OHh = (IDX)a.oh;
    for (IDX it = (IDX)(blockIdx.x * blockDim.x + threadIdx.x); it < (IDX)a.items; it += (IDX)(gridDim.x * blockDim.x)) {
        const IDX px = it / fv_per_px;
        const int64_t fv = it - px * fv_per_px;
        const IDX t = px / OW;
        const int64_t ow = px - t * OW;
        const IDX b_ = t / OHh;
        const int64_t oh = t - b_ * OHh;
        const int64_t b = b_;
        float acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
        const int64_t h0 = oh * a.stride - a.pad, w0 = ow * a.stride - a.pad;
        const float *Tb = a.T + (b * a.h) * a.w * a.ldT + fv * VEC;
        if (VEC == 4 && a.r == 3 && a.s == 3) {
            // 3x3: issue all nine (predicated) 16-byte loads before summing, in (i, j) order
            float4 tv[9];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int64_t t1 = h0 + i * a.dil, t2 = w0 + j * a.dil;
                    const bool in = t1 >= 0 && t1 < a.h && t2 >= 0 && t2 < a.w;
                    tv[i * 3 + j] = in ? ld_stream_f4(Tb + (t1 * a.w + t2) * a.ldT + (i * 3 + j) * a.f)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                acc[0] += tv[q].x;
                if constexpr (VEC == 4) { acc[1] += tv[q].y; acc[2] += tv[q].z; acc[3] += tv[q].w; }
            }
            if (a.epi.on) epi_apply<kOutBF16, VEC>(a.epi, acc, px * a.f + fv * VEC, (int)(fv * VEC), VEC);
            store_y<VEC, kOutBF16>(a.y, px * a.f + fv * VEC, acc);
            continue;
        }
        for (int64_t i = 0; i < a.r; ++i) {
            const int64_t t1 = h0 + i * a.dil;
            if (t1 < 0 || t1 >= a.h) continue;
            const float *Trow = Tb + t1 * a.w * a.ldT + i * a.s * a.f;
#pragma unroll 3
            for (int64_t j = 0; j < a.s; ++j) {
                const int64_t t2 = w0 + j * a.dil;
                if (t2 < 0 || t2 >= a.w) continue;
                accum_tap<VEC>(acc, Trow + t2 * a.ldT + j * a.f);
            }
        }
        if (a.epi.on) epi_apply<kOutBF16, VEC>(a.epi, acc, px * a.f + fv * VEC, (int)(fv * VEC), VEC);
        store_y<VEC, kOutBF16>(a.y, px * a.f + fv * VEC, acc);
    }
}

// a4: ConvTranspose selective addition (dilation 1).  Only the taps i == (oh+p) mod st
// (mod st) are visited: each output reads exactly the Matmul outputs that land on it.
template <int VEC, bool kOutBF16, typename IDX>
__global__ void __launch_bounds__(256) selective_add_kernel(OffsetAddArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const IDX fv_per_px = (IDX)(a.f / VEC);
    const IDX OW = (IDX)a.ow, OHh = (IDX)a.oh;
    const int64_t st = a.stride;
    for (IDX it = (IDX)(blockIdx.x * blockDim.x + threadIdx.x); it < (IDX)a.items; it += (IDX)(gridDim.x * blockDim.x)) {
        const IDX px = it / fv_per_px;
        const int64_t fv = it - px * fv_per_px;
        const IDX t = px / OW;
        const int64_t ow = px - t * OW;
        const IDX b_ = t / OHh;
        const int64_t oh = t - b_ * OHh;
        const int64_t b = b_;
        float acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
        const int64_t th = oh + a.pad, tw = ow + a.pad;
        const float *Tb = a.T + (b * a.h) * a.w * a.ldT + fv * VEC;
        if (VEC == 4 && a.r <= 2 * st && a.s <= 2 * st) {
            // at most 2 x 2 selected taps (4x4 / 3x3 kernels at stride 2): issue the four
            // predicated 16-byte loads before summing, in the same (i, j) order as below
            float4 tv[4];
            const int64_t i0 = th % st, j0 = tw % st;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t i = i0 + (q >> 1) * st, j = j0 + (q & 1) * st;
                const int64_t ih = (th - i) / st, iw = (tw - j) / st;
                const bool in = i < a.r && i <= th && ih < a.h && j < a.s && j <= tw && iw < a.w;
                tv[q] = in ? ld_stream_f4(Tb + (ih * a.w + iw) * a.ldT + (i * a.s + j) * a.f)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc[0] += tv[q].x;
                if constexpr (VEC == 4) { acc[1] += tv[q].y; acc[2] += tv[q].z; acc[3] += tv[q].w; }
            }
            if (a.epi.on) epi_apply<kOutBF16, VEC>(a.epi, acc, px * a.f + fv * VEC, (int)(fv * VEC), VEC);
            store_y<VEC, kOutBF16>(a.y, px * a.f + fv * VEC, acc);
            continue;
        }
        // th = oh + p >= 0, so th % st is the smallest selected kernel row; rows past th
        // would need a negative input row, and the input row falls as i grows.
        for (int64_t i = th % st; i < a.r && i <= th; i += st) {
            const int64_t ih = (th - i) / st;
            if (ih >= a.h) continue;
            const float *Trow = Tb + ih * a.w * a.ldT + i * a.s * a.f;
            for (int64_t j = tw % st; j < a.s && j <= tw; j += st) {
                const int64_t iw = (tw - j) / st;
                if (iw >= a.w) continue;
                accum_tap<VEC>(acc, Trow + iw * a.ldT + j * a.f);
            }
        }
        if (a.epi.on) epi_apply<kOutBF16, VEC>(a.epi, acc, px * a.f + fv * VEC, (int)(fv * VEC), VEC);
        store_y<VEC, kOutBF16>(a.y, px * a.f + fv * VEC, acc);
    }
}

// OLLIE_PLAN_SMALL: the fused derived program on CUDA cores, one thread per output element
// (b, oh, ow, f) -- Y[m, f] = Sum_{i,j} Sum_c X[m + Delta_ij, c] W'[(i*S+j)*F + f, c], taps in (i, j)
// order (Conv2d: in-image taps; ConvTranspose2d, dilation 1: the selected taps i = (oh+p) mod st
// + st*k of the selective addition), channels in order, fp32.  For layers of a few thousand
// outputs, where the tensor-core kernels' setup (barriers, TMEM, TMA descriptors) dominates.
struct SmallConvArgs {
    const void *x, *w;           // NHWC input, W' [(i*S+j)*F + f][C]
    void *y;
    int32_t n, H, W, C, F, R, S, pad, st, dil, OH, OW;
    int64_t items;               // n * OH * OW * F
    EpiArgs epi;
};

template <bool kF32, bool kTr>
__global__ void __launch_bounds__(256) small_conv_kernel(const __grid_constant__ SmallConvArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < a.items; it += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)(it % a.F);
        int64_t px = it / a.F;
        const int ow = (int)(px % a.OW);
        const int64_t t = px / a.OW;
        const int oh = (int)(t % a.OH);
        const int64_t b = t / a.OH;
        float acc = 0.f;
        for (int i = 0; i < a.R; ++i) {
            int ih;
            if constexpr (kTr) {
                const int th = oh + a.pad - i;
                if (th < 0 || th % a.st) continue;
                ih = th / a.st;
            } else {
                ih = oh * a.st - a.pad + i * a.dil;
            }
            if (ih < 0 || ih >= a.H) continue;
            for (int j = 0; j < a.S; ++j) {
                int iw;
                if constexpr (kTr) {
                    const int tw = ow + a.pad - j;
                    if (tw < 0 || tw % a.st) continue;
                    iw = tw / a.st;
                } else {
                    iw = ow * a.st - a.pad + j * a.dil;
                }
                if (iw < 0 || iw >= a.W) continue;
                const int64_t xo = ((b * a.H + ih) * a.W + iw) * a.C;
                const int64_t wo = ((int64_t)(i * a.S + j) * a.F + f) * a.C;
                if constexpr (kF32) {
                    const float *xp = reinterpret_cast<const float *>(a.x) + xo;
                    const float *wq = reinterpret_cast<const float *>(a.w) + wo;
                    for (int c = 0; c < a.C; ++c) acc = fmaf(__ldg(xp + c), __ldg(wq + c), acc);
                } else {
                    const uint16_t *xp = reinterpret_cast<const uint16_t *>(a.x) + xo;
                    const uint16_t *wq = reinterpret_cast<const uint16_t *>(a.w) + wo;
                    for (int c = 0; c < a.C; ++c)
                        acc = fmaf(bf16_bits_to_float(__ldg(xp + c)), bf16_bits_to_float(__ldg(wq + c)), acc);
                }
            }
        }
        float v[1] = {acc};
        if (a.epi.on) epi_apply<!kF32, 1>(a.epi, v, it, f, 1);
        if constexpr (kF32) reinterpret_cast<float *>(a.y)[it] = v[0];
        else reinterpret_cast<uint16_t *>(a.y)[it] = float_to_bf16_rne(v[0]);
    }
}

// GEMM_RED plan, last step: Y = epilogue(acc) in Y's dtype (acc is the fp32 sum the GEMM's
// reductions produced; 4 channels per thread).
template <bool kOutBF16>
__global__ void __launch_bounds__(256) red_finish_kernel(const float *__restrict__ acc, void *y, int64_t n4, int32_t F,
                                                         EpiArgs epi) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 s4 = *reinterpret_cast<const float4 *>(acc + 4 * i);
        float v[4] = {s4.x, s4.y, s4.z, s4.w};
        if (epi.on) epi_apply<kOutBF16, 4>(epi, v, 4 * i, (int)((4 * i) % F), 4);
        store_y<4, kOutBF16>(y, 4 * i, v);
    }
}

// a0: weight DLT  wp[(ij)*F + f][c] = src[f*sz + c*sc + ij]   (ij = i*S+j)
//   Conv2d  W[f][c][i][j]: sz = C*RS, sc = RS;   ConvT W[c][f][i][j]: sz = RS, sc = F*RS.
// Per f a [C x RS] -> [RS x C] transpose through a 32x33 smem tile; pure data movement.
template <typename E>
__global__ void __launch_bounds__(256) weight_dlt_kernel(const E *__restrict__ src, E *__restrict__ dst, int64_t F,
                                                         int64_t C, int64_t RS, int64_t sz, int64_t sc) {
    // no early trigger: kernels after this one may load the prepared weights before their own
    // griddepcontrol.wait (fused_conv), so they must not start until W' is complete
    pdl_wait();
    __shared__ E tile[32][33];
    const int64_t f = blockIdx.z;
    const int64_t c0 = (int64_t)blockIdx.y * 32, ij0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, ij = ij0 + tx;
        if (c < C && ij < RS) tile[k][tx] = src[f * sz + c * sc + ij];
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t ij = ij0 + k, c = c0 + tx;
        if (c < C && ij < RS) dst[(ij * F + f) * C + c] = tile[tx][k];
    }
}

// a7 instance: the im2col ("tap folding") layout eOperator of a Conv2d -- variable substitution of
// E1 that moves the taps into the Matmul's reduction index (operator matching):
//     A'[b, oy, ox, k] = X[b, oy*st - p + i*d, ox*st - p + j*d, c],   k = (i*S + j)*C + c < R*S*C
// zero outside the image and for R*S*C <= k < KP.  A layer with few channels (FSRCNN's
// c = 1 feature extraction) then runs as a 1x1 conv over KP-wide pixels instead of r*s taps that
// each use one channel of a 16-wide MMA K.  One thread writes one 16-byte chunk of one output pixel
// (coalesced stores, the HBM-bound side); the r*s gathered reads hit L1 / L2 (every input pixel is
// read by r*s neighbours).
struct TapFoldArgs {
    const void *x;
    void *out;
    int32_t H, W, C, R, S, pad, st, dil, OH, OW, KP, RSC;
    int64_t items;             // n * OH * OW * (KP / VE)
};

template <bool kF32, typename I>
__global__ void __launch_bounds__(256) tap_fold_kernel(TapFoldArgs a) {
    constexpr int VE = kF32 ? 4 : 8;                 // elements per 16-byte chunk
    using E = typename std::conditional<kF32, uint32_t, uint16_t>::type;
    pdl_wait();                                      // X may be written by the previous kernel
    const E *x = reinterpret_cast<const E *>(a.x);
    const I chunks = (I)(a.KP / VE);
    const I stride = (I)gridDim.x * blockDim.x;
    for (I it = (I)blockIdx.x * blockDim.x + threadIdx.x; it < (I)a.items; it += stride) {
        const I kc = it % chunks;
        I pix = it / chunks;
        const int ox = (int)(pix % a.OW);
        pix /= a.OW;
        const int oy = (int)(pix % a.OH);
        const I b = pix / a.OH;
        // (i, j, c) of the chunk's first k, then walked incrementally
        const int k0 = (int)kc * VE;
        int c = k0 % a.C, tap = k0 / a.C;
        int j = tap % a.S, i = tap / a.S;
        E v[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            E val = 0;
            if (k0 + e < a.RSC) {
                const int iy = oy * a.st - a.pad + i * a.dil, ix = ox * a.st - a.pad + j * a.dil;
                if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W)
                    val = __ldg(x + (((int64_t)b * a.H + iy) * a.W + ix) * a.C + c);
                if (++c == a.C) {
                    c = 0;
                    if (++j == a.S) { j = 0; ++i; }
                }
            }
            v[e] = val;
        }
        uint4 pk;
        if constexpr (kF32) {
            pk = make_uint4(v[0], v[1], v[2], v[3]);
        } else {
            pk = make_uint4((uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16),
                            (uint32_t)v[4] | ((uint32_t)v[5] << 16), (uint32_t)v[6] | ((uint32_t)v[7] << 16));
        }
        *reinterpret_cast<uint4 *>(reinterpret_cast<E *>(a.out) + (int64_t)it * VE) = pk;
    }
}

// Row-tiled form: one CTA per output row (b, oy) stages the r input rows the row reads
// (oy*st - p + i*d, zero outside the image) in shared memory, then writes the row's OW * KP outputs
// as consecutive 16-byte chunks (lane t -> chunk t: fully coalesced stores).  The staged rows carry
// zero halo columns on both sides (row pitch rpitch elements, image column 0 at element `roff`,
// 16-byte aligned) and one zero cell past the last row, so an output element is ONE shared-memory
// read at addr_e + ox * step_e with no bounds test: a thread's k-chunk is fixed, (addr_e, step_e) are
// decoded once (k >= r*s*c: the zero cell, step 0).  ncu on the earlier form (per-element bounds
// tests, a division per staged element): 227 instructions per 16-byte output chunk, issue-bound.
struct TapFoldRows {
    int32_t roff, rpitch;       // image column 0 of a staged row (elements, multiple of 16 bytes); row pitch
    int32_t zcell;              // element index of the zero cell
    int32_t vec;                // 1: staged rows are filled with 16-byte loads / stores
};

template <bool kF32>
__global__ void __launch_bounds__(256) tap_fold_rows_kernel(TapFoldArgs a, TapFoldRows g) {
    constexpr int VE = kF32 ? 4 : 8;
    using E = typename std::conditional<kF32, uint32_t, uint16_t>::type;
    extern __shared__ uint8_t tf_smem[];
    E *rows = reinterpret_cast<E *>(tf_smem);        // [R][rpitch] + the zero cell
    pdl_wait();
    const E *x = reinterpret_cast<const E *>(a.x);
    const int WC = a.W * a.C;
    const int cpp = a.KP / VE;                       // 16-byte chunks per output pixel
    const int chunks = a.OW * cpp;
    int addr[VE], step[VE];
    {
        const int k0 = (threadIdx.x % cpp) * VE;
        int c = k0 % a.C, tap = k0 / a.C;
        int j = tap % a.S, i = tap / a.S;
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            const bool kv = k0 + e < a.RSC;
            addr[e] = kv ? i * g.rpitch + g.roff + (j * a.dil - a.pad) * a.C + c : g.zcell;
            step[e] = kv ? a.st * a.C : 0;
            if (++c == a.C) {
                c = 0;
                if (++j == a.S) { j = 0; ++i; }
            }
        }
    }
    // the halo columns and the zero cell are never written with data: zero them once
    for (int t = threadIdx.x; t < a.R * g.rpitch + 1; t += blockDim.x) {
        const int col = t % g.rpitch;
        if (t == g.zcell || col < g.roff || col >= g.roff + WC) rows[t] = (E)0;
    }
    for (int64_t row = blockIdx.x; row < a.items; row += gridDim.x) {   // items = n * OH output rows
        const int oy = (int)(row % a.OH);
        const int64_t b = row / a.OH;
        __syncthreads();                             // the previous row's readers are done
        for (int i = 0; i < a.R; ++i) {
            const int iy = oy * a.st - a.pad + i * a.dil;
            const bool in = iy >= 0 && iy < a.H;
            E *dst = rows + i * g.rpitch + g.roff;
            const E *src = x + (b * a.H + iy) * (int64_t)WC;
            if (g.vec) {
                for (int t = threadIdx.x; t < WC / VE; t += blockDim.x)
                    reinterpret_cast<uint4 *>(dst)[t] = in ? __ldg(reinterpret_cast<const uint4 *>(src) + t) : make_uint4(0, 0, 0, 0);
            } else {
                for (int t = threadIdx.x; t < WC; t += blockDim.x) dst[t] = in ? __ldg(src + t) : (E)0;
            }
        }
        __syncthreads();
        E *orow = reinterpret_cast<E *>(a.out) + row * (int64_t)a.OW * a.KP;
        for (int ch = threadIdx.x; ch < chunks; ch += blockDim.x) {
            const int ox = ch / cpp;
            E v[VE];
#pragma unroll
            for (int e = 0; e < VE; ++e) v[e] = rows[addr[e] + ox * step[e]];
            uint4 pk;
            if constexpr (kF32) pk = make_uint4(v[0], v[1], v[2], v[3]);
            else
                pk = make_uint4((uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16),
                                (uint32_t)v[4] | ((uint32_t)v[5] << 16), (uint32_t)v[6] | ((uint32_t)v[7] << 16));
            *reinterpret_cast<uint4 *>(orow + (int64_t)ch * VE) = pk;
        }
    }
}

}  // namespace ollie
