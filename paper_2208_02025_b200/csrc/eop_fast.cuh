// eop_fast.cuh -- fast paths of the eOperator evaluator for PURE-INDEXING AFFINE eOperators
// (one input, no summation, body = the access, every index term a plain iterator):
// layout transforms (DLT), channel pads, reshapes.  Such an eOp is
//     out[o] = in[B + sum_d s_d * o_d]   if every input index b_k + sum_d a_kd * o_d is inside
//                                         the tensor, else 0 (pad band)
// over the dense output coordinates o.  HBM-bound: bytes = |in| + |out|.
//  - gather kernel: one thread per 8 consecutive elements of an output row (innermost output
//    dimension), 32-bit index math after collapsing output dims that merge linearly, bounds tests
//    only on input dims that have a pad band, 16-byte stores; reads are coalesced across the warp
//    when the innermost output dimension has input stride 1 (pads, reshapes).
//  - transpose kernel: when the innermost output dimension is strided in the input, a 32x32 tile
//    of (input-contiguous dim, output-contiguous dim) goes through shared memory so both the
//    reads and the writes are coalesced (NCHW <-> NHWC).
#pragma once
#include <type_traits>
#include "sm100_ptx.cuh"

namespace ollie {

constexpr int FAST_MAX_D = 6;

struct AffineEop {
    const void *in;
    void *out;
    int32_t in_bf16, out_bf16;
    int32_t nd_out, nd_in;
    int32_t w[FAST_MAX_D];                  // output widths (dense, traversal order)
    int32_t s[FAST_MAX_D];                  // input element stride per output dim
    int32_t a[FAST_MAX_D][FAST_MAX_D];      // a[k][d]: coefficient of output dim d in input index k
    int32_t b[FAST_MAX_D];                  // input index k at o = 0
    int32_t shape[FAST_MAX_D];              // input extents
    int32_t base;                           // input linear offset at o = 0 (may be negative: pad band)
    int32_t rows;                           // product of all output widths but the last
    int32_t inner;                          // last output width
    // transpose kernel: output dim dt (input stride 1) and the innermost output dim
    int32_t dt;
    int32_t chk;                            // bit k: input dim k has a pad band (needs a bounds test)
};

__device__ __forceinline__ float fast_ld(const AffineEop &e, int32_t off) {
    if (e.in_bf16) return bf16_bits_to_float(__ldg(reinterpret_cast<const uint16_t *>(e.in) + off));
    return __ldg(reinterpret_cast<const float *>(e.in) + off);
}
__device__ __forceinline__ void fast_st(const AffineEop &e, int64_t off, float v) {
    if (e.out_bf16) reinterpret_cast<uint16_t *>(e.out)[off] = float_to_bf16_rne(v);
    else reinterpret_cast<float *>(e.out)[off] = v;
}

__device__ __forceinline__ int32_t fdiv32(int32_t a, int32_t b) {   // floor(a / b), b != 0
    int32_t q = a / b;
    return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ int32_t cdiv32(int32_t a, int32_t b) { return -fdiv32(-a, b); }   // ceil(a / b)

// Raw element move (dtypes equal): bits are copied, zero is the all-zero pattern.
template <typename E>
__device__ __forceinline__ E raw_ld(const void *p, int32_t off) { return __ldg(reinterpret_cast<const E *>(p) + off); }

// VEC consecutive inner elements per thread, 32-bit index math (the host guarantees every
// extent and offset fits), outer coordinates decoded once per thread.  Input dims with a pad
// band (bit k of `chk`) are affine in the inner coordinate j, so each thread turns them into one
// valid interval [jlo, jhi) before touching memory.  E = element type when in/out dtypes match
// (raw bit copy); E = void converts through fp32.
template <int VEC, typename E>
__global__ void __launch_bounds__(256) eop_affine_gather_kernel(const __grid_constant__ AffineEop e) {
    pdl_launch_dependents();
    pdl_wait();
    const int32_t vec_per_row = (e.inner + VEC - 1) / VEC;
    const int32_t total = e.rows * vec_per_row;
    const int dl = e.nd_out - 1;
    for (int32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < total; it += gridDim.x * blockDim.x) {
        const int32_t row0 = it / vec_per_row;
        const int32_t j0 = (it - row0 * vec_per_row) * VEC;
        int32_t row = row0;
        int32_t off = e.base;
        int32_t idx[FAST_MAX_D];
#pragma unroll
        for (int k = 0; k < FAST_MAX_D; ++k) idx[k] = e.b[k];
        for (int d = e.nd_out - 2; d >= 0; --d) {
            const int32_t q = row / e.w[d];
            const int32_t od = row - q * e.w[d];
            row = q;
            off += e.s[d] * od;
#pragma unroll
            for (int k = 0; k < FAST_MAX_D; ++k) idx[k] += e.a[k][d] * od;
        }
        int32_t jlo = 0, jhi = e.inner;
        if (e.chk) {
#pragma unroll
            for (int k = 0; k < FAST_MAX_D; ++k)
                if (e.chk & (1 << k)) {
                    const int32_t c = e.a[k][dl], b = idx[k], n = e.shape[k];
                    if (c == 0) {
                        if (b < 0 || b >= n) jhi = 0;
                    } else if (c == 1) {                 // the common cases, division-free
                        jlo = max(jlo, -b);
                        jhi = min(jhi, n - b);
                    } else if (c == -1) {
                        jlo = max(jlo, b - n + 1);
                        jhi = min(jhi, b + 1);
                    } else if (c > 0) {
                        jlo = max(jlo, cdiv32(-b, c));
                        jhi = min(jhi, fdiv32(n - 1 - b, c) + 1);
                    } else {
                        jlo = max(jlo, cdiv32(n - 1 - b, c));
                        jhi = min(jhi, fdiv32(-b, c) + 1);
                    }
                }
        }
        const int32_t sl = e.s[dl];
        const int64_t obase = (int64_t)row0 * e.inner + j0;
        if constexpr (!std::is_void<E>::value) {
            E v[VEC];
            const E *src = reinterpret_cast<const E *>(e.in) + (off + j0);
            if (VEC * sizeof(E) == 16 && sl == 1 && j0 >= jlo && j0 + VEC <= jhi &&
                (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                // contiguous, in-bounds, aligned: one 16-byte load (layout DLTs, space <-> batch)
                const uint4 pk = __ldg(reinterpret_cast<const uint4 *>(src));
                memcpy(v, &pk, 16);
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    const int32_t j = j0 + q;
                    v[q] = (j >= jlo && j < jhi) ? raw_ld<E>(e.in, off + sl * j) : E(0);
                }
            }
            E *o = reinterpret_cast<E *>(e.out) + obase;
            if (j0 + VEC <= e.inner && ((obase * (int64_t)sizeof(E)) & 15) == 0 && VEC * sizeof(E) == 16) {
                uint4 pk;
                memcpy(&pk, v, 16);
                *reinterpret_cast<uint4 *>(o) = pk;
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                    if (j0 + q < e.inner) o[q] = v[q];
            }
        } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const int32_t j = j0 + q;
                if (j < e.inner) fast_st(e, obase + q, (j >= jlo && j < jhi) ? fast_ld(e, off + sl * j) : 0.f);
            }
        }
    }
}

// Narrow output rows (inner <= 64 elements, same dtype in and out): one thread per output row,
// one decode per row, the row's input run read element by element inside its valid interval and
// written back as 16-byte vectors (channel pads / crops of NHWC rows: FSRCNN's 1 -> 16, 12 -> 16).
// Row decode + valid interval of the innermost output dim (shared by the row kernels).
__device__ __forceinline__ void affine_row(const AffineEop &e, int32_t row, int32_t &off, int32_t &jlo, int32_t &jhi) {
    const int dl = e.nd_out - 1;
    off = e.base;
    int32_t idx[FAST_MAX_D];
#pragma unroll
    for (int k = 0; k < FAST_MAX_D; ++k) idx[k] = e.b[k];
    for (int d = e.nd_out - 2; d >= 0; --d) {
        const int32_t q = row / e.w[d];
        const int32_t od = row - q * e.w[d];
        row = q;
        off += e.s[d] * od;
#pragma unroll
        for (int k = 0; k < FAST_MAX_D; ++k) idx[k] += e.a[k][d] * od;
    }
    jlo = 0;
    jhi = e.inner;
    if (e.chk) {
#pragma unroll
        for (int k = 0; k < FAST_MAX_D; ++k)
            if (e.chk & (1 << k)) {
                const int32_t c = e.a[k][dl], b = idx[k], n = e.shape[k];
                if (c == 0) {
                    if (b < 0 || b >= n) jhi = 0;
                } else if (c == 1) {
                    jlo = max(jlo, -b);
                    jhi = min(jhi, n - b);
                } else if (c == -1) {
                    jlo = max(jlo, b - n + 1);
                    jhi = min(jhi, b + 1);
                } else if (c > 0) {
                    jlo = max(jlo, cdiv32(-b, c));
                    jhi = min(jhi, fdiv32(n - 1 - b, c) + 1);
                } else {
                    jlo = max(jlo, cdiv32(n - 1 - b, c));
                    jhi = min(jhi, fdiv32(-b, c) + 1);
                }
            }
    }
}

template <typename E>
__global__ void __launch_bounds__(256) eop_affine_rows_kernel(const __grid_constant__ AffineEop e) {
    pdl_launch_dependents();
    pdl_wait();
    constexpr int VEC = 16 / (int)sizeof(E);
    const int dl = e.nd_out - 1;
    const int nvec = (e.inner + VEC - 1) / VEC;
    for (int32_t row0 = blockIdx.x * blockDim.x + threadIdx.x; row0 < e.rows; row0 += gridDim.x * blockDim.x) {
        int32_t off, jlo, jhi;
        affine_row(e, row0, off, jlo, jhi);
        const int32_t sl = e.s[dl];
        const E *src = reinterpret_cast<const E *>(e.in) + off;
        E *o = reinterpret_cast<E *>(e.out) + (int64_t)row0 * e.inner;
        const bool vec_ok = (e.inner % VEC) == 0;    // rows start 16-byte aligned (host: out aligned)
        for (int vv = 0; vv < nvec; ++vv) {
            E v[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const int32_t j = vv * VEC + q;
                v[q] = (j >= jlo && j < jhi) ? __ldg(src + sl * j) : E(0);
            }
            if (vec_ok) {
                uint4 pk;
                memcpy(&pk, v, 16);
                *reinterpret_cast<uint4 *>(o + vv * VEC) = pk;
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                    if (vv * VEC + q < e.inner) o[vv * VEC + q] = v[q];
            }
        }
    }
}

// Staged narrow rows (channel pads / crops of NHWC rows: FSRCNN's 1 -> 16, 12 -> 16): two collapsed
// output dims [rows][inner], input row r at base + r * s0 (s0 <= 128 bytes), every row's valid column
// interval [jlo, jhi) the same.  A block moves kR rows per pass: the contiguous input span of those rows
// comes in with 16-byte loads (when aligned) into shared memory, the kR * inner outputs leave as
// consecutive 16-byte stores (one chunk per thread, fully coalesced on both sides).  The one-thread-
// per-row kernel above wrote each row's 32 bytes as two strided 16-byte stores and read its elements
// one by one.
template <typename E>
__global__ void __launch_bounds__(256) eop_staged_rows_kernel(const __grid_constant__ AffineEop e, int32_t jlo, int32_t jhi,
                                                             int32_t kR, int32_t vec_in) {
    pdl_launch_dependents();
    pdl_wait();
    constexpr int VE = 16 / (int)sizeof(E);
    extern __shared__ uint8_t st_smem[];
    E *sm = reinterpret_cast<E *>(st_smem);
    const int32_t s0 = e.s[0], inner = e.inner, cpr = inner / VE;
    const E *in = reinterpret_cast<const E *>(e.in);
    E *out = reinterpret_cast<E *>(e.out);
    for (int32_t row0 = blockIdx.x * kR; row0 < e.rows; row0 += gridDim.x * kR) {
        const int32_t nr = min(kR, e.rows - row0);
        const int32_t span = (nr - 1) * s0 + jhi;               // input elements the pass reads
        const E *src = in + e.base + (int64_t)row0 * s0;
        __syncthreads();                                         // the previous pass's readers are done
        if (vec_in) {
            for (int32_t t = threadIdx.x; t < (span + VE - 1) / VE; t += blockDim.x)
                reinterpret_cast<uint4 *>(sm)[t] = __ldg(reinterpret_cast<const uint4 *>(src) + t);
        } else {
            for (int32_t t = threadIdx.x; t < span; t += blockDim.x) sm[t] = __ldg(src + t);
        }
        __syncthreads();
        E *dst = out + (int64_t)row0 * inner;
        for (int32_t q = threadIdx.x; q < nr * cpr; q += blockDim.x) {
            const int32_t r = q / cpr, j0 = (q - r * cpr) * VE;
            E v[VE];
#pragma unroll
            for (int k = 0; k < VE; ++k) {
                const int32_t j = j0 + k;
                v[k] = (j >= jlo && j < jhi) ? sm[r * s0 + j] : E(0);
            }
            uint4 pk;
            memcpy(&pk, v, 16);
            reinterpret_cast<uint4 *>(dst)[q] = pk;
        }
    }
}

// Tiled transpose: the output's innermost dim (dl) is strided in the input and dim dt has input
// stride 1.  A block moves a 32 (dt) x 128 (dl) strip as four 32 x 32 tiles through shared
// memory, so both the reads (along dt) and the writes (along dl) are coalesced; same-dtype moves
// copy raw bits.  No pad band (checked on the host).  grid.x = strips, grid.y = other dims.
template <typename E>
__global__ void __launch_bounds__(256) eop_affine_transpose_kernel(const __grid_constant__ AffineEop e) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ E tile[32][33];
    const int dl = e.nd_out - 1, dt = e.dt;
    const int32_t ns_l = (e.w[dl] + 127) / 128;
    const int32_t sl = (int32_t)(blockIdx.x % ns_l), tt = (int32_t)(blockIdx.x / ns_l);
    int32_t rest = (int32_t)blockIdx.y;
    int32_t off = e.base;
    int64_t obase = 0, ostride = 1;
    int64_t ostr[FAST_MAX_D];
    for (int d = e.nd_out - 1; d >= 0; --d) {
        ostr[d] = ostride;
        ostride *= e.w[d];
    }
    for (int d = e.nd_out - 1; d >= 0; --d) {
        if (d == dl || d == dt) continue;
        const int32_t q = rest / e.w[d];
        const int32_t od = rest - q * e.w[d];
        rest = q;
        off += e.s[d] * od;
        obase += ostr[d] * od;
    }
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const E *in = reinterpret_cast<const E *>(e.in);
    E *out = reinterpret_cast<E *>(e.out);
    for (int sub = 0; sub < 4; ++sub) {
        const int32_t l0 = sl * 128 + sub * 32;
        if (l0 >= e.w[dl]) break;
        for (int r = ty; r < 32; r += 8) {           // read: coalesced along dt (input stride 1)
            const int32_t ol = l0 + r, ot = tt * 32 + tx;
            if (ol < e.w[dl] && ot < e.w[dt]) tile[r][tx] = __ldg(in + off + e.s[dl] * ol + ot);
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {           // write: coalesced along dl (output stride 1)
            const int32_t ot = tt * 32 + r, ol = l0 + tx;
            if (ol < e.w[dl] && ot < e.w[dt]) out[obase + ostr[dt] * ot + ol] = tile[tx][r];
        }
        __syncthreads();
    }
}

// 2-byte transpose with 16-byte global accesses: a block moves a 64 (dt) x TL (dl) tile, TL = 64 or
// 128.  Reads: 8 lanes cover one 128-byte run along dt (input stride 1) with uint4 loads, TL / 32
// runs per thread in flight; writes: TL / 8 lanes cover one output run along dl (output stride 1)
// with uint4 stores; the tile goes through shared memory as 16-bit elements (row pitch TL + 2 halves
// the bank conflicts of the column gathers).  Used when both dims are multiples of 8 and both base
// offsets are 16-byte aligned (host-checked); TL = 128 when the dl extent is a multiple of 128 (four
// loads in flight per thread instead of two: E-b NCHW -> NHWC).
template <int TL>
__global__ void __launch_bounds__(256) eop_affine_transpose16_kernel(const __grid_constant__ AffineEop e) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ uint16_t tile[64][TL + 2];
    const int dl = e.nd_out - 1, dt = e.dt;
    const int32_t ns_l = (e.w[dl] + TL - 1) / TL;
    const int32_t sl = (int32_t)(blockIdx.x % ns_l), tt = (int32_t)(blockIdx.x / ns_l);
    int32_t rest = (int32_t)blockIdx.y;
    int32_t off = e.base;
    int64_t obase = 0, ostride = 1;
    int64_t ostr[FAST_MAX_D];
    for (int d = e.nd_out - 1; d >= 0; --d) {
        ostr[d] = ostride;
        ostride *= e.w[d];
    }
    for (int d = e.nd_out - 1; d >= 0; --d) {
        if (d == dl || d == dt) continue;
        const int32_t q = rest / e.w[d];
        const int32_t od = rest - q * e.w[d];
        rest = q;
        off += e.s[d] * od;
        obase += ostr[d] * od;
    }
    const uint16_t *in = reinterpret_cast<const uint16_t *>(e.in);
    uint16_t *out = reinterpret_cast<uint16_t *>(e.out);
    const int32_t l0 = sl * TL, t0 = tt * 64;
    {
        const int c8 = threadIdx.x & 7, r = threadIdx.x >> 3;     // 8 lanes x 16 B = one 128-byte run; 32 runs
        uint4 v[TL / 32];
#pragma unroll
        for (int h = 0; h < TL / 32; ++h) {                     // read TL runs along dt: rows ol = l0 + rr
            const int rr = r + 32 * h;
            const int32_t ol = l0 + rr, ot = t0 + 8 * c8;
            v[h] = make_uint4(0, 0, 0, 0);
            if (ol < e.w[dl] && ot < e.w[dt]) v[h] = __ldg(reinterpret_cast<const uint4 *>(in + off + e.s[dl] * ol + ot));
        }
#pragma unroll
        for (int h = 0; h < TL / 32; ++h) {
            const uint16_t *hv = reinterpret_cast<const uint16_t *>(&v[h]);
#pragma unroll
            for (int k = 0; k < 8; ++k) tile[8 * c8 + k][r + 32 * h] = hv[k];
        }
    }
    __syncthreads();
    constexpr int CPR = TL / 8;                                  // 16-byte chunks per output run
    const int cq = threadIdx.x % CPR, rq = threadIdx.x / CPR;
#pragma unroll
    for (int h = 0; h < 64 / (256 / CPR); ++h) {                // write 64 runs along dl: rows ot = t0 + rr
        const int rr = rq + (256 / CPR) * h;
        const int32_t ot = t0 + rr, ol = l0 + 8 * cq;
        if (ot >= e.w[dt] || ol >= e.w[dl]) continue;
        uint4 v;
        uint16_t *hv = reinterpret_cast<uint16_t *>(&v);
#pragma unroll
        for (int k = 0; k < 8; ++k) hv[k] = tile[rr][8 * cq + k];
        *reinterpret_cast<uint4 *>(out + obase + ostr[dt] * ot + ol) = v;
    }
}

}  // namespace ollie
