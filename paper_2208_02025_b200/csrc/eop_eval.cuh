// eop_eval.cuh -- a7 / a5: generic evaluator of a scoped index-expression eOperator
//     L_{x in X} Sum_{y in Y} f( T[tau(x, y)] )          (general format)
// with affine + floordiv / mod index functions, zero pad bands
// and an optional nested scope read through the chain rule (expression fusion,
// P:955-963; fused eOperator pairs).  The host (ollie.cu) validates the
// descriptor, proves every read lies inside its pad band by interval arithmetic, drops
// identity eOperators and compiles the rest into this compact form.
//
// One thread per output element (grid-stride); the output is written densely in
// traversal order, so stores are coalesced.  Arithmetic is fp32.  Pure-indexing eOps are
// bit-exact copies (no arithmetic touches the value).
#pragma once
#include "sm100_ptx.cuh"

namespace ollie {

constexpr int EOPD_MAX_TERMS = 48;
constexpr int EOPD_MAX_DIMS = 24;
constexpr int EOPD_MAX_ACC = 8;
constexpr int EOPD_MAX_ITERS = 16;
constexpr int EOPD_MAX_INS = 32;
constexpr int EOPD_STACK = 8;

struct DTerm {           // coef * atom(iter)
    int32_t iter, kind;  // kind: 0 iterator, 1 floordiv, 2 mod
    int32_t div, coef;
};
struct DDim {            // one coordinate of one access
    int32_t t_begin, t_count;
    int64_t c0;
    int64_t extent;      // tensor extent (input) or trav width (scope 1)
    int64_t lo;          // 0 for inputs; traversal lo for scope 1
    int64_t stride;      // element stride (input) or dense stride of scope 1's coordinate space
};
struct DAcc {
    int32_t tensor;      // >= 0 input, -1 = scope 1
    int32_t d_begin, ndim;
};
struct DScope {
    int32_t n_trav, n_sum, n_ins, a_begin, n_acc;
    int64_t lo[EOPD_MAX_ITERS];      // traversal then summation iterator lower bounds
    int64_t width[EOPD_MAX_ITERS];
    int32_t op[EOPD_MAX_INS];
    int32_t arg[EOPD_MAX_INS];
    float cval[EOPD_MAX_INS];
    int64_t sum_count;
};
struct EopDev {
    const void *in[8];
    int32_t in_bf16[8];
    void *out;
    int32_t out_bf16;
    int32_t n_scopes;
    int64_t out_elems;
    DScope sc[2];
    DAcc acc[2 * EOPD_MAX_ACC];
    DDim dims[EOPD_MAX_DIMS];
    DTerm terms[EOPD_MAX_TERMS];
};

__device__ __forceinline__ int64_t floordiv64(int64_t a, int64_t d) {
    int64_t q = a / d;
    return (q * d > a) ? q - 1 : q;
}
__device__ __forceinline__ int64_t eval_dim(const EopDev &e, const DDim &d, const int64_t *it) {
    int64_t v = d.c0;
    for (int t = 0; t < d.t_count; ++t) {
        const DTerm &tm = e.terms[d.t_begin + t];
        int64_t a = it[tm.iter];
        if (tm.kind == 1) a = floordiv64(a, tm.div);
        else if (tm.kind == 2) a = a - floordiv64(a, tm.div) * tm.div;
        v += (int64_t)tm.coef * a;
    }
    return v;
}
__device__ __forceinline__ float load_in(const EopDev &e, int k, int64_t off) {
    if (e.in_bf16[k]) return bf16_bits_to_float(reinterpret_cast<const uint16_t *>(e.in[k])[off]);
    return reinterpret_cast<const float *>(e.in[k])[off];
}

template <int SC>
__device__ float scope_value(const EopDev &e, int64_t *it);

// Read accessed element: 0 in the pad band (validated on the host to never leave it).
template <int SC>
__device__ __forceinline__ float read_access(const EopDev &e, const DAcc &a, const int64_t *it) {
    if constexpr (SC == 0) {
        if (a.tensor < 0) {
            int64_t it1[EOPD_MAX_ITERS];
            const DScope &s1 = e.sc[1];
            for (int d = 0; d < a.ndim; ++d) {
                const DDim &dd = e.dims[a.d_begin + d];
                const int64_t v = eval_dim(e, dd, it);
                if (v < dd.lo || v >= dd.lo + dd.extent) return 0.f;
                it1[d] = v;
            }
            (void)s1;
            return scope_value<1>(e, it1);
        }
    }
    int64_t off = 0;
    for (int d = 0; d < a.ndim; ++d) {
        const DDim &dd = e.dims[a.d_begin + d];
        const int64_t v = eval_dim(e, dd, it);
        if (v < 0 || v >= dd.extent) return 0.f;
        off += v * dd.stride;
    }
    return load_in(e, a.tensor, off);
}

template <int SC>
__device__ __forceinline__ float body(const EopDev &e, const int64_t *it) {
    const DScope &s = e.sc[SC];
    float stk[EOPD_STACK];
    int sp = 0;
    for (int p = 0; p < s.n_ins; ++p) {
        const int op = s.op[p];
        if (op == 0) {
            stk[sp++] = read_access<SC>(e, e.acc[s.a_begin + s.arg[p]], it);
        } else if (op == 1) {
            stk[sp++] = s.cval[p];
        } else if (op == 5) {
            stk[sp - 1] = -stk[sp - 1];
        } else {
            const float b = stk[--sp];
            const float a = stk[sp - 1];
            float r;
            switch (op) {
                case 2: r = a + b; break;
                case 3: r = a * b; break;
                case 4: r = a - b; break;
                case 6: r = fmaxf(a, b); break;
                default: r = fminf(a, b); break;
            }
            stk[sp - 1] = r;
        }
    }
    return stk[0];
}

// Value of scope SC at traversal point it[0..n_trav): Sum_y f(...).
template <int SC>
__device__ float scope_value(const EopDev &e, int64_t *it) {
    const DScope &s = e.sc[SC];
    if (s.n_sum == 0) return body<SC>(e, it);
    float acc = 0.f;
    for (int64_t k = 0; k < s.sum_count; ++k) {
        int64_t q = k;
        for (int d = s.n_trav + s.n_sum - 1; d >= s.n_trav; --d) {
            it[d] = s.lo[d] + q % s.width[d];
            q /= s.width[d];
        }
        acc += body<SC>(e, it);
    }
    return acc;
}

__global__ void __launch_bounds__(256) eop_eval_kernel(const __grid_constant__ EopDev e) {
    pdl_launch_dependents();
    pdl_wait();
    const DScope &s = e.sc[0];
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < e.out_elems;
         o += (int64_t)gridDim.x * blockDim.x) {
        int64_t it[EOPD_MAX_ITERS];
        int64_t q = o;
        for (int d = s.n_trav - 1; d >= 0; --d) {
            it[d] = s.lo[d] + q % s.width[d];
            q /= s.width[d];
        }
        const float v = scope_value<0>(e, it);
        if (e.out_bf16) reinterpret_cast<uint16_t *>(e.out)[o] = float_to_bf16_rne(v);
        else reinterpret_cast<float *>(e.out)[o] = v;
    }
}

}  // namespace ollie
