// epilogue.cuh -- NEXT-3: the element-wise operators that follow the convolution, fused into
// whichever kernel writes Y ("OffsetAdd ... fused with following element-wise operators",
// P:1572; reading Q19):
//     v = acc + bias[f] (+ residual[pixel, f]);   y = act(v)
// act: none | ReLU max(v, 0) | PReLU (v > 0 ? v : alpha[f] * v).  fp32 arithmetic on the fp32
// accumulator, then the usual RNE store.  A residual is read in Y's storage dtype from the
// same element offset Y is written to (it may alias Y: each element is read before the same
// thread writes it).
#pragma once
#include "sm100_ptx.cuh"

namespace ollie {

struct EpiArgs {
    const float *bias;      // [F] or nullptr
    const void *res;        // NHWC like Y, or nullptr
    const float *alpha;     // [F] PReLU slopes (act == 2)
    int32_t act;            // 0 none, 1 ReLU, 2 PReLU
    int32_t on;             // any of the above present (uniform fast-path test)
};

__device__ __forceinline__ float epi_act(const EpiArgs &e, float v, int f) {
    if (e.act == 1) return fmaxf(v, 0.f);
    if (e.act == 2) return v > 0.f ? v : __ldg(e.alpha + f) * v;
    return v;
}

// v[0..n) are the values of Y[off + k] (channel f0 + k), k < n; off counts Y elements.
template <bool kBF16, int NMAX>
__device__ __forceinline__ void epi_apply(const EpiArgs &e, float *v, int64_t off, int f0, int n) {
#pragma unroll
    for (int k = 0; k < NMAX; ++k) {
        if (k < n) {
            float t = v[k];
            if (e.bias) t += __ldg(e.bias + f0 + k);
            if (e.res) {
                if constexpr (kBF16) t += bf16_bits_to_float(reinterpret_cast<const uint16_t *>(e.res)[off + k]);
                else t += reinterpret_cast<const float *>(e.res)[off + k];
            }
            v[k] = epi_act(e, t, f0 + k);
        }
    }
}

// Same for a register array of raw fp32 bits (TMEM loads).
template <bool kBF16, int NMAX>
__device__ __forceinline__ void epi_apply_bits(const EpiArgs &e, uint32_t *v, int64_t off, int f0, int n) {
#pragma unroll
    for (int k = 0; k < NMAX; ++k) {
        if (k < n) {
            float t = __uint_as_float(v[k]);
            if (e.bias) t += __ldg(e.bias + f0 + k);
            if (e.res) {
                if constexpr (kBF16) t += bf16_bits_to_float(reinterpret_cast<const uint16_t *>(e.res)[off + k]);
                else t += reinterpret_cast<const float *>(e.res)[off + k];
            }
            v[k] = __float_as_uint(epi_act(e, t, f0 + k));
        }
    }
}

}  // namespace ollie
