// fused_conv.cuh -- a8: merged GEMM with the OffsetAdd / selective addition fused into its
// epilogue, so the r*s*f intermediate T never round-trips HBM (expression fusion).
// (placeholder: the fused plan is reported unsupported until implemented)
#pragma once
#include "../../include/ollie.h"
#include "sm100_ptx.cuh"

namespace ollie {
static inline bool fused_supported(const ollie_conv_shape *, bool, int) { return false; }
static inline ollie_status run_fused(const ollie_conv_shape *, bool, int, const void *, const void *, void *, int64_t,
                                     int64_t, cudaStream_t) {
    return OLLIE_E_UNSUPPORTED;
}
}  // namespace ollie
