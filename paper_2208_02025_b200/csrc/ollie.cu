// ollie.cu -- libollie: the C ABI of include/ollie.h.  Host-side validation, plan choice,
// TMA tensor-map encoding, eOperator analysis (interval-arithmetic bounds, identity
// elimination) and kernel launches.  No device memory is allocated here; every buffer
// is caller-owned.  There is no CPU fallback: every step of the path runs in the
// kernels of merged_gemm.cuh / eop_kernels.cuh / eop_eval.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ollie.h"
#include "eop_eval.cuh"
#include "eop_fast.cuh"
#include "eop_kernels.cuh"
#include "fused_conv.cuh"
#include "g2bmm.cuh"
#include "merged_gemm.cuh"
#include "rowstream_conv.cuh"

using namespace ollie;

// ------------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

static ollie_status fail(ollie_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}
static ollie_status ok() {
    g_last_error.clear();
    return OLLIE_OK;
}
#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess) return fail(OLLIE_E_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)
#define CHECK_LAUNCH()                                                                                   \
    do {                                                                                                 \
        cudaError_t _e = cudaGetLastError();                                                             \
        if (_e != cudaSuccess) return fail(OLLIE_E_CUDA, "kernel launch: %s", cudaGetErrorString(_e)); \
    } while (0)

extern "C" int ollie_abi_version(void) { return OLLIE_ABI_VERSION; }

extern "C" const char *ollie_status_string(ollie_status st) {
    switch (st) {
        case OLLIE_OK: return "OLLIE_OK";
        case OLLIE_E_INVALID: return "OLLIE_E_INVALID";
        case OLLIE_E_UNSUPPORTED: return "OLLIE_E_UNSUPPORTED";
        case OLLIE_E_WORKSPACE: return "OLLIE_E_WORKSPACE";
        case OLLIE_E_OOB: return "OLLIE_E_OOB";
        case OLLIE_E_ALIGN: return "OLLIE_E_ALIGN";
        case OLLIE_E_CUDA: return "OLLIE_E_CUDA";
    }
    return "OLLIE_E_UNKNOWN";
}
extern "C" const char *ollie_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------------ device info
static int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

static size_t elem_size(ollie_dtype d) { return d == OLLIE_BF16 ? 2 : 4; }
static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------------ launches
// Every libollie kernel is launched with programmatic stream serialization (PDL): it may start
// while the previous kernel on the stream finishes; kernels call griddepcontrol.wait before
// touching data another kernel produces (sm100_ptx.cuh).  OLLIE_PDL=0 disables it (A/B tests).
static bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("OLLIE_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// Same, with thread-block clusters of `cluster_x` CTAs along x (CTA pairs for cta_group::2,
// split-K clusters).  Launched WITHOUT programmatic stream serialization: a cluster kernel launched
// early behind a running grid deadlocked on B200 (eOperator -> CTA-pair conv chain on a side
// stream, tools/next1_hang.py); it now starts after its predecessor completes (its
// griddepcontrol.wait is then a no-op), and may still let its own dependents start early.
template <typename... KArgs, typename... Args>
static cudaError_t launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                  int cluster_x, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cluster_x;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------------ TMA
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

// 2-D K-major operand: dims {inner, outer}, row stride in bytes, box {box_inner, box_outer}.
static ollie_status make_tmap_2d(CUtensorMap *m, const void *base, bool tf32, uint64_t inner, uint64_t outer,
                                 uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return OLLIE_OK;
}

// 4-D activation map NHWC: dims {c, w, h, n}; box {box_c, box_w, box_h, box_n}.
static ollie_status make_tmap_nhwc(CUtensorMap *m, const void *base, bool tf32, int64_t n, int64_t h, int64_t w,
                                   int64_t c, uint32_t bc, uint32_t bw, uint32_t bh, uint32_t bn) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
    const uint64_t es = tf32 ? 4 : 2;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(c * es), (cuuint64_t)(w * c * es), (cuuint64_t)(h * w * c * es)};
    cuuint32_t box[4] = {bc, bw, bh, bn};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                     const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (4d) failed (%d)", (int)r);
    return OLLIE_OK;
}

// ------------------------------------------------------------------------ merged GEMM launch
static const bool g_gemm_no_tma_out = [] {   // OLLIE_GEMM_NO_TMA_OUT=1: thread-per-row stores (A/B switch)
    const char *e = getenv("OLLIE_GEMM_NO_TMA_OUT");
    return e && e[0] == '1';
}();
// UMMA N per tile: multiple of 16 in [16, 256] minimising the padded N, larger on ties.
static int choose_bn(int64_t N) {
    int best = 256;
    int64_t best_pad = ceil_div(N, 256) * 256;
    for (int bn = 256; bn >= 16; bn -= 16) {
        int64_t padded = ceil_div(N, bn) * bn;
        if (padded < best_pad) {
            best_pad = padded;
            best = bn;
        }
    }
    return best;
}

// Few tiles (small M): narrower N tiles spread the GEMM over more SMs -- a CTA's TMA ops and MMAs
// are serial, so 18 CTAs x 256 columns lose to 72 x 64 (ResNet-18 512x7 batch 1).
static int gemm_bn(int64_t M, int64_t N) {
    int BN = choose_bn(N);
    const int64_t mt = ceil_div(M, GEMM_BM);
    while (BN % 64 == 0 && BN > 64 && mt * ceil_div(N, BN / 2) <= num_sms()) BN /= 2;
    return BN;
}

template <bool TF32, bool OUTBF16, bool RED = false>
static ollie_status launch_gemm_t(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &to, const GemmArgs &ga,
                                  cudaStream_t stream) {
    auto kern = merged_gemm_kernel<TF32, OUTBF16, RED>;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_done[dev & 63]) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes()));
        attr_done[dev & 63] = true;
    }
    const int64_t tiles = ceil_div(ga.M, GEMM_BM) * ceil_div(ga.N, ga.BN);
    const int grid = (int)std::min<int64_t>(tiles, num_sms());
    CUDA_TRY(launch(kern, dim3(grid), dim3(GEMM_THREADS), gemm_smem_bytes(), stream, ta, tb, to, ga));
    return OLLIE_OK;
}

// out = A[M,K] * B[N,K]^T ; out fp32 (out_bf16 = false) or bf16, leading dim ldo.
static ollie_status run_gemm(int64_t M, int64_t N, int64_t K, bool tf32, const void *A, const void *B, void *out,
                             int64_t ldo, bool out_bf16, cudaStream_t stream, const EpiArgs *epi = nullptr,
                             const RedArgs *red = nullptr) {
    const size_t es = tf32 ? 4 : 2;
    if ((K * es) % 16 != 0)
        return fail(OLLIE_E_ALIGN, "K*sizeof(elem) = %lld is not a multiple of 16 (TMA rule); pad channels",
                    (long long)(K * es));
    if (!aligned16(A) || !aligned16(B)) return fail(OLLIE_E_ALIGN, "GEMM operand base not 16-byte aligned");
    if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31))
        return fail(OLLIE_E_UNSUPPORTED, "GEMM extent exceeds int32 TMA coordinates");
    const int BN = gemm_bn(M, N);
    const uint32_t BK = (uint32_t)(GEMM_BK_BYTES / es);
    CUtensorMap ta, tb;
    ollie_status st = make_tmap_2d(&ta, A, tf32, (uint64_t)K, (uint64_t)M, (uint64_t)(K * es), BK, GEMM_BM);
    if (st != OLLIE_OK) return st;
    st = make_tmap_2d(&tb, B, tf32, (uint64_t)K, (uint64_t)N, (uint64_t)(K * es), BK, (uint32_t)BN);
    if (st != OLLIE_OK) return st;
    GemmArgs ga{M, N, K, BN, out, ldo, 0, epi ? *epi : EpiArgs{}, red ? *red : RedArgs{}};
    // staged TMA stores of the output tile (the unfused plan's fp32 T, the identity plan's bf16 / fp32 Y
    // with its NEXT-3 epilogue): 128-byte boxes of 32 fp32 / 64 bf16 columns x 32 rows
    CUtensorMap to = tb;   // placeholder when unused
    const int cw = out_bf16 ? 64 : 32;
    const int oes = out_bf16 ? 2 : 4;
    if (!red && BN % cw == 0 && aligned16(out) && (ldo * oes) % 16 == 0 &&
        !g_gemm_no_tma_out) {   // (store boxes must not cross into the next tile)
        st = make_tmap_2d(&to, out, !out_bf16, (uint64_t)N, (uint64_t)M, (uint64_t)(ldo * oes), (uint32_t)cw, 32);
        if (st != OLLIE_OK) return st;
        ga.tma_out = 1;
    }
    if (red) return tf32 ? launch_gemm_t<true, false, true>(ta, tb, to, ga, stream) : launch_gemm_t<false, false, true>(ta, tb, to, ga, stream);
    if (tf32) return out_bf16 ? launch_gemm_t<true, true>(ta, tb, to, ga, stream) : launch_gemm_t<true, false>(ta, tb, to, ga, stream);
    return out_bf16 ? launch_gemm_t<false, true>(ta, tb, to, ga, stream) : launch_gemm_t<false, false>(ta, tb, to, ga, stream);
}

extern "C" ollie_status ollie_merged_gemm(int64_t M, int64_t N, int64_t K, ollie_dtype dtype, const void *A,
                                          const void *B, float *T, int64_t ldT, ollie_stream_t stream) {
    if (M <= 0 || N <= 0 || K <= 0) return fail(OLLIE_E_INVALID, "GEMM extents must be positive");
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32) return fail(OLLIE_E_UNSUPPORTED, "GEMM dtype must be BF16 or TF32");
    if (!A || !B || !T) return fail(OLLIE_E_INVALID, "null pointer");
    if (ldT < N) return fail(OLLIE_E_INVALID, "ldT < N");
    // the epilogue's vector / TMA stores assume a 16-byte aligned T and 16-byte row pitch (header)
    if (!aligned16(T) || ldT % 4 != 0) return fail(OLLIE_E_ALIGN, "T must be 16-byte aligned with ldT %% 4 == 0");
    ollie_status st = run_gemm(M, N, K, dtype == OLLIE_TF32, A, B, T, ldT, false, (cudaStream_t)stream);
    return st == OLLIE_OK ? ok() : st;
}

// ------------------------------------------------------------------------ fused plan (a8)
// Tile geometry + f-slice choice for fused_conv_kernel; see fused_conv.cuh for the design.
static int g_force_mt = 0, g_force_fs = 0, g_force_res = -1;   // debug plan overrides (0 / -1 = auto)
static int g_force_pair = -1;                                   // debug: -1 auto, 0 single CTAs, 1 CTA pairs
static int g_force_occ = 0;                                     // debug: 0 auto, else CTAs per SM (1 or 2)
static int g_force_ks = -1;                                     // debug: -1 auto, else the split-K factor
static int g_force_ipt = 0;                                     // debug: 0 auto, else images per tile
static int g_force_g8 = -1;                                     // debug: -1 auto, else the lane layout (grp8)
static const bool g_no_tma_y = [] {   // OLLIE_NO_TMA_Y=1: fused-kernel Y by thread stores (A/B switch)
    const char *e = getenv("OLLIE_NO_TMA_Y");
    return e && e[0] == '1';
}();
static thread_local double g_last_fused_cost = 0, g_last_unfused_cost = 0;
static thread_local std::vector<FusedArgs> g_last_cands;

// Per-class tap tables (see fused_conv.cuh).  Conv2d: one class, every tap (i, j) at patch row
// offset i*dil*Xb + j*dil.  ConvTranspose2d (dilation 1): class (a, b) = output residue; kernel
// rows i = i0 + st*k with i0 = (a + pad) mod st read input row u + c_a - k, c_a = (a+pad-i0)/st.
struct ClassGeom {
    int ntaps_r, ntaps_s, i0, j0, ca, cb;
};
static void class_geom(const ollie_conv_shape *s, int a, int b, ClassGeom *g) {
    const int st = s->stride;
    g->i0 = (a + s->pad) % st;
    g->j0 = (b + s->pad) % st;
    g->ntaps_r = g->i0 < s->r ? (int)((s->r - g->i0 + st - 1) / st) : 0;
    g->ntaps_s = g->j0 < s->s ? (int)((s->s - g->j0 + st - 1) / st) : 0;
    g->ca = (a + s->pad - g->i0) / st;
    g->cb = (b + s->pad - g->j0) / st;
}

// Strided Conv2d input phases (NEXT-2, expression splitting by input residue): tap i reads
// input row st*(oy + q_i) + rho_i with i*dil - pad = st*q_i + rho_i, 0 <= rho_i < st, so the taps
// of one residue (rho_y, rho_x) are a stride-1 convolution over the subsampled image
// X_rho[u][v] = X[st*u + rho_y][st*v + rho_x] -- which TMA loads directly with element stride st.
// Stride 1 gives one phase with q_i = i*dil - pad (the plain haloed patch).
static int floordiv_i(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
struct PhaseGeom {
    int nph, qmin_y, qmin_x, span_y, span_x, max_taps, westr;
    int rho_y[FC_MAX_CLASSES], rho_x[FC_MAX_CLASSES], ntaps[FC_MAX_CLASSES];
    int nr[FC_MAX_CLASSES], ns[FC_MAX_CLASSES], wi0[FC_MAX_CLASSES], wj0[FC_MAX_CLASSES];
};
static int gcd_i(int a, int b) { while (b) { int t = a % b; a = b; b = t; } return a; }
static bool conv_phases(const ollie_conv_shape *s, PhaseGeom *g) {
    const int st = s->stride, dil = s->dilation, pad = s->pad;
    if (st * st > FC_MAX_CLASSES) return false;
    int qy0 = INT32_MAX, qy1 = INT32_MIN, qx0 = INT32_MAX, qx1 = INT32_MIN;
    for (int i = 0; i < s->r; ++i) {
        const int q = floordiv_i(i * dil - pad, st);
        qy0 = std::min(qy0, q); qy1 = std::max(qy1, q);
    }
    for (int j = 0; j < s->s; ++j) {
        const int q = floordiv_i(j * dil - pad, st);
        qx0 = std::min(qx0, q); qx1 = std::max(qx1, q);
    }
    g->qmin_y = qy0; g->qmin_x = qx0; g->span_y = qy1 - qy0; g->span_x = qx1 - qx0;
    g->westr = st / gcd_i(st, dil);
    g->nph = 0; g->max_taps = 0;
    for (int ry = 0; ry < st; ++ry)
        for (int rx = 0; rx < st; ++rx) {
            int n = 0;
            for (int i = 0; i < s->r; ++i)
                for (int j = 0; j < s->s; ++j)
                    if (i * dil - pad - st * floordiv_i(i * dil - pad, st) == ry &&
                        j * dil - pad - st * floordiv_i(j * dil - pad, st) == rx)
                        ++n;
            if (n == 0) continue;                       // residue no tap reads: no load, no work
            if (n > FC_MAX_TAPS) return false;
            // the phase's kernel rows / cols are arithmetic progressions of step st / gcd(st, dil)
            int nr = 0, ns = 0, i0 = -1, j0 = -1;
            for (int i = 0; i < s->r; ++i)
                if (i * dil - pad - st * floordiv_i(i * dil - pad, st) == ry) { if (i0 < 0) i0 = i; ++nr; }
            for (int j = 0; j < s->s; ++j)
                if (j * dil - pad - st * floordiv_i(j * dil - pad, st) == rx) { if (j0 < 0) j0 = j; ++ns; }
            g->nr[g->nph] = nr; g->ns[g->nph] = ns; g->wi0[g->nph] = i0; g->wj0[g->nph] = j0;
            g->rho_y[g->nph] = ry; g->rho_x[g->nph] = rx; g->ntaps[g->nph] = n;
            g->max_taps = std::max(g->max_taps, n);
            ++g->nph;
        }
    return g->nph > 0;
}

static bool no_clusters() {   // OLLIE_NO_CLUSTERS=1: plan without CTA pairs / split-K clusters (A/B tests)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("OLLIE_NO_CLUSTERS");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

static int nb_cap() {   // B ring depth cap (OLLIE_NB_MAX overrides, for experiments)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("OLLIE_NB_MAX");
        v = e ? std::max(2, std::min(32, atoi(e))) : 8;
    }
    return v;
}

static int na_cap() {   // OLLIE_NA_MAX: deepest patch ring of streamed fused plans (experiments)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("OLLIE_NA_MAX");
        v = e ? std::max(2, std::min(16, atoi(e))) : 3;
    }
    return v;
}
static int split_prod_env() {   // OLLIE_FC_SPLIT_PROD=0/1 forces the producer split, else the plan's
    static int v = -2;
    if (v == -2) {
        const char *e = getenv("OLLIE_FC_SPLIT_PROD");
        v = e ? (atoi(e) ? 1 : 0) : -1;
    }
    return v;
}
static int grb_cap() {   // OLLIE_GRB_MAX caps the kernel rows per weight box (experiments: deeper rings)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("OLLIE_GRB_MAX");
        v = e ? std::max(1, atoi(e)) : 64;
    }
    return v;
}

static bool plan_fused_search(const ollie_conv_shape *s, bool tf32, int transposed, FusedArgs *out, int64_t OH,
                              int64_t OW) {
    const int es = tf32 ? 4 : 2;
    if ((s->c * es) % 16 != 0) return false;
    if (s->n > INT32_MAX || s->h > 32768 || s->w > 32768 || s->c > 65535 || s->f > 65535) return false;
    FusedArgs base{};
    // patches from warp 0, weight boxes from warp 3: A/B on recorded plans (OLLIE_FC_SPLIT_PROD=0/1) --
    // ResNet-18 78.5 -> 77.1, stride-2 44.7 -> 42.3, InfoGAN 15.2 -> 14.4, CSRNet 173.7 -> 171.6 us
    base.split_prod = 1;
    int span_y, span_x, max_taps, nclass, taps_item;
    int64_t GH, GW;                               // class-grid (tile space) extent
    PhaseGeom pg{};
    // weight-box geometry of every table entry (class x phase): kernel rows / cols it reads
    int nent = 0, ent_nr[FC_MAX_CLASSES], ent_ns[FC_MAX_CLASSES];
    int westr = 1;
    if (!transposed) {
        if (!conv_phases(s, &pg)) return false;
        span_y = pg.span_y;
        span_x = pg.span_x;
        max_taps = pg.max_taps;
        taps_item = (int)(s->r * s->s);             // every tap once per item, over all phases
        nclass = 1;
        GH = OH; GW = OW;
        base.ost = 1;
        base.ist = s->stride;
        base.nph = pg.nph;
        westr = pg.westr;
        for (int ph = 0; ph < pg.nph; ++ph) {
            ent_nr[ph] = pg.nr[ph]; ent_ns[ph] = pg.ns[ph];
        }
        nent = pg.nph;
    } else {
        const int st = s->stride;
        if (s->dilation != 1 || st * st > FC_MAX_CLASSES) return false;
        int kr = 0, ks = 0;
        max_taps = 0;
        for (int a = 0; a < st; ++a)
            for (int b = 0; b < st; ++b) {
                ClassGeom g;
                class_geom(s, a, b, &g);
                if (g.ntaps_r == 0 || g.ntaps_s == 0) return false;      // class of pure zeros: not fused
                ent_nr[nent] = g.ntaps_r; ent_ns[nent] = g.ntaps_s;
                ++nent;
                kr = std::max(kr, g.ntaps_r);
                ks = std::max(ks, g.ntaps_s);
                max_taps = std::max(max_taps, g.ntaps_r * g.ntaps_s);
            }
        if (max_taps > FC_MAX_TAPS) return false;
        span_y = kr - 1;
        span_x = ks - 1;
        nclass = st * st;
        taps_item = max_taps;
        GH = ceil_div(OH, st); GW = ceil_div(OW, st);
        base.ost = st;
        base.ist = 1;
        base.nph = 1;
        westr = st;
    }
    const int ist = base.ist, nph = base.nph;
    int nsb = 0, max_rows = 0;
    for (int e = 0; e < nent; ++e) { nsb = std::max(nsb, ent_ns[e]); max_rows = std::max(max_rows, ent_nr[e]); }
    if ((nsb - 1) * westr + 1 > 256 || (max_rows - 1) * westr + 1 > 256) return false;
    // weight boxes of grb kernel rows: tiles per channel chunk (resident) and boxes per item step
    auto box_geom = [&](int grb, int *kc_tiles, int *ops_item) {
        int tiles = 0, ops_max = 0;
        for (int c0 = 0; c0 < nclass; ++c0) {
            int ops = 0;
            for (int ph = 0; ph < nph; ++ph) {
                const int e = c0 * nph + ph, ng = (ent_nr[e] + grb - 1) / grb;
                tiles += ng * nsb * grb;
                ops += ng;
            }
            ops_max = std::max(ops_max, ops);
        }
        *kc_tiles = tiles;
        *ops_item = ops_max;
    };
    const int CI = 16 / es, KI = 32 / es, BKfull = 128 / es;
    base.n = (int)s->n; base.H = (int)s->h; base.W = (int)s->w; base.C = (int)s->c; base.F = (int)s->f;
    base.R = (int)s->r; base.S = (int)s->s; base.pad = s->pad; base.dil = s->dilation;
    base.OH = (int)OH; base.OW = (int)OW;
    base.nclass = nclass; base.max_taps = max_taps;
    base.BK = s->c >= BKfull ? BKfull : (int)((s->c + KI - 1) / KI * KI);
    base.kchunks = (int)ceil_div(s->c, base.BK);
    const int nchunk = base.BK / CI;
    const bool sw128 = base.BK * es == 128;      // full 128-byte channel chunks: SWIZZLE_128B pixel rows
    const int rowbytes = sw128 ? 128 : 16;
    const int ksteps = base.BK / KI;
    const int sms = num_sms();
    const int64_t Fp = ceil_div(s->f, 16) * 16;
    const int budget = FC_SMEM_BUDGET - 1024 - 1024;
    // Cost model (SM cycles), calibrated on B200 with tools/sweep_plans.py: real-data tcgen05.mma
    // issues at ~max(N/2, 40 + N/3) cycles; a streamed weight tile costs a ~250-cycle handshake;
    // TMA streams ~40 B/clk per SM; single-buffered TMEM exposes the epilogue.
    double best = 1e300;
    FusedArgs a_best{};
    bool found = false;
    std::vector<std::pair<double, FusedArgs>> all;   // every evaluated plan (autotune candidates)
    // Two lane layouts of the 128-row A operand (fused_conv.cuh, FusedArgs::grp8):
    //  g8 = 0: 128 consecutive patch rows, lane = y*Xr + image*Xb + x -- the lanes of the Xb - XB halo
    //          columns of each row compute nothing;
    //  g8 = 1: 16 groups of 8 consecutive rows, group g = y*ipt + image at patch row g*Xb (the
    //          descriptor's 8-row stride SBO = Xb rows): XB <= 8 output columns per tile, every lane an
    //          output pixel (CSRNet 64x64: 128 of 128 lanes instead of 110, 64 of 64 columns instead of 66)
    for (int g8 = 0; g8 <= 1; ++g8) {
    if (g_force_g8 >= 0 && g8 != g_force_g8) continue;
    const int xb_hi = (int)std::min<int64_t>(GW, g8 ? 8 : 128);
    for (int XB = xb_hi; XB >= (g8 ? xb_hi : 1); --XB) {
      const int Xb = XB + span_x;
      if (Xb * ist > 256) continue;                // TMA box: <= 256 traversed elements
      // ipt > 1: several images share a tile, patch rows interleaved [y][image][x] (row pitch
      // Xr = ipt * Xb), so every tap is still one row offset -- small images fill the 128 lanes
      for (int ipt = 1; ipt <= 16; ++ipt) {   // up to 16 images: 2x2 / 4x4 GAN inputs fill the lanes
        if (ipt > 1 && (GW > XB || base.n < ipt)) break;
        if (g_force_ipt > 0 && ipt != g_force_ipt) continue;
        if (g8 && 16 % ipt) continue;
        const int Xr = ipt * Xb;
        const int lanes_fixed = (ipt - 1) * Xb + XB;     // lanes of the last output row
        if (!g8 && lanes_fixed > 128) break;
        const int Yb = g8 ? (int)std::min<int64_t>(GH, 16 / ipt) : (int)std::min<int64_t>(GH, (128 - lanes_fixed) / Xr + 1);
        if (Yb < 1) continue;
        if (!g8 && ipt == 1 && XB < std::min<int64_t>(GW, 128) && ceil_div(GW, XB) == ceil_div(GW, XB + 1) &&
            (128 - (XB + 1)) / (Xb + 1) + 1 >= Yb)
            continue;
        const int lane_span = g8 ? 15 * Xb + 8 : 128;   // patch rows the 128 lanes of one tap read
        for (int MT = 1; MT <= 4; ++MT) {
            if (g_force_mt > 0 && MT != g_force_mt) continue;
            if (MT > 1 && (int64_t)(MT - 1) * Yb >= GH) break;
            const int Yp = MT * Yb + span_y;
            if (Yp * ist > 256) break;
            const int max_off = span_y * Xr + span_x + (MT - 1) * Yb * Xr;
            if (max_off >= 65536) break;
            const int box = 16 * Xb * Yp * ipt * nchunk;   // same bytes in both layouts
            const int need = sw128 ? (max_off + lane_span) * 128
                                   : (nchunk - 1) * 16 * Xb * Yp * ipt + (max_off + lane_span) * 16;
            const int astage = (int)ceil_div(std::max(box, need), 1024) * 1024;
            if (2 * astage > budget) break;
            const int64_t items_sp = (int64_t)nclass * ceil_div(base.n, ipt) * ceil_div(GW, XB) * ceil_div(GH, (int64_t)Yb * MT);
            for (int FS : {(int)std::min<int64_t>(Fp, 256), 256, 192, 128, 96, 64, 48, 32, 16}) {
                if (FS > Fp) continue;
                if (g_force_fs > 0 && FS != g_force_fs) continue;
                const int acc_cols = (FS + 31) / 32 * 32;
                if (MT * acc_cols > 512) continue;
                const int nbuf = 2 * MT * acc_cols <= 512 ? 2 : 1;
                const int bstage = FS * 128;
                const int64_t slices = ceil_div(s->f, FS);
                const int64_t items = items_sp * slices;
                if (items > INT32_MAX) continue;
                for (int ksp : {1, 2, 4})
                for (int pair = 0; pair <= 1; ++pair)
                for (int occ = 1; occ <= 2; ++occ)
                for (int resident = 0; resident <= 1; ++resident) {
                    if (g_force_res >= 0 && resident != g_force_res) continue;
                    if (g_force_pair >= 0 && pair != g_force_pair) continue;
                    if (g_force_occ > 0 && occ != g_force_occ) continue;
                    if (g_force_ks >= 0 && ksp != g_force_ks) continue;
                    // split-K over a cluster of ksp CTAs (DSMEM reduction): single CTAs, streamed
                    // weights, one M-tile, at least one (chunk, phase) step per CTA
                    if (ksp > 1 && (pair || resident || MT != 1 || base.kchunks * nph < ksp)) continue;
                    if ((pair || ksp > 1) && no_clusters()) continue;
                    // pair = 1: a CTA pair computes two spatial tiles with M = 256 cta_group::2 MMAs;
                    // each CTA holds half of every weight tile (FS / 2 rows, SW128 atoms of 8 rows)
                    if (pair && (FS % 16 != 0 || items_sp < 2)) continue;
                    const int btile = pair ? bstage / 2 : bstage;      // one tap's tile in this CTA
                    const int64_t items_c = pair ? nclass * ceil_div(items_sp / nclass, 2) * slices : items;
                    // occ = 2: two CTAs per SM, each with half the smem and 256 TMEM columns
                    // Y through a smem stage + TMA stores: Conv2d (one output class), no split-K, whole
                    // 128-byte channel chunks per slice, 16-byte output rows
                    // (ConvTranspose classes store their interleaved outputs with TMA element strides)
                    const int ostr = transposed ? (int)s->stride : 1;
                    const int tma_y = (ksp == 1 && FS % (128 / es) == 0 && (s->f * es) % 16 == 0 &&
                                       XB * ostr <= 256 && Yb * ostr <= 256 && !g_no_tma_y) ? 1 : 0;
                    const int bud = (occ == 1 ? budget : (113 * 1024 - 2048)) - fc_red_bytes(ksp, FS) -
                                    (tma_y ? FC_YSTAGE_BYTES : 0);
                    const int nbuf_o = occ == 1 ? nbuf : (2 * MT * acc_cols <= 256 ? 2 : 1);
                    if (occ == 2 && MT * acc_cols > 256) continue;
                    // largest weight box (fewest TMA ops) that fits: grb kernel rows per box
                    int na = 0, nb = 0, grb = 0, kc_tiles = 0, ops_item = 0;
                    for (int g = std::min(max_rows, grb_cap()); g >= 1; --g) {
                        int kt, oi;
                        box_geom(g, &kt, &oi);
                        const int bst = nsb * g * btile;
                        if (resident) {
                            const int64_t wb = (int64_t)base.kchunks * kt * btile;
                            if (wb + 2 * astage > bud) continue;
                            na = (int)std::min<int64_t>(4, (bud - wb) / astage);
                            nb = 1;
                        } else {
                            // patch ring depth: a chunk's patch can only be reloaded once every MMA of
                            // the chunk two stages back retired, so with whole-chunk stages the depth
                            // decides how much of the L2 latency the MMAs hide (OLLIE_NA_MAX, default 3)
                            // The weight ring turns over once per box, the patch ring once per chunk: a
                            // third weight stage is worth more than a third patch stage (CSRNet, FS = 256
                            // pairs: 2 / 3 runs 170 us, 3 / 2 176 us), so the patch ring only deepens
                            // past 2 while 3 weight stages still fit -- or when they never would.
                            const int na_hi = std::max(2, std::min(na_cap(), base.kchunks * nph * MT));
                            const int nb_keep = bud >= 2 * astage + 3 * bst ? 3 : 2;
                            na = 2;
                            while (na < na_hi && bud >= (na + 1) * astage + nb_keep * bst) ++na;
                            nb = std::min(nb_cap(), (bud - na * astage) / bst);
                            if (nb < 2) continue;
                        }
                        grb = g; kc_tiles = kt; ops_item = oi;
                        break;
                    }
                    if (grb == 0) continue;
                    const int bstage_c = nsb * grb * btile;
                    // grid in work units: CTAs (single), CTA pairs, or split-K clusters
                    const int units = pair ? occ * sms / 2 : occ * sms / ksp;
                    int grid = (int)std::min<int64_t>(items_c, (int64_t)units);
                    if (resident) grid = (int)std::max<int64_t>(slices, grid / slices * slices);
                    const double per_cta = (double)ceil_div(items_c, grid);
                    // Measured on B200 (tools/mma_bench2.cu, tools/tma_bench.cu): a 128xNx16 MMA costs
                    // max(61, N/2) cycles; a CTA's TMA ops run ~one at a time at max(275, bytes/103)
                    // cycles (16-byte planar patch rows: ~8 B/clk); a weight-box handshake ~100 cycles.
                    const double instr = (double)base.kchunks * taps_item * ksteps * MT;
                    const double mma = instr * std::max(61.0, FS / 2.0) +
                                       (resident ? 0.0 : 100.0 * base.kchunks * ops_item);
                    const double a_op = sw128 ? std::max(275.0, box / 103.0) : std::max(275.0, box / 8.0);
                    const double b_op = std::max(275.0, bstage_c / 103.0);
                    const double ld = (double)base.kchunks * nph * a_op + (resident ? 0.0 : (double)base.kchunks * ops_item * b_op);
                    const double epi = nbuf_o == 2 ? 0.0 : MT * (FS / 32.0) * 400.0;
                    // co-resident CTAs share the SM's tensor core but each has its own TMA stream
                    double t = per_cta * (std::max(occ * mma / ksp, ld / ksp) + epi + 600.0);
                    if (ksp > 1) t += per_cta * (1500.0 + FS * 4.0);   // push + one cluster round trip per item
                    if (resident) t += (double)base.kchunks * (kc_tiles / (nsb * grb)) * b_op;
                    if (pair) t *= 1.1;   // measured: pairs rarely beat single CTAs on these layers (autotune decides)
                    {
                        FusedArgs a = base;
                        a.XB = XB; a.Xb = Xb; a.Yb = Yb; a.Yp = Yp; a.MT = MT;
                        a.ipt = ipt; a.Xr = Xr; a.ngrp = (int)ceil_div(base.n, ipt);
                        a.grp8 = g8;
                        a.lane_lp = g8 ? 8 * ipt : Xr;
                        a.lane_ip = g8 ? 8 : Xb;
                        a.a_sbo = g8 ? Xb * rowbytes : 8 * rowbytes;
                        a.tma_y = tma_y;
                        a.a_box_bytes = box; a.a_stage_bytes = astage;
                        a.FS = FS; a.acc_cols = acc_cols; a.nbuf = nbuf_o; a.b_stage_bytes = bstage_c;
                        a.b_tile_bytes = btile; a.nsb = nsb; a.grb = grb; a.westr = westr;
                        a.box_tiles = nsb * grb; a.kc_tiles = kc_tiles;
                        a.resident = resident; a.na = na; a.nb = nb;
                        a.tmem_cols = occ == 1 ? 512 : 256;
                        a.pair = pair;
                        a.ksplit = ksp;
                        all.emplace_back(t, a);
                        if (t < best * 0.995) {
                            best = t;
                            a_best = a;
                            found = true;
                        }
                    }
                }
            }
        }
      }
    }
    }
    if (!found) return false;
    auto finalize = [&](FusedArgs a) -> FusedArgs {
    a.lbo = 16 * a.Xb * a.Yp * a.ipt;
    a.sw128 = sw128 ? 1 : 0;
    (void)rowbytes;
    a.tiles_x = (int)ceil_div(GW, a.XB);
    a.tiles_y = (int)ceil_div(GH, (int64_t)a.Yb * a.MT);
    a.f_slices = (int)ceil_div(s->f, a.FS);
    a.num_tiles = (int)((int64_t)nclass * a.ngrp * a.tiles_x * a.tiles_y * a.f_slices);
    a.spatial = (int)((int64_t)nclass * a.ngrp * a.tiles_x * a.tiles_y);
    a.num_items = a.pair ? (int)(nclass * ceil_div(a.spatial / nclass, 2) * a.f_slices) : a.num_tiles;
    // class tables
    if (!transposed) {
        const int st = s->stride, dil = s->dilation;
        for (int ph = 0; ph < pg.nph; ++ph) {
            FusedClass &c = a.cls[ph];
            c.ntaps = 0;
            c.oy0 = c.ox0 = 0;
            c.py = st * pg.qmin_y + pg.rho_y[ph];      // full-resolution input coordinates
            c.px = st * pg.qmin_x + pg.rho_x[ph];
            c.wi0 = pg.wi0[ph];
            c.wj0 = pg.wj0[ph];
            c.nr = pg.nr[ph];
            c.ns = pg.ns[ph];
            c.ntaps = c.nr * c.ns;
            // kernel row wi0 + westr*k reads subsampled-patch row q(k) - qmin with q(k) = q(0) + k*dil/g
            const int step = dil / gcd_i(st, dil);
            const int q0y = floordiv_i((int)(c.wi0 * dil - s->pad), st), q0x = floordiv_i((int)(c.wj0 * dil - s->pad), st);
            c.a_base = (q0y - pg.qmin_y) * a.Xr + (q0x - pg.qmin_x);
            c.a_dk = step * a.Xr;
            c.a_dl = step;
        }
    } else {
        const int st = s->stride;
        for (int ca = 0; ca < st; ++ca)
            for (int cb = 0; cb < st; ++cb) {
                ClassGeom g;
                class_geom(s, ca, cb, &g);
                FusedClass &c = a.cls[ca * st + cb];
                c.ntaps = g.ntaps_r * g.ntaps_s;
                c.oy0 = ca;
                c.ox0 = cb;
                c.py = g.ca - (g.ntaps_r - 1);
                c.px = g.cb - (g.ntaps_s - 1);
                c.wi0 = g.i0;
                c.wj0 = g.j0;
                c.nr = g.ntaps_r;
                c.ns = g.ntaps_s;
                // kernel row i0 + st*k reads input row (tile row) + c_a - k: patch row nr-1-k
                c.a_base = (g.ntaps_r - 1) * a.Xr + (g.ntaps_s - 1);
                c.a_dk = -a.Xr;
                c.a_dl = -1;
            }
    }
    // weight boxes: groups of grb kernel rows per entry, resident tile offsets
    {
        int bres = 0;
        for (int e = 0; e < nent; ++e) {
            FusedClass &c = a.cls[e];
            c.ngroups = (ent_nr[e] + a.grb - 1) / a.grb;
            c.bres = bres;
            bres += c.ngroups * a.box_tiles;
        }
    }
    return a;
    };
    *out = finalize(a_best);
    // autotune candidates: the model's best few, distinct in (geometry, MT, FS, residency)
    std::sort(all.begin(), all.end(), [](const auto &x, const auto &y) { return x.first < y.first; });
    g_last_cands.clear();
    g_last_cands.push_back(*out);
    // the model's best geometry for every (MT, FS, residency, CTAs-per-SM) family, cheapest first:
    // structurally different plans the cost model cannot rank reliably are measured instead
    for (auto &c : all) {
        if ((int)g_last_cands.size() >= 40) break;
        bool dup = false;
        for (auto &d : g_last_cands)
            dup |= d.MT == c.second.MT && d.FS == c.second.FS && d.resident == c.second.resident && d.ipt == c.second.ipt &&
                   d.tmem_cols == c.second.tmem_cols && d.pair == c.second.pair && d.ksplit == c.second.ksplit &&
                   d.grp8 == c.second.grp8;
        if (!dup && c.first < 4.0 * best) g_last_cands.push_back(finalize(c.second));
    }
    // the staged TMA-store epilogue is not always the faster one (very large HBM-bound outputs can
    // prefer thread stores that overlap the next item's MMAs): measure both for the leading plans
    {
        const size_t n0 = g_last_cands.size();
        for (size_t i = 0; i < n0 && i < 8; ++i)
            if (g_last_cands[i].tma_y) {
                FusedArgs c = g_last_cands[i];
                c.tma_y = 0;
                g_last_cands.push_back(c);
            }
    }
    // the cost of the same layer unfused (GEMM writes T, OffsetAdd reads it back): AUTO only fuses
    // when the fused estimate is lower
    const double tbytes_unf = (double)(s->n * s->h * s->w) * (double)(s->r * s->s * s->f) * 4.0;
    const double unf = (2.0 * tbytes_unf + (double)(s->n * s->h * s->w * s->c) * es +
                        (double)(s->n * OH * OW * s->f) * es) / (23.0 * sms) + 8000.0;
    g_last_fused_cost = best;
    g_last_unfused_cost = unf;
    return true;
}

// Plans are pure functions of (shape, dtype, SM count, overrides): cache them so the host cost of
// a launch is a lookup (the search is O(10^4) cost-model evaluations).
struct PlanKey {
    int64_t v[12];
    bool operator<(const PlanKey &o) const { return std::lexicographical_compare(v, v + 12, o.v, o.v + 12); }
};
struct PlanEntry {
    bool ok;
    FusedArgs args;                 // the plan in use (model's best, or the autotuned winner)
    std::vector<FusedArgs> cands;   // autotune candidates (cands[0] = model's best)
    double fused_cost, unfused_cost;
    int tuned;                      // 0: model decides; 1: autotuned fused; 2: autotuned unfused; 3: GEMM_RED;
                                    // 5 / 6: row-streaming ysum / direct (OLLIE_PLAN_ROWSTREAM_*)
};
static std::mutex g_plan_mu;
static std::map<PlanKey, PlanEntry> g_plan_cache;

static PlanEntry *plan_entry_mut(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW) {
    PlanKey k{{s->n, s->c, s->h, s->w, s->f, s->r * 65536 + s->s, s->pad, s->stride * 65536 + s->dilation,
               (int64_t)tf32 * 2 + transposed + 4 * (int64_t)s->output_padding, num_sms(),
               g_force_mt * 1000 + g_force_fs + 1000000 * g_force_ipt + 100000000ll * g_force_occ,
               ((g_force_res * 16 + g_force_pair) * 16 + g_force_ks) * 16 + g_force_g8}};
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        auto it = g_plan_cache.find(k);
        if (it != g_plan_cache.end()) return &it->second;
    }
    PlanEntry e{};
    e.ok = plan_fused_search(s, tf32, transposed, &e.args, OH, OW);
    e.fused_cost = g_last_fused_cost;
    e.unfused_cost = g_last_unfused_cost;
    if (e.ok) e.cands = g_last_cands;
    std::lock_guard<std::mutex> g(g_plan_mu);
    return &g_plan_cache.emplace(k, e).first->second;   // std::map nodes are stable
}
static const PlanEntry &plan_entry(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW) {
    return *plan_entry_mut(s, tf32, transposed, OH, OW);
}

static bool plan_fused(const ollie_conv_shape *s, bool tf32, int transposed, FusedArgs *out, int64_t OH, int64_t OW) {
    const PlanEntry &e = plan_entry(s, tf32, transposed, OH, OW);
    std::lock_guard<std::mutex> g(g_plan_mu);
    if (e.ok) *out = e.args;
    return e.ok;
}

// CTAs launched: work units (CTAs, CTA pairs, or split-K clusters) x CTAs per unit.  max_units
// caps the units at what can be co-resident (clusters: cudaOccupancyMaxActiveClusters).
static int fused_grid(const FusedArgs &a, int max_units = 0) {
    const int occ = a.tmem_cols == 256 ? 2 : 1;
    const int csz = a.pair ? 2 : (a.ksplit > 1 ? a.ksplit : 1);     // CTAs per work unit (cluster)
    int units = occ * num_sms() / csz;
    if (max_units > 0) units = std::min(units, max_units);
    int grid = (int)std::min<int64_t>(a.num_items, (int64_t)units);
    if (a.resident) grid = std::max(a.f_slices, grid / a.f_slices * a.f_slices);   // fixed f-slice per unit
    return csz * grid;
}

static size_t fused_smem_bytes(const FusedArgs &a) {
    const size_t b_region = a.resident ? (size_t)a.kchunks * a.kc_tiles * a.b_tile_bytes : (size_t)a.nb * a.b_stage_bytes;
    return 1024 + (size_t)a.na * a.a_stage_bytes + b_region + (size_t)fc_red_bytes(a.ksplit, a.FS) +
           (a.tma_y ? FC_YSTAGE_BYTES : 0) + 1024;
}

static bool out_hw(const ollie_conv_shape *s, int transposed, int64_t *OH, int64_t *OW) {
    if (!transposed) {
        *OH = (s->h + 2 * s->pad - (int64_t)s->dilation * (s->r - 1) - 1) / s->stride + 1;
        *OW = (s->w + 2 * s->pad - (int64_t)s->dilation * (s->s - 1) - 1) / s->stride + 1;
    } else {
        *OH = (s->h - 1) * s->stride - 2 * (int64_t)s->pad + (int64_t)s->dilation * (s->r - 1) + s->output_padding + 1;
        *OW = (s->w - 1) * s->stride - 2 * (int64_t)s->pad + (int64_t)s->dilation * (s->s - 1) + s->output_padding + 1;
    }
    return *OH > 0 && *OW > 0;
}

// Fused kernel can run this layer (explicit OLLIE_PLAN_FUSED).
static bool fused_supported(const ollie_conv_shape *s, bool tf32, int transposed) {
    int64_t OH, OW;
    if (!out_hw(s, transposed, &OH, &OW)) return false;
    return plan_entry(s, tf32, transposed, OH, OW).ok;
}

// OLLIE_PLAN_AUTO picks the fused kernel when it can run the layer and its cost estimate beats
// the unfused GEMM + OffsetAdd estimate (small-F, many-tap layers such as FSRCNN's 9x9 deconv
// keep the literal merged-GEMM form, where N = r*s*f stays wide).
static int tuned_choice(const ollie_conv_shape *s, bool tf32, int transposed) {
    int64_t OH, OW;
    if (!out_hw(s, transposed, &OH, &OW)) return 0;
    const PlanEntry &e = plan_entry(s, tf32, transposed, OH, OW);
    std::lock_guard<std::mutex> g(g_plan_mu);
    return e.tuned;
}

static bool fused_preferred(const ollie_conv_shape *s, bool tf32, int transposed) {
    int64_t OH, OW;
    if (!out_hw(s, transposed, &OH, &OW)) return false;
    const PlanEntry &e = plan_entry(s, tf32, transposed, OH, OW);
    std::lock_guard<std::mutex> g(g_plan_mu);
    if (e.tuned) return e.ok && e.tuned == 1;
    return e.ok && e.fused_cost <= e.unfused_cost;
}

template <bool TF32, bool PAIR, bool ONE, bool SPLIT>
static ollie_status launch_fused_t(const CUtensorMap &tx, const CUtensorMap &tw, const CUtensorMap &ty, const FusedArgs &a,
                                   cudaStream_t stream) {
    auto kern = fused_conv_kernel<TF32, PAIR, ONE, SPLIT>;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_done[dev & 63]) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done[dev & 63] = true;
    }
    const int csz = PAIR ? 2 : a.ksplit;
    if (csz > 1) {
        // clusters must all be co-resident for one wave: cap the grid at the active-cluster limit
        static std::mutex mu;
        static std::map<std::tuple<const void *, size_t, int>, int> cache;
        const size_t smem = fused_smem_bytes(a);
        int maxc = 0;
        {
            std::lock_guard<std::mutex> g(mu);
            auto key = std::make_tuple((const void *)kern, smem, csz);
            auto it = cache.find(key);
            if (it != cache.end()) {
                maxc = it->second;
            } else {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(csz * 64);
                cfg.blockDim = dim3(FC_THREADS);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = (unsigned)csz;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess) {
                    cudaGetLastError();
                    maxc = 0;
                }
                cache[key] = maxc;
            }
        }
        CUDA_TRY(launch_cluster(kern, dim3(fused_grid(a, maxc)), dim3(FC_THREADS), smem, stream, csz, tx, tw, ty, a));
    } else
        CUDA_TRY(launch(kern, dim3(fused_grid(a)), dim3(FC_THREADS), fused_smem_bytes(a), stream, tx, tw, ty, a));
    return OLLIE_OK;
}

static long long *g_fc_trace = nullptr;   // debug timeline buffer (ollie_debug_set_trace), off by default

static ollie_status run_fused(const ollie_conv_shape *s, bool tf32, int transposed, const void *x, const void *wp,
                              void *y, int64_t OH, int64_t OW, cudaStream_t stream, const EpiArgs *epi = nullptr) {
    FusedArgs a;
    if (!plan_fused(s, tf32, transposed, &a, OH, OW)) return fail(OLLIE_E_UNSUPPORTED, "no fused plan for this shape");
    a.y = y;
    a.epi = epi ? *epi : EpiArgs{};
    a.trace = g_fc_trace;
    {   // debug-only ablations (OLLIE_RS_DBG, see RsArgs::dbg); 0 in production
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("OLLIE_RS_DBG");
            dbg = e ? atoi(e) : 0;
        }
        a.dbg = dbg;
    }
    {   // debug-only kernel switches (OLLIE_FC_DBG, see FusedArgs::dbg); 0 in production
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("OLLIE_FC_DBG");
            dbg = e ? atoi(e) : 0;
        }
        a.dbg = dbg;
    }
    if (split_prod_env() >= 0) a.split_prod = split_prod_env();
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
    const int es = tf32 ? 4 : 2, CI = 16 / es;
    const CUtensorMapDataType dt = tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap tx, tw;
    // strided Conv2d: the patch is the subsampled image of one input phase, traversed with element
    // stride ist along w and h (ist * Xb traversed elements load Xb pixels)
    const uint32_t ist = (uint32_t)a.ist;
    // X is viewed with dims ordered {c, w, n, h} (strides need not be monotonic), so a box of ipt
    // images lands in smem as [y][image][x] rows: the interleaved patch of multi-image tiles
    if (a.sw128) {   // X as 4-D {c, w, n, h}, box = 128-byte pixel rows, SWIZZLE_128B
        cuuint64_t dims[4] = {(cuuint64_t)s->c, (cuuint64_t)s->w, (cuuint64_t)s->n, (cuuint64_t)s->h};
        cuuint64_t strides[3] = {(cuuint64_t)(s->c * es), (cuuint64_t)(s->h * s->w * s->c * es),
                                 (cuuint64_t)(s->w * s->c * es)};
        cuuint32_t box[4] = {(cuuint32_t)a.BK, (cuuint32_t)(a.Xb * ist), (cuuint32_t)a.ipt, (cuuint32_t)(a.Yp * ist)};
        cuuint32_t estr[4] = {1, ist, 1, ist};
        CUresult r = enc(&tx, dt, 4, const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (patch 4d) failed (%d)", (int)r);
    } else {   // X as 5-D planar view {c_in (16 B), w, n, h, c_out}
        cuuint64_t dims[5] = {(cuuint64_t)CI, (cuuint64_t)s->w, (cuuint64_t)s->n, (cuuint64_t)s->h,
                              (cuuint64_t)(s->c / CI)};
        cuuint64_t strides[4] = {(cuuint64_t)(s->c * es), (cuuint64_t)(s->h * s->w * s->c * es),
                                 (cuuint64_t)(s->w * s->c * es), 16};
        cuuint32_t box[5] = {(cuuint32_t)CI, (cuuint32_t)(a.Xb * ist), (cuuint32_t)a.ipt, (cuuint32_t)(a.Yp * ist),
                             (cuuint32_t)(a.BK / CI)};
        cuuint32_t estr[5] = {1, ist, 1, ist, 1};
        CUresult r = enc(&tx, dt, 5, const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (patch) failed (%d)", (int)r);
    }
    {   // W' as 4-D {c, f, j, i} (tap = i*S + j): one box = nsb x grb taps of an entry, kernel rows /
        // cols element-strided by westr (ConvT class / strided-conv phase); f >= F and taps past the
        // kernel are out of bounds -> zero
        cuuint64_t dims[4] = {(cuuint64_t)s->c, (cuuint64_t)s->f, (cuuint64_t)s->s, (cuuint64_t)s->r};
        cuuint64_t strides[3] = {(cuuint64_t)(s->c * es), (cuuint64_t)(s->f * s->c * es),
                                 (cuuint64_t)(s->s * s->f * s->c * es)};
        cuuint32_t box[4] = {(cuuint32_t)(128 / es), (cuuint32_t)(a.pair ? a.FS / 2 : a.FS),   // pair: this CTA's half
                             (cuuint32_t)((a.nsb - 1) * a.westr + 1), (cuuint32_t)((a.grb - 1) * a.westr + 1)};
        cuuint32_t estr[4] = {1, 1, (cuuint32_t)a.westr, (cuuint32_t)a.westr};
        CUresult r = enc(&tw, dt, 4, const_cast<void *>(wp), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (weights) failed (%d)", (int)r);
    }
    // Y as 4-D {f, ow, n, oh} (the tile's box {128-byte channel chunk, XB, ipt, Yb} in the stage's row
    // order); without a usable map (misaligned Y) the kernel falls back to thread stores
    CUtensorMap ty = tx;
    if (a.tma_y) {
        if (!aligned16(y)) {
            a.tma_y = 0;   // (the stage stays reserved in smem; only the store path changes)
        } else {
            cuuint64_t dims[4] = {(cuuint64_t)s->f, (cuuint64_t)OW, (cuuint64_t)s->n, (cuuint64_t)OH};
            cuuint64_t strides[3] = {(cuuint64_t)(s->f * es), (cuuint64_t)(OH * OW * s->f * es),
                                     (cuuint64_t)(OW * s->f * es)};
            const cuuint32_t o = (cuuint32_t)a.ost;   // ConvT class: every ost-th output pixel
            cuuint32_t box[4] = {(cuuint32_t)(128 / es), (cuuint32_t)a.XB * o, (cuuint32_t)a.ipt, (cuuint32_t)a.Yb * o};
            cuuint32_t estr[4] = {1, o, 1, o};
            CUresult r = enc(&ty, dt, 4, y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (Y store) failed (%d)", (int)r);
        }
    }
    const bool one = a.nclass * a.nph == 1;
    if (a.pair) {
        if (one) return tf32 ? launch_fused_t<true, true, true, false>(tx, tw, ty, a, stream) : launch_fused_t<false, true, true, false>(tx, tw, ty, a, stream);
        return tf32 ? launch_fused_t<true, true, false, false>(tx, tw, ty, a, stream) : launch_fused_t<false, true, false, false>(tx, tw, ty, a, stream);
    }
    if (a.ksplit > 1) {
        if (one) return tf32 ? launch_fused_t<true, false, true, true>(tx, tw, ty, a, stream) : launch_fused_t<false, false, true, true>(tx, tw, ty, a, stream);
        return tf32 ? launch_fused_t<true, false, false, true>(tx, tw, ty, a, stream) : launch_fused_t<false, false, false, true>(tx, tw, ty, a, stream);
    }
    if (one) return tf32 ? launch_fused_t<true, false, true, false>(tx, tw, ty, a, stream) : launch_fused_t<false, false, true, false>(tx, tw, ty, a, stream);
    return tf32 ? launch_fused_t<true, false, false, false>(tx, tw, ty, a, stream) : launch_fused_t<false, false, false, false>(tx, tw, ty, a, stream);
}

// ------------------------------------------------------------------------ row-streaming plan (a8, narrow f)
// rowstream_conv.cuh: kernel columns (and, for a ConvTranspose2d, the output residue classes) on
// the MMA's N, kernel rows as A-row shifts, the column OffsetAdd in the epilogue.  Plannable when
// the layer is (or rewrites to) a stride-1 program with s' * sigma^2 * f <= 64 columns per kernel
// row, one <= 128-byte channel chunk, and image rows of <= 512 pixels.
// Two forms share the kernel: "ysum" (kernel rows on N, the row OffsetAdd in the epilogue) and
// "direct" (N = f, all r*s taps as A-row shifts over the r resident input rows, one accumulator per
// OUTPUT row: no epilogue sum and no MMA <-> epilogue lockstep across rows).  mode: 0 ysum,
// 1 direct, -1 the planner's choice (direct for Conv2d when it needs <= 12 MMAs per M-tile, i.e.
// r*s*ksteps <= 12, else ysum; OLLIE_RS_MODE=0/1 forces one for ablations).
static bool plan_rowstream_mode(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW, int mode,
                                RsArgs *out);
static bool plan_rowstream(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW, RsArgs *out,
                           int mode = -1) {
    if (mode == 0 || mode == 1) return plan_rowstream_mode(s, tf32, transposed, OH, OW, mode, out);
    static int forced = -2;
    if (forced == -2) {
        const char *e = getenv("OLLIE_RS_MODE");
        forced = e ? atoi(e) : -1;
    }
    if (forced == 0 || forced == 1) return plan_rowstream_mode(s, tf32, transposed, OH, OW, forced, out);
    RsArgs d;
    if (plan_rowstream_mode(s, tf32, transposed, OH, OW, 1, &d) && d.R * d.S * d.ksteps <= 12) {
        *out = d;
        return true;
    }
    if (plan_rowstream_mode(s, tf32, transposed, OH, OW, 0, out)) return true;
    if (plan_rowstream_mode(s, tf32, transposed, OH, OW, 1, &d)) { *out = d; return true; }
    return false;
}
static bool plan_rowstream_mode(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW, int mode,
                                RsArgs *out) {
    const int es = tf32 ? 4 : 2;
    if (mode == 1 && transposed) return false;        // direct form: Conv2d only
    if (s->dilation != 1) return false;
    if (!transposed && s->stride != 1) return false;
    if ((s->c * es) % 16 != 0 || s->c * es > 128) return false;
    if (s->n > INT32_MAX || s->h > 32768 || s->w > 512 || s->f > 64) return false;
    RsArgs a{};
    a.n = (int)s->n; a.H = (int)s->h; a.W = (int)s->w; a.C = (int)s->c; a.F = (int)s->f;
    a.R0 = (int)s->r; a.S0 = (int)s->s; a.pad0 = s->pad;
    a.OH = (int)OH; a.OW = (int)OW;
    if (!transposed) {
        a.sub = 1;
        a.R = a.R0; a.S = a.S0; a.pad_y = a.pad_x = s->pad;
        a.OHc = (int)OH; a.OWc = (int)OW;
    } else {
        // class cy of output row sigma*q + cy reads input row q + d with kernel row k = cy + p - sigma*d:
        // the stride-1 program runs over the union of the classes' offsets d
        const int st = s->stride, p = s->pad;
        auto span = [&](int K, int *dmin, int *dmax) {
            *dmin = INT32_MAX; *dmax = INT32_MIN;
            for (int cy = 0; cy < st; ++cy)
                for (int k = 0; k < K; ++k)
                    if ((cy + p - k) % st == 0) {
                        const int d = (cy + p - k) / st;
                        *dmin = std::min(*dmin, d); *dmax = std::max(*dmax, d);
                    }
        };
        int dy0, dy1, dx0, dx1;
        span(a.R0, &dy0, &dy1);
        span(a.S0, &dx0, &dx1);
        if (dy0 > dy1 || dx0 > dx1) return false;
        a.sub = st;
        a.tr = 1;
        a.R = dy1 - dy0 + 1; a.S = dx1 - dx0 + 1;
        a.pad_y = -dy0; a.pad_x = -dx0;
        a.OHc = (int)ceil_div(OH, st); a.OWc = (int)ceil_div(OW, st);
    }
    a.Fp = a.sub * a.sub * a.F;
    if (mode == 1) {
        a.direct = 1;
        a.N = a.F;                                                            // output channels on N
    } else {
        if (a.Fp != 4 && a.Fp != 8 && a.Fp != 12 && a.Fp != 16) return false;   // kernel variants
        a.N = a.R * a.Fp;                                                     // kernel rows x f' on N
    }
    if (a.N > RS_MAX_NP || a.S > RS_MAX_S || a.pad_y < 0) return false;
    // column shifts read the zero pixel rows kept on both sides of a slot
    if (a.pad_x < 0 || a.pad_x > RS_ZR || a.S - 1 - a.pad_x > RS_ZR) return false;
    a.NP = (int)ceil_div(a.N, 16) * 16;
    a.acc_cols = a.NP;                                  // accumulators packed at 16-column granularity
    const int cb = (int)(s->c * es);
    a.rowbytes = cb <= 32 ? 32 : (cb <= 64 ? 64 : 128);
    a.swz = a.rowbytes == 32 ? 6 : (a.rowbytes == 64 ? 4 : 2);
    a.ksteps = (int)ceil_div(cb, 32);
    a.mtr = (int)ceil_div(std::max<int64_t>(s->w, a.OWc), 128);
    if (a.mtr > 4) return false;
    a.slot_bytes = (2 * RS_ZR + a.mtr * 128) * a.rowbytes;
    // one TMA box per <= 256 pixels; boxes land on whole swizzle atoms (8 rows) and fit the slot
    a.nbox = (int)ceil_div(s->w, 256);
    a.wbox = a.nbox == 1 ? (int)s->w : (int)ceil_div(ceil_div(s->w, a.nbox), 8) * 8;
    if (a.wbox > 256 || a.nbox * a.wbox > a.mtr * 128 + RS_ZR) return false;
    a.rows_total = s->n * a.OHc;
    a.tmem_cols = 512;
    a.row_cols = a.mtr * a.acc_cols;
    a.nt = std::min(16, 512 / a.row_cols);
    // ysum: the r-row window plus one row of look-ahead in TMEM; direct: two output rows in flight
    if (a.nt < (a.direct ? 2 : a.R + 1)) return false;
    a.ring = 0;
    const int fixed = (int)rs_smem_bytes(a) + 8 * 2 * 16;
    a.ring = std::min(16, (227 * 1024 - fixed) / a.slot_bytes);
    if (a.ring < (a.direct ? a.R + 1 : 2)) return false;   // direct: the r-row window stays resident
    if (rs_smem_bytes(a) > (size_t)227 * 1024) return false;
    *out = a;
    return true;
}
static int rowstream_grid(const RsArgs &a) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(a.rows_total, (int64_t)num_sms()));
}
static bool rowstream_supported(const ollie_conv_shape *s, bool tf32, int transposed, int64_t OH, int64_t OW,
                                int mode = -1) {
    RsArgs a;
    return plan_rowstream(s, tf32, transposed, OH, OW, &a, mode);
}
static bool is_rowstream_plan(int p) {
    return p == OLLIE_PLAN_ROWSTREAM || p == OLLIE_PLAN_ROWSTREAM_YSUM || p == OLLIE_PLAN_ROWSTREAM_DIRECT;
}
static int rowstream_mode_of(int p) {
    return p == OLLIE_PLAN_ROWSTREAM_YSUM ? 0 : (p == OLLIE_PLAN_ROWSTREAM_DIRECT ? 1 : -1);
}

template <bool TF32, int FP, bool DIRECT = false>
static ollie_status launch_rowstream_t(const CUtensorMap &tx, const RsArgs &a, cudaStream_t stream) {
    auto kern = rowstream_conv_kernel<TF32, FP, DIRECT>;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_done[dev & 63]) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done[dev & 63] = true;
    }
    CUDA_TRY(launch(kern, dim3(rowstream_grid(a)), dim3(RS_THREADS), rs_smem_bytes(a), stream, tx, a));
    return OLLIE_OK;
}

static ollie_status run_rowstream(const ollie_conv_shape *s, bool tf32, int transposed, const void *x, const void *wp,
                                  void *y, int64_t OH, int64_t OW, cudaStream_t stream, const EpiArgs *epi = nullptr,
                                  int mode = -1) {
    RsArgs a;
    if (!plan_rowstream(s, tf32, transposed, OH, OW, &a, mode)) return fail(OLLIE_E_UNSUPPORTED, "no row-streaming plan for this shape");
    a.wprep = wp;
    a.y = y;
    a.epi = epi ? *epi : EpiArgs{};
    a.trace = g_fc_trace;
    {   // debug-only ablations (OLLIE_RS_DBG, see RsArgs::dbg); 0 in production
        static int dbg = -1;
        if (dbg < 0) {
            const char *e = getenv("OLLIE_RS_DBG");
            dbg = e ? atoi(e) : 0;
        }
        a.dbg = dbg;
    }
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
    const int es = tf32 ? 4 : 2;
    CUtensorMap tx;
    {   // X as 4-D {c, w, h, n}; one box = wbox pixel rows of one image row, swizzled like the UMMA operand
        cuuint64_t dims[4] = {(cuuint64_t)s->c, (cuuint64_t)s->w, (cuuint64_t)s->h, (cuuint64_t)s->n};
        cuuint64_t strides[3] = {(cuuint64_t)(s->c * es), (cuuint64_t)(s->w * s->c * es), (cuuint64_t)(s->h * s->w * s->c * es)};
        cuuint32_t box[4] = {(cuuint32_t)(a.rowbytes / es), (cuuint32_t)a.wbox, 1, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        const CUtensorMapSwizzle sw = a.rowbytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                      : (a.rowbytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
        CUresult r = enc(&tx, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                         const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (row stream) failed (%d)", (int)r);
    }
    if (a.direct) return tf32 ? launch_rowstream_t<true, 16, true>(tx, a, stream) : launch_rowstream_t<false, 16, true>(tx, a, stream);
    switch (a.Fp) {
        case 4: return tf32 ? launch_rowstream_t<true, 4>(tx, a, stream) : launch_rowstream_t<false, 4>(tx, a, stream);
        case 8: return tf32 ? launch_rowstream_t<true, 8>(tx, a, stream) : launch_rowstream_t<false, 8>(tx, a, stream);
        case 12: return tf32 ? launch_rowstream_t<true, 12>(tx, a, stream) : launch_rowstream_t<false, 12>(tx, a, stream);
        default: return tf32 ? launch_rowstream_t<true, 16>(tx, a, stream) : launch_rowstream_t<false, 16>(tx, a, stream);
    }
}

// ------------------------------------------------------------------------ shapes
static ollie_status check_shape(const ollie_conv_shape *s, int transposed, int64_t *oh, int64_t *ow) {
    if (!s) return fail(OLLIE_E_INVALID, "null shape");
    if (s->n <= 0 || s->c <= 0 || s->h <= 0 || s->w <= 0 || s->f <= 0 || s->r <= 0 || s->s <= 0)
        return fail(OLLIE_E_INVALID, "EmptyRange: every extent must be positive");
    if (s->pad < 0 || s->stride < 1 || s->dilation < 1 || s->output_padding < 0)
        return fail(OLLIE_E_INVALID, "pad >= 0, stride >= 1, dilation >= 1, output_padding >= 0 required");
    int64_t H, W;
    if (!transposed) {
        if (s->output_padding != 0) return fail(OLLIE_E_INVALID, "output_padding is ConvTranspose2d-only");
        H = (s->h + 2 * s->pad - (int64_t)s->dilation * (s->r - 1) - 1) / s->stride + 1;
        W = (s->w + 2 * s->pad - (int64_t)s->dilation * (s->s - 1) - 1) / s->stride + 1;
        if (s->h + 2 * s->pad - (int64_t)s->dilation * (s->r - 1) - 1 < 0 ||
            s->w + 2 * s->pad - (int64_t)s->dilation * (s->s - 1) - 1 < 0)
            H = W = 0;
    } else {
        if (s->output_padding >= std::max(s->stride, s->dilation))
            return fail(OLLIE_E_INVALID, "output_padding must be < max(stride, dilation)");
        H = (s->h - 1) * s->stride - 2 * (int64_t)s->pad + (int64_t)s->dilation * (s->r - 1) + s->output_padding + 1;
        W = (s->w - 1) * s->stride - 2 * (int64_t)s->pad + (int64_t)s->dilation * (s->s - 1) + s->output_padding + 1;
    }
    if (H <= 0 || W <= 0) return fail(OLLIE_E_INVALID, "EmptyRange: output size is not positive");
    if (oh) *oh = H;
    if (ow) *ow = W;
    return OLLIE_OK;
}

extern "C" ollie_status ollie_output_hw(const ollie_conv_shape *shape, int transposed, int64_t *oh, int64_t *ow) {
    ollie_status st = check_shape(shape, transposed, oh, ow);
    return st == OLLIE_OK ? ok() : st;
}

static int64_t ldT_of(const ollie_conv_shape *s) { return ceil_div(s->r * s->s * s->f, 4) * 4; }

// ------------------------------------------------------------------------ a0 weight DLT
extern "C" size_t ollie_prepared_weight_bytes(const ollie_conv_shape *s, ollie_dtype dtype) {
    if (!s || s->r <= 0 || s->s <= 0 || s->f <= 0 || s->c <= 0) return 0;
    return (size_t)(s->r * s->s * s->f * s->c) * elem_size(dtype);
}

static ollie_status prepare_weight(const ollie_conv_shape *s, ollie_dtype dtype, const void *w, void *wp,
                                   cudaStream_t stream, bool transposed) {
    ollie_status st = check_shape(s, transposed, nullptr, nullptr);
    if (st != OLLIE_OK) return st;
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32) return fail(OLLIE_E_UNSUPPORTED, "weight dtype must be BF16 or TF32");
    if (!w || !wp) return fail(OLLIE_E_INVALID, "null pointer");
    const int64_t F = s->f, C = s->c, RS = s->r * s->s;
    if (F > 65535) return fail(OLLIE_E_UNSUPPORTED, "f > 65535");
    const int64_t sz = transposed ? RS : C * RS;
    const int64_t sc = transposed ? F * RS : RS;
    dim3 grid((unsigned)ceil_div(RS, 32), (unsigned)ceil_div(C, 32), (unsigned)F);
    if (dtype == OLLIE_BF16)
        CUDA_TRY(launch(weight_dlt_kernel<uint16_t>, grid, dim3(256), 0, stream, (const uint16_t *)w, (uint16_t *)wp, F, C,
                        RS, sz, sc));
    else
        CUDA_TRY(launch(weight_dlt_kernel<float>, grid, dim3(256), 0, stream, (const float *)w, (float *)wp, F, C, RS, sz,
                        sc));
    CHECK_LAUNCH();
    return ok();
}

extern "C" ollie_status ollie_prepare_weight_conv2d(const ollie_conv_shape *shape, ollie_dtype dtype,
                                                    const void *w_fcrs, void *w_prep, ollie_stream_t stream) {
    return prepare_weight(shape, dtype, w_fcrs, w_prep, (cudaStream_t)stream, false);
}
extern "C" ollie_status ollie_prepare_weight_convtranspose2d(const ollie_conv_shape *shape, ollie_dtype dtype,
                                                             const void *w_cfrs, void *w_prep, ollie_stream_t stream) {
    return prepare_weight(shape, dtype, w_cfrs, w_prep, (cudaStream_t)stream, true);
}

// ------------------------------------------------------------------------ a3 / a4 standalone
static ollie_status run_offset_add(const ollie_conv_shape *s, int transposed, const float *T, int64_t ldT, bool out_bf16,
                                   void *y, int64_t OH, int64_t OW, cudaStream_t stream, const EpiArgs *epi = nullptr) {
    OffsetAddArgs a;
    a.epi = epi ? *epi : EpiArgs{};
    a.T = T;
    a.ldT = ldT;
    a.y = y;
    a.n = s->n; a.h = s->h; a.w = s->w; a.f = s->f; a.r = s->r; a.s = s->s;
    a.oh = OH; a.ow = OW;
    a.pad = s->pad; a.stride = s->stride; a.dil = s->dilation;
    const bool vec4 = (s->f % 4 == 0) && (ldT % 4 == 0) && aligned16(T) && (out_bf16 ? (reinterpret_cast<uintptr_t>(y) & 7) == 0 : aligned16(y));
    const int VEC = vec4 ? 4 : 1;
    a.items = s->n * OH * OW * (s->f / VEC);
    // small outputs (ResNet b1 layers: a few thousand items) use 64-thread blocks so the loads spread
    // over more SMs; large ones 256-thread blocks, grid capped at 16 per SM (grid-stride loop)
    static const int tpb_env = [] { const char *e = getenv("OLLIE_OA_TPB"); return e ? atoi(e) : 0; }();
    const int tpb = tpb_env > 0 ? tpb_env : (a.items < (int64_t)num_sms() * 512 ? 64 : 256);
    const int64_t blocks = std::min<int64_t>(ceil_div(a.items, tpb), (int64_t)num_sms() * 16);
    const unsigned g = (unsigned)std::max<int64_t>(blocks, 1);
    // 32-bit index decoding when the item count and the grid stride fit comfortably
    const bool i32 = a.items + (int64_t)g * tpb < (1ll << 31);
#define OA_LAUNCH(K, V, B)                                                                 \
    do {                                                                                   \
        if (i32) CUDA_TRY(launch(K<V, B, int32_t>, dim3(g), dim3(tpb), 0, stream, a));        \
        else CUDA_TRY(launch(K<V, B, int64_t>, dim3(g), dim3(tpb), 0, stream, a));            \
    } while (0)
    if (!transposed) {
        if (vec4) { if (out_bf16) OA_LAUNCH(offset_add_kernel, 4, true); else OA_LAUNCH(offset_add_kernel, 4, false); }
        else { if (out_bf16) OA_LAUNCH(offset_add_kernel, 1, true); else OA_LAUNCH(offset_add_kernel, 1, false); }
    } else {
        if (vec4) { if (out_bf16) OA_LAUNCH(selective_add_kernel, 4, true); else OA_LAUNCH(selective_add_kernel, 4, false); }
        else { if (out_bf16) OA_LAUNCH(selective_add_kernel, 1, true); else OA_LAUNCH(selective_add_kernel, 1, false); }
    }
#undef OA_LAUNCH
    CHECK_LAUNCH();
    return OLLIE_OK;
}

// ------------------------------------------------------------------------ im2col ("tap folding") eOperator
extern "C" ollie_status ollie_tap_fold(const ollie_conv_shape *shape, ollie_dtype dtype, const void *x_nhwc, int64_t kp,
                                       void *out, ollie_stream_t stream) {
    if (!shape) return fail(OLLIE_E_INVALID, "null shape");
    int64_t OH, OW;
    ollie_status st = check_shape(shape, 0, &OH, &OW);
    if (st != OLLIE_OK) return st;
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32 && dtype != OLLIE_FP32)
        return fail(OLLIE_E_UNSUPPORTED, "tap fold dtype must be BF16 or TF32 / FP32");
    const int es = dtype == OLLIE_BF16 ? 2 : 4;
    const int64_t rsc = shape->r * shape->s * shape->c;
    if (kp < rsc) return fail(OLLIE_E_INVALID, "kp = %lld < r*s*c = %lld", (long long)kp, (long long)rsc);
    if ((kp * es) % 16 != 0) return fail(OLLIE_E_ALIGN, "kp * sizeof(elem) must be a multiple of 16");
    if (!x_nhwc || !out) return fail(OLLIE_E_INVALID, "null pointer");
    if (!aligned16(out)) return fail(OLLIE_E_ALIGN, "out must be 16-byte aligned");
    if (shape->h > INT32_MAX || shape->w > INT32_MAX || shape->c > INT32_MAX || kp > INT32_MAX)
        return fail(OLLIE_E_UNSUPPORTED, "tap fold extents exceed int32");
    TapFoldArgs a{};
    a.x = x_nhwc;
    a.out = out;
    a.H = (int)shape->h; a.W = (int)shape->w; a.C = (int)shape->c; a.R = (int)shape->r; a.S = (int)shape->s;
    a.pad = shape->pad; a.st = shape->stride; a.dil = shape->dilation;
    a.OH = (int)OH; a.OW = (int)OW; a.KP = (int)kp; a.RSC = (int)rsc;
    const int ve = 16 / es;
    cudaStream_t s = (cudaStream_t)stream;
    // row-tiled: the r input rows in smem with zero halo columns (left: every column a tap reads left of
    // the image, rounded up to 16 bytes; right: past the last image column), coalesced stores
    TapFoldRows tr{};
    {
        const int64_t lo = std::min<int64_t>(0, -(int64_t)shape->pad);                              // leftmost column read
        const int64_t hi = std::max<int64_t>(shape->w - 1, (OW - 1) * shape->stride - shape->pad +
                                                               (shape->s - 1) * (int64_t)shape->dilation);
        const int64_t roff = ceil_div(-lo * shape->c, ve) * ve;
        const int64_t rpitch = ceil_div(roff + (hi + 1) * shape->c, ve) * ve;
        tr.roff = (int)std::min<int64_t>(roff, INT32_MAX);
        tr.rpitch = (int)std::min<int64_t>(rpitch, INT32_MAX);
        tr.zcell = (int)std::min<int64_t>(shape->r * rpitch, INT32_MAX);
        tr.vec = ((shape->w * shape->c) % ve == 0 && aligned16(x_nhwc)) ? 1 : 0;
    }
    const size_t rows_smem = ((size_t)tr.zcell + 1) * es;
    if (rows_smem <= 48 * 1024 && 256 % (kp / ve) == 0 && (int64_t)tr.zcell < INT32_MAX) {
        a.items = shape->n * OH;
        const unsigned g1 = (unsigned)std::max<int64_t>(std::min<int64_t>(a.items, (int64_t)num_sms() * 64), 1);
        if (es == 2) CUDA_TRY(launch(tap_fold_rows_kernel<false>, dim3(g1), dim3(256), rows_smem, s, a, tr));
        else CUDA_TRY(launch(tap_fold_rows_kernel<true>, dim3(g1), dim3(256), rows_smem, s, a, tr));
        CHECK_LAUNCH();
        return ok();
    }
    a.items = shape->n * OH * OW * (kp / ve);
    const int tpb = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(a.items, tpb), (int64_t)num_sms() * 16);
    const unsigned g = (unsigned)std::max<int64_t>(blocks, 1);
    const bool i32 = a.items + (int64_t)g * tpb < (1ll << 31);
    if (es == 2) {
        if (i32) CUDA_TRY(launch(tap_fold_kernel<false, int32_t>, dim3(g), dim3(tpb), 0, s, a));
        else CUDA_TRY(launch(tap_fold_kernel<false, int64_t>, dim3(g), dim3(tpb), 0, s, a));
    } else {
        if (i32) CUDA_TRY(launch(tap_fold_kernel<true, int32_t>, dim3(g), dim3(tpb), 0, s, a));
        else CUDA_TRY(launch(tap_fold_kernel<true, int64_t>, dim3(g), dim3(tpb), 0, s, a));
    }
    CHECK_LAUNCH();
    return ok();
}

extern "C" ollie_status ollie_offset_add(const ollie_conv_shape *shape, int transposed, const float *T, int64_t ldT,
                                         ollie_dtype y_dtype, void *y_nhwc, ollie_stream_t stream) {
    int64_t OH, OW;
    ollie_status st = check_shape(shape, transposed, &OH, &OW);
    if (st != OLLIE_OK) return st;
    if (transposed && shape->dilation != 1)
        return fail(OLLIE_E_UNSUPPORTED, "selective addition implemented for dilation 1 only");
    if (!T || !y_nhwc) return fail(OLLIE_E_INVALID, "null pointer");
    if (ldT < shape->r * shape->s * shape->f) return fail(OLLIE_E_INVALID, "ldT < r*s*f");
    st = run_offset_add(shape, transposed, T, ldT, y_dtype == OLLIE_BF16, y_nhwc, OH, OW, (cudaStream_t)stream);
    return st == OLLIE_OK ? ok() : st;
}

// ------------------------------------------------------------------------ derived layers
static bool is_identity_offset_add(const ollie_conv_shape *s, int transposed) {
    // r = s = 1, pad 0, stride 1: OffsetAdd / selective add is the identity eOperator
    // (SURVEY 8(d) note) and is eliminated -- the GEMM epilogue writes Y.
    return s->r == 1 && s->s == 1 && s->pad == 0 && s->stride == 1 && (!transposed || s->output_padding == 0);
}

static int tuned_choice(const ollie_conv_shape *s, bool tf32, int transposed);   // autotune result (0 none)

static int resolve_plan(const ollie_conv_shape *s, ollie_dtype dtype, int plan, int transposed) {
    if (plan == OLLIE_PLAN_FUSED || plan == OLLIE_PLAN_UNFUSED || plan == OLLIE_PLAN_GEMM_RED || is_rowstream_plan(plan) ||
        plan == OLLIE_PLAN_SMALL)
        return plan;
    const bool tf32 = dtype == OLLIE_TF32;
    const int tc = tuned_choice(s, tf32, transposed);
    if (tc == 3) return OLLIE_PLAN_GEMM_RED;
    if (tc == OLLIE_PLAN_SMALL) return OLLIE_PLAN_SMALL;
    if (is_rowstream_plan(tc)) return tc;
    if (is_identity_offset_add(s, transposed)) return tc == 1 ? OLLIE_PLAN_FUSED : OLLIE_PLAN_UNFUSED;
    if (tc == 0 && s->w >= 96) {   // untuned: narrow layers over wide rows stream rows (>= 75% of the lanes busy)
        int64_t OH, OW;
        if (out_hw(s, transposed, &OH, &OW) && rowstream_supported(s, tf32, transposed, OH, OW)) return OLLIE_PLAN_ROWSTREAM;
    }
    return fused_preferred(s, tf32, transposed) ? OLLIE_PLAN_FUSED : OLLIE_PLAN_UNFUSED;
}

// GEMM_RED plan: fp32 output accumulator [n][OH][OW][F] in the workspace.
static size_t red_acc_bytes(const ollie_conv_shape *s, int64_t OH, int64_t OW) {
    return (size_t)(s->n * OH * OW * s->f) * sizeof(float);
}
static bool red_supported(const ollie_conv_shape *s, int transposed) {
    return s->f % 4 == 0 && !is_identity_offset_add(s, transposed) && s->h * s->w < (1ll << 30);
}

extern "C" size_t ollie_workspace_bytes(const ollie_conv_shape *s, ollie_dtype dtype, int plan, int transposed) {
    int64_t OH = 0, OW = 0;
    if (!s || check_shape(s, transposed, &OH, &OW) != OLLIE_OK) return 0;
    const int rp = resolve_plan(s, dtype, plan, transposed);
    if (rp == OLLIE_PLAN_GEMM_RED) return red_supported(s, transposed) ? red_acc_bytes(s, OH, OW) : 0;
    if (rp != OLLIE_PLAN_UNFUSED) return 0;
    if (is_identity_offset_add(s, transposed)) return 0;
    return (size_t)(s->n * s->h * s->w) * (size_t)ldT_of(s) * sizeof(float);
}

// NEXT-3 epilogue descriptor -> device form (validated before any launch).
static ollie_status make_epi(const ollie_epilogue *e, EpiArgs *out) {
    *out = EpiArgs{};
    if (!e) return OLLIE_OK;
    if (e->act < OLLIE_ACT_NONE || e->act > OLLIE_ACT_PRELU) return fail(OLLIE_E_INVALID, "unknown activation %d", e->act);
    if (e->act == OLLIE_ACT_PRELU && !e->alpha) return fail(OLLIE_E_INVALID, "PReLU needs alpha[f]");
    out->bias = e->bias;
    out->res = e->residual;
    out->alpha = e->alpha;
    out->act = e->act;
    out->on = (e->bias || e->residual || e->act != OLLIE_ACT_NONE) ? 1 : 0;
    return OLLIE_OK;
}

// GEMM_RED: zero the fp32 accumulator, merged GEMM whose epilogue reduces every T element into
// its output pixel (L2 atomics), then Y = epilogue(acc) in Y's dtype.  Three stream operations.
static ollie_status run_gemm_red(const ollie_conv_shape *s, int transposed, bool tf32, const void *x, const void *wp,
                                 float *acc, void *y, int64_t OH, int64_t OW, cudaStream_t stream, const EpiArgs *epi) {
    CUDA_TRY(cudaMemsetAsync(acc, 0, red_acc_bytes(s, OH, OW), stream));
    RedArgs rd{acc, (int)s->h, (int)s->w, (int)s->f, (int)s->s, s->pad, s->stride, s->dilation, (int)OH, (int)OW,
               transposed};
    const int64_t M = s->n * s->h * s->w, N = s->r * s->s * s->f;
    ollie_status st = run_gemm(M, N, s->c, tf32, x, wp, nullptr, 0, false, stream, nullptr, &rd);
    if (st != OLLIE_OK) return st;
    const int64_t n4 = s->n * OH * OW * s->f / 4;
    const unsigned g = (unsigned)std::max<int64_t>(std::min<int64_t>(ceil_div(n4, 256), (int64_t)num_sms() * 16), 1);
    const EpiArgs e = epi ? *epi : EpiArgs{};
    if (tf32) CUDA_TRY(launch(red_finish_kernel<false>, dim3(g), dim3(256), 0, stream, (const float *)acc, y, n4, (int32_t)s->f, e));
    else CUDA_TRY(launch(red_finish_kernel<true>, dim3(g), dim3(256), 0, stream, (const float *)acc, y, n4, (int32_t)s->f, e));
    return OLLIE_OK;
}

// OLLIE_PLAN_SMALL (eop_kernels.cuh small_conv_kernel): layers of at most 2^22 multiply-adds
static bool small_supported(const ollie_conv_shape *s, int transposed, int64_t OH, int64_t OW) {
    const int64_t macs = s->n * OH * OW * s->f * s->c * s->r * s->s;
    return macs <= (1ll << 22) && !(transposed && s->dilation != 1) && s->h < 65536 && s->w < 65536 &&
           OH < 65536 && OW < 65536 && s->c < 65536 && s->f < 65536 && s->r < 256 && s->s < 256;
}
static ollie_status run_small(const ollie_conv_shape *s, bool tf32, int transposed, const void *x, const void *wp, void *y,
                              int64_t OH, int64_t OW, cudaStream_t stream, const EpiArgs *epi) {
    if (!small_supported(s, transposed, OH, OW))
        return fail(OLLIE_E_UNSUPPORTED, "small plan: more than 2^22 multiply-adds (or extents too large)");
    SmallConvArgs a{};
    a.x = x; a.w = wp; a.y = y;
    a.n = (int)s->n; a.H = (int)s->h; a.W = (int)s->w; a.C = (int)s->c; a.F = (int)s->f; a.R = (int)s->r; a.S = (int)s->s;
    a.pad = s->pad; a.st = s->stride; a.dil = s->dilation; a.OH = (int)OH; a.OW = (int)OW;
    a.items = s->n * OH * OW * s->f;
    a.epi = epi ? *epi : EpiArgs{};
    const unsigned g = (unsigned)std::max<int64_t>(std::min<int64_t>(ceil_div(a.items, 256), (int64_t)num_sms() * 8), 1);
    if (tf32) {
        if (transposed) CUDA_TRY(launch(small_conv_kernel<true, true>, dim3(g), dim3(256), 0, stream, a));
        else CUDA_TRY(launch(small_conv_kernel<true, false>, dim3(g), dim3(256), 0, stream, a));
    } else {
        if (transposed) CUDA_TRY(launch(small_conv_kernel<false, true>, dim3(g), dim3(256), 0, stream, a));
        else CUDA_TRY(launch(small_conv_kernel<false, false>, dim3(g), dim3(256), 0, stream, a));
    }
    return OLLIE_OK;
}

static ollie_status derived_layer(const ollie_conv_shape *s, ollie_dtype dtype, const void *x, const void *wp, void *y,
                                  void *ws, size_t ws_bytes, int plan, cudaStream_t stream, int transposed,
                                  const ollie_epilogue *epilogue = nullptr) {
    int64_t OH, OW;
    ollie_status st = check_shape(s, transposed, &OH, &OW);
    if (st != OLLIE_OK) return st;
    EpiArgs epi;
    st = make_epi(epilogue, &epi);
    if (st != OLLIE_OK) return st;
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32) return fail(OLLIE_E_UNSUPPORTED, "dtype must be BF16 or TF32");
    if (transposed && s->dilation != 1) return fail(OLLIE_E_UNSUPPORTED, "ConvTranspose2d with dilation != 1");
    if (!x || !wp || !y) return fail(OLLIE_E_INVALID, "null pointer");
    if (!aligned16(x) || !aligned16(wp) || !aligned16(y)) return fail(OLLIE_E_ALIGN, "base pointers must be 16-byte aligned");
    const bool tf32 = dtype == OLLIE_TF32;
    if ((s->c * elem_size(dtype)) % 16 != 0)
        return fail(OLLIE_E_ALIGN, "c*sizeof(elem) = %lld not a multiple of 16: channel-pad x with an eOperator",
                    (long long)(s->c * elem_size(dtype)));
    int rp = resolve_plan(s, dtype, plan, transposed);
    const int64_t M = s->n * s->h * s->w, N = s->r * s->s * s->f, K = s->c;
    if (plan == OLLIE_PLAN_AUTO && !is_identity_offset_add(s, transposed) &&
        (rp == OLLIE_PLAN_UNFUSED || rp == OLLIE_PLAN_GEMM_RED)) {
        // AUTO follows the (process-wide) autotuned choice; a caller that sized its workspace
        // before another instance tuned this shape may not hold that plan's T / accumulator:
        // then AUTO runs the fused plan instead of failing (ollie.h, OLLIE_PLAN_AUTO)
        const size_t need = rp == OLLIE_PLAN_GEMM_RED ? red_acc_bytes(s, OH, OW)
                                                      : (size_t)M * (size_t)ldT_of(s) * sizeof(float);
        if ((!ws || ws_bytes < need) && fused_supported(s, tf32, transposed)) rp = OLLIE_PLAN_FUSED;
    }
    if (is_rowstream_plan(rp)) {
        st = run_rowstream(s, tf32, transposed, x, wp, y, OH, OW, stream, &epi, rowstream_mode_of(rp));
        return st == OLLIE_OK ? ok() : st;
    }
    if (rp == OLLIE_PLAN_SMALL) {
        st = run_small(s, tf32, transposed, x, wp, y, OH, OW, stream, &epi);
        return st == OLLIE_OK ? ok() : st;
    }
    if (rp == OLLIE_PLAN_FUSED) {
        if (!fused_supported(s, tf32, transposed))
            return fail(OLLIE_E_UNSUPPORTED, "fused plan not available for this shape/dtype");
        st = run_fused(s, tf32, transposed, x, wp, y, OH, OW, stream, &epi);
        return st == OLLIE_OK ? ok() : st;
    }
    if (rp == OLLIE_PLAN_GEMM_RED) {
        if (!red_supported(s, transposed))
            return fail(OLLIE_E_UNSUPPORTED, "GEMM_RED plan needs f %% 4 == 0 and a non-identity OffsetAdd");
        const size_t need = red_acc_bytes(s, OH, OW);
        if (!ws || ws_bytes < need) return fail(OLLIE_E_WORKSPACE, "GEMM_RED plan needs %zu workspace bytes (got %zu)", need, ws_bytes);
        if (!aligned16(ws)) return fail(OLLIE_E_ALIGN, "workspace must be 16-byte aligned");
        st = run_gemm_red(s, transposed, tf32, x, wp, (float *)ws, y, OH, OW, stream, &epi);
        return st == OLLIE_OK ? ok() : st;
    }
    if (is_identity_offset_add(s, transposed)) {
        // a6: identity eOperator eliminated -- the GEMM writes Y = X W'^T directly.
        st = run_gemm(M, N, K, tf32, x, wp, y, N, !tf32, stream, &epi);
        return st == OLLIE_OK ? ok() : st;
    }
    const int64_t ldT = ldT_of(s);
    const size_t need = (size_t)M * (size_t)ldT * sizeof(float);
    if (!ws || ws_bytes < need)
        return fail(OLLIE_E_WORKSPACE, "unfused plan needs %zu workspace bytes for T (got %zu)", need, ws_bytes);
    if (!aligned16(ws)) return fail(OLLIE_E_ALIGN, "workspace must be 16-byte aligned");
    st = run_gemm(M, N, K, tf32, x, wp, ws, ldT, false, stream);
    if (st != OLLIE_OK) return st;
    st = run_offset_add(s, transposed, (const float *)ws, ldT, !tf32, y, OH, OW, stream, &epi);
    return st == OLLIE_OK ? ok() : st;
}

extern "C" ollie_status ollie_conv2d_derived(const ollie_conv_shape *shape, ollie_dtype dtype, const void *x_nhwc,
                                             const void *w_prep, void *y_nhwc, void *ws, size_t ws_bytes, int plan,
                                             ollie_stream_t stream) {
    return derived_layer(shape, dtype, x_nhwc, w_prep, y_nhwc, ws, ws_bytes, plan, (cudaStream_t)stream, 0);
}
extern "C" ollie_status ollie_convtranspose2d_derived(const ollie_conv_shape *shape, ollie_dtype dtype,
                                                      const void *x_nhwc, const void *w_prep, void *y_nhwc, void *ws,
                                                      size_t ws_bytes, int plan, ollie_stream_t stream) {
    return derived_layer(shape, dtype, x_nhwc, w_prep, y_nhwc, ws, ws_bytes, plan, (cudaStream_t)stream, 1);
}
extern "C" ollie_status ollie_conv2d_derived_ex(const ollie_conv_shape *shape, ollie_dtype dtype, const void *x_nhwc,
                                                const void *w_prep, void *y_nhwc, void *ws, size_t ws_bytes, int plan,
                                                const ollie_epilogue *epilogue, ollie_stream_t stream) {
    return derived_layer(shape, dtype, x_nhwc, w_prep, y_nhwc, ws, ws_bytes, plan, (cudaStream_t)stream, 0, epilogue);
}
extern "C" ollie_status ollie_convtranspose2d_derived_ex(const ollie_conv_shape *shape, ollie_dtype dtype,
                                                         const void *x_nhwc, const void *w_prep, void *y_nhwc, void *ws,
                                                         size_t ws_bytes, int plan, const ollie_epilogue *epilogue,
                                                         ollie_stream_t stream) {
    return derived_layer(shape, dtype, x_nhwc, w_prep, y_nhwc, ws, ws_bytes, plan, (cudaStream_t)stream, 1, epilogue);
}

// ------------------------------------------------------------------------ eOperators
namespace {

struct Interval {
    int64_t lo, hi;  // inclusive
};

int64_t fdiv(int64_t a, int64_t d) {
    int64_t q = a / d;
    return (q * d > a) ? q - 1 : q;
}

// Symbolic simplification used by both the bounds check and the identity test:
// coef_div * (x // d) + coef_mod * (x % d) == coef_mod * x  when coef_div == coef_mod * d.
struct NormTerm {
    int32_t iter, kind;
    int64_t div, coef;
};
std::vector<NormTerm> normalize(const ollie_index &ix) {
    std::vector<NormTerm> ts;
    for (int t = 0; t < ix.nterms; ++t) ts.push_back({ix.term[t].iter, ix.term[t].kind, ix.term[t].div, ix.term[t].coef});
    bool changed = true;
    while (changed) {
        changed = false;
        for (size_t a = 0; a < ts.size() && !changed; ++a) {
            if (ts[a].kind != OLLIE_ATOM_FLOORDIV) continue;
            for (size_t b = 0; b < ts.size() && !changed; ++b) {
                if (ts[b].kind == OLLIE_ATOM_MOD && ts[b].iter == ts[a].iter && ts[b].div == ts[a].div &&
                    ts[a].coef == ts[b].coef * ts[a].div) {
                    NormTerm m{ts[a].iter, OLLIE_ATOM_ITER, 1, ts[b].coef};
                    std::vector<NormTerm> nt;
                    for (size_t k = 0; k < ts.size(); ++k)
                        if (k != a && k != b) nt.push_back(ts[k]);
                    nt.push_back(m);
                    ts.swap(nt);
                    changed = true;
                }
            }
        }
    }
    // merge plain terms of the same iterator
    std::vector<NormTerm> out;
    for (auto &t : ts) {
        bool merged = false;
        for (auto &o : out)
            if (o.kind == t.kind && o.iter == t.iter && o.div == t.div) {
                o.coef += t.coef;
                merged = true;
            }
        if (!merged) out.push_back(t);
    }
    std::vector<NormTerm> nz;
    for (auto &o : out)
        if (o.coef != 0) nz.push_back(o);
    return nz;
}

Interval index_interval(const ollie_index &ix, const int64_t *lo, const int64_t *hi /*exclusive*/) {
    Interval r{ix.c0, ix.c0};
    for (const NormTerm &t : normalize(ix)) {
        int64_t a = lo[t.iter], b = hi[t.iter] - 1;
        Interval at;
        if (t.kind == OLLIE_ATOM_ITER) at = {a, b};
        else if (t.kind == OLLIE_ATOM_FLOORDIV) at = {fdiv(a, t.div), fdiv(b, t.div)};
        else {
            if (b - a + 1 >= t.div) at = {0, t.div - 1};
            else {
                int64_t ma = a - fdiv(a, t.div) * t.div, mb = b - fdiv(b, t.div) * t.div;
                at = ma <= mb ? Interval{ma, mb} : Interval{0, t.div - 1};
            }
        }
        if (t.coef >= 0) {
            r.lo += t.coef * at.lo;
            r.hi += t.coef * at.hi;
        } else {
            r.lo += t.coef * at.hi;
            r.hi += t.coef * at.lo;
        }
    }
    return r;
}

ollie_status validate_scope(const ollie_eop *e, int k) {
    const ollie_scope &s = e->scope[k];
    if (s.n_trav < 1 || s.n_trav > OLLIE_MAX_DIMS || s.n_sum < 0 || s.n_sum > OLLIE_MAX_DIMS ||
        s.n_trav + s.n_sum > EOPD_MAX_ITERS)
        return fail(OLLIE_E_INVALID, "scope %d: iterator counts out of range", k);
    for (int d = 0; d < s.n_trav; ++d)
        if (s.trav_lo[d] >= s.trav_hi[d]) return fail(OLLIE_E_INVALID, "scope %d: EmptyRange (traversal %d)", k, d);
    for (int d = 0; d < s.n_sum; ++d)
        if (s.sum_lo[d] >= s.sum_hi[d]) return fail(OLLIE_E_INVALID, "scope %d: EmptyRange (summation %d)", k, d);
    if (s.n_acc < 0 || s.n_acc > OLLIE_MAX_ACCESS) return fail(OLLIE_E_INVALID, "scope %d: too many accesses", k);
    if (s.n_ins < 1 || s.n_ins > OLLIE_MAX_INSTR) return fail(OLLIE_E_INVALID, "scope %d: body length", k);
    const int nit = s.n_trav + s.n_sum;
    int64_t lo[EOPD_MAX_ITERS], hi[EOPD_MAX_ITERS];
    for (int d = 0; d < s.n_trav; ++d) { lo[d] = s.trav_lo[d]; hi[d] = s.trav_hi[d]; }
    for (int d = 0; d < s.n_sum; ++d) { lo[s.n_trav + d] = s.sum_lo[d]; hi[s.n_trav + d] = s.sum_hi[d]; }
    for (int a = 0; a < s.n_acc; ++a) {
        const ollie_access &ac = s.acc[a];
        const int64_t *ext_lo, *ext_hi;
        int64_t elo[OLLIE_MAX_DIMS], ehi[OLLIE_MAX_DIMS];
        int nd;
        if (ac.tensor >= 0) {
            if (ac.tensor >= e->n_in) return fail(OLLIE_E_INVALID, "scope %d access %d: unknown tensor", k, a);
            const ollie_tensor &t = e->in[ac.tensor];
            nd = t.ndim;
            for (int d = 0; d < nd; ++d) { elo[d] = -t.pad_lo[d]; ehi[d] = t.shape[d] + t.pad_hi[d]; }
        } else {
            if (ac.tensor != -1 || k != 0 || e->n_scopes != 2)
                return fail(OLLIE_E_INVALID, "scope %d access %d: nested-scope reference invalid", k, a);
            const ollie_scope &s1 = e->scope[1];
            nd = s1.n_trav;
            for (int d = 0; d < nd; ++d) { elo[d] = s1.trav_lo[d] - s1.pad_lo[d]; ehi[d] = s1.trav_hi[d] + s1.pad_hi[d]; }
        }
        ext_lo = elo;
        ext_hi = ehi;
        if (ac.ndim != nd) return fail(OLLIE_E_INVALID, "scope %d access %d: ArityMismatch (%d vs %d)", k, a, ac.ndim, nd);
        for (int d = 0; d < nd; ++d) {
            const ollie_index &ix = ac.idx[d];
            if (ix.nterms < 0 || ix.nterms > OLLIE_MAX_TERMS) return fail(OLLIE_E_INVALID, "too many terms");
            for (int t = 0; t < ix.nterms; ++t) {
                const ollie_term &tm = ix.term[t];
                if (tm.iter < 0 || tm.iter >= nit)
                    return fail(OLLIE_E_INVALID, "scope %d access %d dim %d: UndeclaredIterator %d", k, a, d, tm.iter);
                if (tm.kind < 0 || tm.kind > 2) return fail(OLLIE_E_INVALID, "bad atom kind");
                if (tm.kind != OLLIE_ATOM_ITER && tm.div <= 0) return fail(OLLIE_E_INVALID, "divisor must be > 0");
                if (tm.div > INT32_MAX || tm.coef > INT32_MAX || tm.coef < INT32_MIN)
                    return fail(OLLIE_E_UNSUPPORTED, "coefficient / divisor exceeds int32");
            }
            Interval iv = index_interval(ix, lo, hi);
            if (iv.lo < ext_lo[d] || iv.hi >= ext_hi[d])
                return fail(OLLIE_E_OOB, "scope %d access %d dim %d reads [%lld, %lld] outside the pad band [%lld, %lld)",
                            k, a, d, (long long)iv.lo, (long long)iv.hi, (long long)ext_lo[d], (long long)ext_hi[d]);
        }
    }
    // body: postfix well-formedness
    int depth = 0;
    for (int p = 0; p < s.n_ins; ++p) {
        const ollie_instr &in = s.body[p];
        switch (in.op) {
            case OLLIE_OP_PUSH_ACCESS:
                if (in.arg < 0 || in.arg >= s.n_acc) return fail(OLLIE_E_INVALID, "body: bad access id");
                depth++;
                break;
            case OLLIE_OP_PUSH_CONST: depth++; break;
            case OLLIE_OP_NEG:
                if (depth < 1) return fail(OLLIE_E_INVALID, "body: stack underflow");
                break;
            case OLLIE_OP_ADD: case OLLIE_OP_MUL: case OLLIE_OP_SUB: case OLLIE_OP_MAX: case OLLIE_OP_MIN:
                if (depth < 2) return fail(OLLIE_E_INVALID, "body: stack underflow");
                depth--;
                break;
            default: return fail(OLLIE_E_INVALID, "body: unknown op %d", in.op);
        }
        if (depth > EOPD_STACK) return fail(OLLIE_E_UNSUPPORTED, "body: stack deeper than %d", EOPD_STACK);
    }
    if (depth != 1) return fail(OLLIE_E_INVALID, "body leaves %d values on the stack", depth);
    return OLLIE_OK;
}

ollie_status validate_eop(const ollie_eop *e) {
    if (!e) return fail(OLLIE_E_INVALID, "null eop");
    if (e->n_in < 0 || e->n_in > OLLIE_MAX_INPUTS) return fail(OLLIE_E_INVALID, "n_in out of range");
    if (e->n_scopes < 1 || e->n_scopes > 2) return fail(OLLIE_E_INVALID, "n_scopes must be 1 or 2");
    if (e->out_dtype != OLLIE_BF16 && e->out_dtype != OLLIE_FP32) return fail(OLLIE_E_UNSUPPORTED, "out dtype");
    for (int k = 0; k < e->n_in; ++k) {
        const ollie_tensor &t = e->in[k];
        if (t.ndim < 1 || t.ndim > OLLIE_MAX_DIMS) return fail(OLLIE_E_INVALID, "input %d: ndim", k);
        if (t.dtype != OLLIE_BF16 && t.dtype != OLLIE_FP32) return fail(OLLIE_E_UNSUPPORTED, "input %d dtype", k);
        for (int d = 0; d < t.ndim; ++d)
            if (t.shape[d] <= 0 || t.pad_lo[d] < 0 || t.pad_hi[d] < 0)
                return fail(OLLIE_E_INVALID, "input %d: EmptyRange / negative pad", k);
    }
    if (e->n_scopes == 2) {
        const ollie_scope &s1 = e->scope[1];
        for (int d = 0; d < s1.n_trav && d < OLLIE_MAX_DIMS; ++d)
            if (s1.pad_lo[d] < 0 || s1.pad_hi[d] < 0) return fail(OLLIE_E_INVALID, "scope 1: negative pad");
        for (int a = 0; a < s1.n_acc && a < OLLIE_MAX_ACCESS; ++a)
            if (s1.acc[a].tensor < 0) return fail(OLLIE_E_INVALID, "scope 1 may only read inputs");
    }
    for (int k = 0; k < e->n_scopes; ++k) {
        ollie_status st = validate_scope(e, k);
        if (st != OLLIE_OK) return st;
    }
    return OLLIE_OK;
}

int64_t out_elems_of(const ollie_eop *e) {
    int64_t n = 1;
    for (int d = 0; d < e->scope[0].n_trav; ++d) n *= e->scope[0].trav_hi[d] - e->scope[0].trav_lo[d];
    return n;
}

bool is_pure_indexing(const ollie_eop *e) {
    const ollie_scope &s = e->scope[0];
    return e->n_scopes == 1 && s.n_sum == 0 && s.n_acc == 1 && s.n_ins == 1 && s.body[0].op == OLLIE_OP_PUSH_ACCESS &&
           s.acc[0].tensor >= 0;
}

// Identity eOperator: squash input and output to 1-D and check the map is
// the identity.  Symbolic for affine maps (after the div/mod recombination above);
// exhaustive enumeration for other maps up to 2^22 elements; otherwise "not identity".
bool is_identity(const ollie_eop *e) {
    if (!is_pure_indexing(e) || e->n_in != 1) return false;
    const ollie_scope &s = e->scope[0];
    const ollie_tensor &t = e->in[s.acc[0].tensor];
    if (t.dtype != e->out_dtype) return false;
    int64_t in_elems = 1;
    for (int d = 0; d < t.ndim; ++d) in_elems *= t.shape[d];
    const int64_t oe = out_elems_of(e);
    if (in_elems != oe) return false;
    int64_t lo[EOPD_MAX_ITERS], hi[EOPD_MAX_ITERS];
    for (int d = 0; d < s.n_trav; ++d) { lo[d] = s.trav_lo[d]; hi[d] = s.trav_hi[d]; }
    // no pad-band reads allowed
    for (int d = 0; d < t.ndim; ++d) {
        Interval iv = index_interval(s.acc[0].idx[d], lo, hi);
        if (iv.lo < 0 || iv.hi >= t.shape[d]) return false;
    }
    int64_t istride[OLLIE_MAX_DIMS], ostride[OLLIE_MAX_DIMS];
    istride[t.ndim - 1] = 1;
    for (int d = t.ndim - 2; d >= 0; --d) istride[d] = istride[d + 1] * t.shape[d + 1];
    ostride[s.n_trav - 1] = 1;
    for (int d = s.n_trav - 2; d >= 0; --d) ostride[d] = ostride[d + 1] * (s.trav_hi[d + 1] - s.trav_lo[d + 1]);
    // symbolic attempt
    bool affine = true;
    int64_t coef[EOPD_MAX_ITERS] = {0};
    int64_t c = 0;
    for (int d = 0; d < t.ndim && affine; ++d) {
        c += istride[d] * s.acc[0].idx[d].c0;
        for (const NormTerm &nt : normalize(s.acc[0].idx[d])) {
            if (nt.kind != OLLIE_ATOM_ITER) { affine = false; break; }
            coef[nt.iter] += istride[d] * nt.coef;
        }
    }
    if (affine) {
        // in_linear(x) = c + sum_k coef[k] x_k must equal out_linear(x) = sum_k ostride[k] (x_k - lo_k)
        // on the whole box: equal slopes on every non-degenerate iterator, equal at x = lo.
        int64_t at_lo = c;
        for (int k = 0; k < s.n_trav; ++k) {
            if (s.trav_hi[k] - s.trav_lo[k] > 1 && coef[k] != ostride[k]) return false;
            at_lo += coef[k] * s.trav_lo[k];
        }
        return at_lo == 0;
    }
    if (oe > (1ll << 22)) return false;
    int64_t it[EOPD_MAX_ITERS];
    for (int64_t o = 0; o < oe; ++o) {
        int64_t q = o;
        for (int d = s.n_trav - 1; d >= 0; --d) {
            const int64_t wdt = s.trav_hi[d] - s.trav_lo[d];
            it[d] = s.trav_lo[d] + q % wdt;
            q /= wdt;
        }
        int64_t lin = 0;
        for (int d = 0; d < t.ndim; ++d) {
            const ollie_index &ix = s.acc[0].idx[d];
            int64_t v = ix.c0;
            for (int k = 0; k < ix.nterms; ++k) {
                int64_t a = it[ix.term[k].iter];
                if (ix.term[k].kind == OLLIE_ATOM_FLOORDIV) a = fdiv(a, ix.term[k].div);
                else if (ix.term[k].kind == OLLIE_ATOM_MOD) a = a - fdiv(a, ix.term[k].div) * ix.term[k].div;
                v += ix.term[k].coef * a;
            }
            lin += v * istride[d];
        }
        if (lin != o) return false;
    }
    return true;
}

ollie_status compile_eop(const ollie_eop *e, const void *const *inputs, void *out, EopDev *dv) {
    memset(dv, 0, sizeof *dv);
    for (int k = 0; k < e->n_in; ++k) {
        dv->in[k] = inputs[k];
        dv->in_bf16[k] = e->in[k].dtype == OLLIE_BF16;
    }
    dv->out = out;
    dv->out_bf16 = e->out_dtype == OLLIE_BF16;
    dv->n_scopes = e->n_scopes;
    dv->out_elems = out_elems_of(e);
    int nt = 0, nd = 0, na = 0;
    for (int k = 0; k < e->n_scopes; ++k) {
        const ollie_scope &s = e->scope[k];
        DScope &d = dv->sc[k];
        d.n_trav = s.n_trav;
        d.n_sum = s.n_sum;
        d.n_ins = s.n_ins;
        d.n_acc = s.n_acc;
        d.a_begin = na;
        d.sum_count = 1;
        for (int i = 0; i < s.n_trav; ++i) { d.lo[i] = s.trav_lo[i]; d.width[i] = s.trav_hi[i] - s.trav_lo[i]; }
        for (int i = 0; i < s.n_sum; ++i) {
            d.lo[s.n_trav + i] = s.sum_lo[i];
            d.width[s.n_trav + i] = s.sum_hi[i] - s.sum_lo[i];
            d.sum_count *= d.width[s.n_trav + i];
        }
        for (int p = 0; p < s.n_ins; ++p) { d.op[p] = s.body[p].op; d.arg[p] = s.body[p].arg; d.cval[p] = s.body[p].cval; }
        for (int a = 0; a < s.n_acc; ++a) {
            if (na >= 2 * EOPD_MAX_ACC) return fail(OLLIE_E_UNSUPPORTED, "too many accesses");
            const ollie_access &ac = s.acc[a];
            DAcc &da = dv->acc[na++];
            da.tensor = ac.tensor;
            da.d_begin = nd;
            da.ndim = ac.ndim;
            int64_t stride = 1;
            for (int dd = ac.ndim - 1; dd >= 0; --dd) {
                if (nd >= EOPD_MAX_DIMS) return fail(OLLIE_E_UNSUPPORTED, "eop too large: > %d access dims", EOPD_MAX_DIMS);
                DDim &dm = dv->dims[da.d_begin + dd];
                const ollie_index &ix = ac.idx[dd];
                dm.c0 = ix.c0;
                if (ac.tensor >= 0) {
                    dm.extent = e->in[ac.tensor].shape[dd];
                    dm.lo = 0;
                    dm.stride = stride;
                    stride *= dm.extent;
                } else {
                    dm.extent = e->scope[1].trav_hi[dd] - e->scope[1].trav_lo[dd];
                    dm.lo = e->scope[1].trav_lo[dd];
                    dm.stride = 0;
                }
            }
            nd += ac.ndim;
            for (int dd = 0; dd < ac.ndim; ++dd) {
                DDim &dm = dv->dims[da.d_begin + dd];
                const ollie_index &ix = ac.idx[dd];
                dm.t_begin = nt;
                dm.t_count = ix.nterms;
                for (int t = 0; t < ix.nterms; ++t) {
                    if (nt >= EOPD_MAX_TERMS) return fail(OLLIE_E_UNSUPPORTED, "eop too large: > %d terms", EOPD_MAX_TERMS);
                    DTerm &tm = dv->terms[nt++];
                    tm.iter = ix.term[t].iter;
                    tm.kind = ix.term[t].kind;
                    tm.div = (int32_t)ix.term[t].div;
                    tm.coef = (int32_t)ix.term[t].coef;
                }
            }
        }
    }
    return OLLIE_OK;
}

int64_t tensor_bytes(const ollie_tensor &t) {
    int64_t n = 1;
    for (int d = 0; d < t.ndim; ++d) n *= t.shape[d];
    return n * (int64_t)elem_size(t.dtype);
}

}  // namespace

// Fast-path selection for pure-indexing affine eOperators (eop_fast.cuh).  Returns 0 (generic
// evaluator), 1 (affine gather) or 2 (tiled transpose).
static int affine_fast_plan(const ollie_eop *e, const void *in, void *out, AffineEop *fe) {
    if (!is_pure_indexing(e) || e->n_in != 1) return 0;
    const ollie_scope &s = e->scope[0];
    const ollie_access &ac = s.acc[0];
    const ollie_tensor &t = e->in[ac.tensor];
    if (s.n_trav > FAST_MAX_D || t.ndim > FAST_MAX_D || s.n_trav < 1) return 0;
    memset(fe, 0, sizeof *fe);
    fe->in = in;
    fe->out = out;
    fe->in_bf16 = t.dtype == OLLIE_BF16;
    fe->out_bf16 = e->out_dtype == OLLIE_BF16;
    fe->nd_out = s.n_trav;
    fe->nd_in = t.ndim;
    int64_t in_elems = 1, out_elems = 1;
    for (int k = 0; k < t.ndim; ++k) in_elems *= t.shape[k];
    for (int d = 0; d < s.n_trav; ++d) out_elems *= s.trav_hi[d] - s.trav_lo[d];
    if (in_elems >= (1ll << 31) || out_elems >= (1ll << 31)) return 0;
    int64_t stride[FAST_MAX_D];
    stride[t.ndim - 1] = 1;
    for (int k = t.ndim - 2; k >= 0; --k) stride[k] = stride[k + 1] * t.shape[k + 1];
    int64_t base = 0, sd[FAST_MAX_D] = {0};
    for (int k = 0; k < t.ndim; ++k) {
        const ollie_index &ix = ac.idx[k];
        int64_t b = ix.c0;
        for (int q = 0; q < ix.nterms; ++q) {
            const ollie_term &tm = ix.term[q];
            if (tm.kind != OLLIE_ATOM_ITER || tm.iter >= s.n_trav) return 0;
            fe->a[k][tm.iter] += (int32_t)tm.coef;
            b += tm.coef * s.trav_lo[tm.iter];
        }
        if (b > INT32_MAX || b < INT32_MIN) return 0;
        fe->b[k] = (int32_t)b;
        fe->shape[k] = (int32_t)t.shape[k];
        base += stride[k] * b;
    }
    for (int d = 0; d < s.n_trav; ++d) {
        fe->w[d] = (int32_t)(s.trav_hi[d] - s.trav_lo[d]);
        for (int k = 0; k < t.ndim; ++k) sd[d] += stride[k] * fe->a[k][d];
        if (sd[d] > INT32_MAX || sd[d] < INT32_MIN) return 0;
        fe->s[d] = (int32_t)sd[d];
    }
    if (base > INT32_MAX || base < INT32_MIN) return 0;
    fe->base = (int32_t)base;
    {   // input dims with a pad band need a bounds test; every other read is proven in range
        int64_t lo[EOPD_MAX_ITERS], hi[EOPD_MAX_ITERS];
        for (int d = 0; d < s.n_trav; ++d) { lo[d] = s.trav_lo[d]; hi[d] = s.trav_hi[d]; }
        for (int k = 0; k < t.ndim; ++k) {
            Interval iv = index_interval(ac.idx[k], lo, hi);
            if (iv.lo < 0 || iv.hi >= t.shape[k]) fe->chk |= 1 << k;
        }
    }
    // collapse adjacent output dims (d, d+1) that merge linearly: o' = o_d * w_{d+1} + o_{d+1}
    // keeps both the input offset and every CHECKED input index affine
    int nd = s.n_trav;
    for (int d = nd - 3; d >= 0; --d) {       // never merge into the innermost dim
        bool ok = (int64_t)fe->s[d] == (int64_t)fe->s[d + 1] * fe->w[d + 1];
        for (int k = 0; k < t.ndim && ok; ++k)
            if (fe->chk & (1 << k)) ok = (int64_t)fe->a[k][d] == (int64_t)fe->a[k][d + 1] * fe->w[d + 1];
        if (!ok) continue;
        fe->w[d] *= fe->w[d + 1];
        fe->s[d] = fe->s[d + 1];
        for (int k = 0; k < t.ndim; ++k) fe->a[k][d] = fe->a[k][d + 1];
        for (int e2 = d + 1; e2 < nd - 1; ++e2) {
            fe->w[e2] = fe->w[e2 + 1];
            fe->s[e2] = fe->s[e2 + 1];
            for (int k = 0; k < t.ndim; ++k) fe->a[k][e2] = fe->a[k][e2 + 1];
        }
        --nd;
    }
    fe->nd_out = nd;
    fe->inner = fe->w[nd - 1];
    fe->rows = (int32_t)(out_elems / fe->inner);
    if ((int64_t)fe->rows * ((fe->inner + 7) / 8) >= (1ll << 31)) return 0;
    // transpose path: innermost output dim strided in the input, another output dim with input
    // stride 1, and no pad-band reads (every index interval inside the tensor)
    if (fe->s[nd - 1] != 1 && fe->s[nd - 1] != 0 && nd >= 2 && fe->in_bf16 == fe->out_bf16) {
        const bool inside = fe->chk == 0;
        for (int d = 0; d < nd - 1 && inside; ++d)
            if (fe->s[d] == 1 && out_elems / ((int64_t)fe->w[d] * fe->inner) < 65536) {
                fe->dt = d;
                return 2;
            }
    }
    return 1;
}

extern "C" ollie_status ollie_eop_analyze(const ollie_eop *eop, ollie_eop_info *info) {
    ollie_status st = validate_eop(eop);
    if (st != OLLIE_OK) return st;
    if (!info) return fail(OLLIE_E_INVALID, "null info");
    info->is_identity = is_identity(eop);
    info->pure_indexing = is_pure_indexing(eop);
    info->out_elems = out_elems_of(eop);
    int64_t bi = 0;
    for (int k = 0; k < eop->n_in; ++k) bi += tensor_bytes(eop->in[k]);
    info->bytes_in = info->is_identity ? 0 : bi;
    info->bytes_out = info->is_identity ? 0 : info->out_elems * (int64_t)elem_size(eop->out_dtype);
    return ok();
}

extern "C" ollie_status ollie_eop_eval(const ollie_eop *eop, const void *const *inputs, void *output,
                                       ollie_stream_t stream) {
    ollie_status st = validate_eop(eop);
    if (st != OLLIE_OK) return st;
    if (!output || (eop->n_in > 0 && !inputs)) return fail(OLLIE_E_INVALID, "null pointer");
    for (int k = 0; k < eop->n_in; ++k)
        if (!inputs[k]) return fail(OLLIE_E_INVALID, "null input %d", k);
    cudaStream_t s = (cudaStream_t)stream;
    if (is_identity(eop)) {
        // a6: identity eOperator elimination -- nothing to launch when aliased.
        if (inputs[0] == output) return ok();
        CUDA_TRY(cudaMemcpyAsync(output, inputs[0], (size_t)tensor_bytes(eop->in[0]), cudaMemcpyDeviceToDevice, s));
        return ok();
    }
    {
        AffineEop fe;
        int kind = affine_fast_plan(eop, inputs[0], output, &fe);
        if (kind == 1) {
            const int64_t vec_per_row = (fe.inner + 7) / 8;
            const int64_t blocks = std::min<int64_t>(ceil_div((int64_t)fe.rows * vec_per_row, 256), (int64_t)num_sms() * 32);
            const unsigned gb = (unsigned)std::max<int64_t>(blocks, 1);
            static const int rows_mode = [] { const char *e = getenv("OLLIE_EOP_ROWS"); return e ? atoi(e) : 1; }();
            // staged rows: [rows][inner] with contiguous input rows and one valid column interval for all rows
            if (rows_mode && fe.in_bf16 == fe.out_bf16 && fe.nd_out == 2 && fe.s[1] == 1 && fe.s[0] > 0 &&
                fe.s[0] * (fe.in_bf16 ? 2 : 4) <= 128 && fe.inner * (fe.in_bf16 ? 2 : 4) % 16 == 0 && aligned16(fe.out)) {
                int32_t jlo = 0, jhi = fe.inner;
                bool uniform = true;
                for (int k = 0; k < fe.nd_in && uniform; ++k) {
                    if (!(fe.chk & (1 << k))) continue;
                    const int32_t c = fe.a[k][1], b = fe.b[k], n = fe.shape[k];
                    if (fe.a[k][0] != 0 || (c != 0 && c != 1)) { uniform = false; break; }
                    if (c == 0) { if (b < 0 || b >= n) jhi = 0; }
                    else { jlo = std::max(jlo, -b); jhi = std::min(jhi, n - b); }
                }
                // the span a pass reads: from row0's element 0 to the last row's column jhi
                if (uniform && jhi > jlo && jlo >= 0 && fe.base >= 0) {
                    const int es = fe.in_bf16 ? 2 : 4, ve = 16 / es;
                    const int32_t kR = std::max(1, 8192 / (fe.inner * es));          // 8 KB of output per pass
                    const size_t smem = (size_t)(((int64_t)(kR - 1) * fe.s[0] + jhi + ve) * es + 16);
                    const bool vin = ((int64_t)fe.base * es) % 16 == 0 && ((int64_t)kR * fe.s[0] * es) % 16 == 0 &&
                                     aligned16(fe.in);
                    const int64_t passes = ceil_div((int64_t)fe.rows, kR);
                    const unsigned g = (unsigned)std::max<int64_t>(std::min<int64_t>(passes, (int64_t)num_sms() * 8), 1);
                    if (smem <= 48 * 1024) {
                        if (fe.in_bf16) CUDA_TRY(launch(eop_staged_rows_kernel<uint16_t>, dim3(g), dim3(256), smem, s, fe, jlo, jhi, kR, (int32_t)vin));
                        else CUDA_TRY(launch(eop_staged_rows_kernel<uint32_t>, dim3(g), dim3(256), smem, s, fe, jlo, jhi, kR, (int32_t)vin));
                        CHECK_LAUNCH();
                        return ok();
                    }
                }
            }
            if (rows_mode && fe.in_bf16 == fe.out_bf16 && fe.inner <= 64 && fe.inner * (fe.in_bf16 ? 2 : 4) % 16 == 0 &&
                aligned16(fe.out)) {
                // narrow 16-byte-multiple rows: one thread per row
                const int64_t rb = std::min<int64_t>(ceil_div((int64_t)fe.rows, 256), (int64_t)num_sms() * 32);
                const unsigned g = (unsigned)std::max<int64_t>(rb, 1);
                if (fe.in_bf16) {
                    CUDA_TRY(launch(eop_affine_rows_kernel<uint16_t>, dim3(g), dim3(256), 0, s, fe));
                } else {
                    CUDA_TRY(launch(eop_affine_rows_kernel<uint32_t>, dim3(g), dim3(256), 0, s, fe));
                }
            } else if (fe.in_bf16 == fe.out_bf16) {
                if (fe.in_bf16) CUDA_TRY(launch(eop_affine_gather_kernel<8, uint16_t>, dim3(gb), dim3(256), 0, s, fe));
                else CUDA_TRY(launch(eop_affine_gather_kernel<4, uint32_t>, dim3(gb), dim3(256), 0, s, fe));
            } else {
                CUDA_TRY(launch(eop_affine_gather_kernel<8, void>, dim3(gb), dim3(256), 0, s, fe));
            }
            CHECK_LAUNCH();
            return ok();
        }
        if (kind == 2) {
            int64_t others = 1;
            for (int d = 0; d < fe.nd_out; ++d)
                if (d != fe.dt && d != fe.nd_out - 1) others *= fe.w[d];
            const int dl = fe.nd_out - 1;
            bool v16 = fe.in_bf16 && fe.out_bf16 && fe.w[dl] % 8 == 0 && fe.w[fe.dt] % 8 == 0 && fe.base % 8 == 0 &&
                       aligned16(fe.in) && aligned16(fe.out);
            for (int d = 0; d < fe.nd_out && v16; ++d)
                if (d != fe.dt && fe.s[d] % 8 != 0) v16 = false;
            if (v16) {   // 64 x 64 / 64 x 128 tiles, 16-byte loads and stores
                if (fe.w[dl] % 128 == 0) {
                    const int64_t strips16 = ceil_div(fe.w[dl], 128) * ceil_div(fe.w[fe.dt], 64);
                    CUDA_TRY(launch(eop_affine_transpose16_kernel<128>, dim3((unsigned)strips16, (unsigned)others), dim3(256), 0, s, fe));
                } else {
                    const int64_t strips16 = ceil_div(fe.w[dl], 64) * ceil_div(fe.w[fe.dt], 64);
                    CUDA_TRY(launch(eop_affine_transpose16_kernel<64>, dim3((unsigned)strips16, (unsigned)others), dim3(256), 0, s, fe));
                }
                CHECK_LAUNCH();
                return ok();
            }
            const int64_t strips = ceil_div(fe.w[fe.nd_out - 1], 128) * ceil_div(fe.w[fe.dt], 32);
            dim3 grid((unsigned)strips, (unsigned)others);
            if (fe.in_bf16 && fe.out_bf16) CUDA_TRY(launch(eop_affine_transpose_kernel<uint16_t>, grid, dim3(256), 0, s, fe));
            else if (!fe.in_bf16 && !fe.out_bf16) CUDA_TRY(launch(eop_affine_transpose_kernel<uint32_t>, grid, dim3(256), 0, s, fe));
            else return fail(OLLIE_E_UNSUPPORTED, "internal: converting transpose");
            CHECK_LAUNCH();
            return ok();
        }
    }
    EopDev dv;
    st = compile_eop(eop, inputs, output, &dv);
    if (st != OLLIE_OK) return st;
    const int64_t blocks = std::min<int64_t>(ceil_div(dv.out_elems, 256), (int64_t)num_sms() * 32);
    CUDA_TRY(launch(eop_eval_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, s, dv));
    CHECK_LAUNCH();
    return ok();
}

extern "C" ollie_status ollie_plan_describe(const ollie_conv_shape *s, ollie_dtype dtype, int plan, int transposed,
                                            char *buf, size_t len) {
    int64_t OH, OW;
    ollie_status st = check_shape(s, transposed, &OH, &OW);
    if (st != OLLIE_OK) return st;
    if (!buf || len == 0) return fail(OLLIE_E_INVALID, "null buffer");
    const bool tf32 = dtype == OLLIE_TF32;
    const int rp = resolve_plan(s, dtype, plan, transposed);
    if (rp == OLLIE_PLAN_FUSED) {
        FusedArgs a;
        if (!plan_fused(s, tf32, transposed, &a, OH, OW)) return fail(OLLIE_E_UNSUPPORTED, "no fused plan");
        snprintf(buf, len,
                 "fused XB=%d Yb=%d Xb=%d Yp=%d MT=%d FS=%d f_slices=%d resident=%d nbuf=%d na=%d nb=%d BK=%d "
                 "kchunks=%d tiles=%d grid=%d smem=%zu classes=%d phases=%d ist=%d taps=%d sw128=%d ctas_per_sm=%d "
                 "pair=%d wbox=%dx%d ksplit=%d ipt=%d tma_y=%d grp8=%d",
                 a.XB, a.Yb, a.Xb, a.Yp, a.MT, a.FS, a.f_slices, a.resident, a.nbuf, a.na, a.nb, a.BK, a.kchunks,
                 a.num_tiles, fused_grid(a), fused_smem_bytes(a), a.nclass, a.nph, a.ist, a.max_taps, a.sw128,
                 a.tmem_cols == 256 ? 2 : 1, a.pair, a.grb, a.nsb, a.ksplit, a.ipt, a.tma_y, a.grp8);
    } else if (is_rowstream_plan(rp)) {
        RsArgs a;
        if (!plan_rowstream(s, tf32, transposed, OH, OW, &a, rowstream_mode_of(rp))) return fail(OLLIE_E_UNSUPPORTED, "no row-streaming plan");
        snprintf(buf, len,
                 "rowstream %s R=%d S=%d sub=%d N=%d NP=%d ring=%d mtr=%d rowbytes=%d ksteps=%d tmem_rows=%d grid=%d smem=%zu",
                 a.direct ? "direct" : "ysum", a.R, a.S, a.sub, a.N, a.NP, a.ring, a.mtr, a.rowbytes, a.ksteps, a.nt, rowstream_grid(a), rs_smem_bytes(a));
    } else if (rp == OLLIE_PLAN_SMALL) {
        if (!small_supported(s, transposed, OH, OW)) return fail(OLLIE_E_UNSUPPORTED, "no small plan");
        snprintf(buf, len, "small (fused program on CUDA cores, one thread per output, %lld outputs)",
                 (long long)(s->n * OH * OW * s->f));
    } else if (rp == OLLIE_PLAN_GEMM_RED) {
        snprintf(buf, len, "gemm_red BN=%d (%s as fp32 L2 reductions in the GEMM epilogue) + finish",
                 gemm_bn(s->n * s->h * s->w, s->r * s->s * s->f), transposed ? "selective add" : "OffsetAdd");
    } else if (is_identity_offset_add(s, transposed)) {
        snprintf(buf, len, "unfused-identity gemm BN=%d (OffsetAdd eliminated)", gemm_bn(s->n * s->h * s->w, s->r * s->s * s->f));
    } else {
        snprintf(buf, len, "unfused gemm BN=%d ldT=%lld + %s", gemm_bn(s->n * s->h * s->w, s->r * s->s * s->f), (long long)ldT_of(s),
                 transposed ? "selective_add" : "offset_add");
    }
    return ok();
}

// Debug hook (not part of include/ollie.h): route the fused kernel's per-CTA timestamps into a
// caller-owned device buffer of >= 16 * grid int64 (nullptr switches tracing off).
extern "C" void ollie_debug_set_trace(void *dev_buf) { g_fc_trace = reinterpret_cast<long long *>(dev_buf); }
// Debug hook (not part of include/ollie.h): force fused-plan parameters for sweeps
// (mt / fs <= 0 and resident < 0 mean "auto").
extern "C" void ollie_debug_force_plan(int mt, int fs, int resident) {
    g_force_mt = mt;
    g_force_fs = fs;
    g_force_res = resident;
}
// Debug hook (not part of include/ollie.h): -1 auto, 0 single-CTA plans only, 1 CTA-pair plans only.
extern "C" void ollie_debug_force_pair(int pair) { g_force_pair = pair; }
// Debug hook (not part of include/ollie.h): 0 auto, else the fused plan's CTAs per SM.
extern "C" void ollie_debug_force_occ(int occ) { g_force_occ = occ; }
// Debug hook (not part of include/ollie.h): -1 auto, else only plans with this split-K factor.
extern "C" void ollie_debug_force_ksplit(int ks) { g_force_ks = ks; }
// Debug hook (not part of include/ollie.h): 0 auto, else only plans with this many images per tile.
extern "C" void ollie_debug_force_ipt(int ipt) { g_force_ipt = ipt; }
// Debug hook (not part of include/ollie.h): -1 auto, 0 consecutive-row lanes only, 1 grp8 lanes only.
extern "C" void ollie_debug_force_grp8(int g8) { g_force_g8 = g8; }


// ------------------------------------------------------------------------ autotune
static ollie_status autotune_impl(const ollie_conv_shape *s, ollie_dtype dtype, int transposed, const void *x,
                                  const void *wp, void *y, void *ws, size_t ws_bytes, void *flush_buf,
                                  size_t flush_bytes, ollie_stream_t stream_, float *best_us);

extern "C" ollie_status ollie_autotune_derived(const ollie_conv_shape *s, ollie_dtype dtype, int transposed,
                                               const void *x, const void *wp, void *y, void *ws, size_t ws_bytes,
                                               ollie_stream_t stream_, float *best_us) {
    return autotune_impl(s, dtype, transposed, x, wp, y, ws, ws_bytes, nullptr, 0, stream_, best_us);
}

extern "C" ollie_status ollie_autotune_derived_cold(const ollie_conv_shape *s, ollie_dtype dtype, int transposed,
                                                    const void *x, const void *wp, void *y, void *ws, size_t ws_bytes,
                                                    void *flush_buf, size_t flush_bytes, ollie_stream_t stream_,
                                                    float *best_us) {
    if (!flush_buf || flush_bytes == 0) return fail(OLLIE_E_INVALID, "cold autotune needs a flush buffer");
    return autotune_impl(s, dtype, transposed, x, wp, y, ws, ws_bytes, flush_buf, flush_bytes, stream_, best_us);
}

static ollie_status autotune_impl(const ollie_conv_shape *s, ollie_dtype dtype, int transposed, const void *x,
                                  const void *wp, void *y, void *ws, size_t ws_bytes, void *flush_buf,
                                  size_t flush_bytes, ollie_stream_t stream_, float *best_us) {
    int64_t OH, OW;
    ollie_status st = check_shape(s, transposed, &OH, &OW);
    if (st != OLLIE_OK) return st;
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32) return fail(OLLIE_E_UNSUPPORTED, "dtype must be BF16 or TF32");
    if (!x || !wp || !y) return fail(OLLIE_E_INVALID, "null pointer");
    cudaStream_t stream = (cudaStream_t)stream_;
    const bool tf32 = dtype == OLLIE_TF32;
    // identity OffsetAdd (1x1, a6): the "unfused" candidate is the GEMM writing Y directly; the fused
    // and row-streaming kernels (one tap) compete with it
    const bool ident = is_identity_offset_add(s, transposed);
    PlanEntry *e = plan_entry_mut(s, tf32, transposed, OH, OW);
    const int64_t M = s->n * s->h * s->w;
    const size_t need = ident ? 0 : (size_t)M * (size_t)ldT_of(s) * sizeof(float);
    const bool unfused_ok = (ident || (ws && ws_bytes >= need)) && !(transposed && s->dilation != 1);
    std::vector<FusedArgs> cands;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        if (e->ok) cands = e->cands;
    }
    // OLLIE_TUNE_FILE: record each decision ("<shape key> <f k | u | r>"), and replay a recorded one
    // instead of measuring -- profiler runs (ncu serialises and replays kernels, so timing there is
    // meaningless) then execute exactly the plans the timed bench chose
    const char *tune_file = getenv("OLLIE_TUNE_FILE");
    char key[256];
    snprintf(key, sizeof key, "%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%d,%d,%d",
             (long long)s->n, (long long)s->c, (long long)s->h, (long long)s->w, (long long)s->f, (long long)s->r,
             (long long)s->s, (long long)s->pad, (long long)s->stride, (long long)s->dilation,
             (long long)s->output_padding, (int)tf32, transposed, num_sms());
    if (tune_file) {
        if (FILE *fp = fopen(tune_file, "r")) {
            char k2[256], d[16];
            int idx = -1;
            bool hit = false;
            while (fscanf(fp, "%255s %15s %d", k2, d, &idx) == 3) {
                if (strcmp(k2, key) != 0) continue;
                std::lock_guard<std::mutex> g(g_plan_mu);
                if (d[0] == 'f' && idx >= 0 && idx < (int)cands.size()) { e->args = cands[idx]; e->tuned = 1; hit = true; }
                else if (d[0] == 'u' && unfused_ok) { e->tuned = 2; hit = true; }
                else if (d[0] == 'r') { e->tuned = 3; hit = true; }
                else if (d[0] == 's' && rowstream_supported(s, tf32, transposed, OH, OW, 0)) { e->tuned = OLLIE_PLAN_ROWSTREAM_YSUM; hit = true; }
                else if (d[0] == 'd' && rowstream_supported(s, tf32, transposed, OH, OW, 1)) { e->tuned = OLLIE_PLAN_ROWSTREAM_DIRECT; hit = true; }
                else if (d[0] == 'c' && small_supported(s, transposed, OH, OW)) { e->tuned = OLLIE_PLAN_SMALL; hit = true; }
            }
            fclose(fp);
            if (hit) {
                if (best_us) *best_us = 0.f;
                return derived_layer(s, dtype, x, wp, y, ws, ws_bytes, OLLIE_PLAN_AUTO, stream, transposed);
            }
        }
    }
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    // Each candidate is timed as a burst of back-to-back launches between two events, so the
    // programmatic-dependent-launch overlap a candidate gets inside a CUDA graph of layers (its
    // prologue under the previous kernel's tail; cluster kernels get none) is part of its time.
    constexpr int kBurst = 5;
    auto time_it = [&](auto &&run) -> float {
        if (run() != OLLIE_OK) return 1e30f;                  // warm-up (and plan check)
        float best = 1e30f;
        if (flush_buf) {
            // cold: the caller's buffer (>= 2x L2) is rewritten before every timed launch, so each
            // candidate is measured from an evicted L2 -- the condition of a flushed benchmark step
            // and of a layer whose weights were evicted by the rest of the network
            float sum = 0.f;
            constexpr int kCold = 5;
            for (int r = 0; r < kCold; ++r) {
                cudaMemsetAsync(flush_buf, r & 0xFF, flush_bytes, stream);
                cudaEventRecord(e0, stream);
                if (run() != OLLIE_OK) return 1e30f;
                cudaEventRecord(e1, stream);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                sum += ms;
            }
            return sum / kCold;   // mean: event timestamps are coarse (~2 us) against one short launch
        }
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0, stream);
            for (int b = 0; b < kBurst; ++b)
                if (run() != OLLIE_OK) return 1e30f;
            cudaEventRecord(e1, stream);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms / kBurst);
        }
        return best;
    };
    float best = 1e30f;
    int best_k = -1;                                          // -1: unfused
    for (int k = 0; k < (int)cands.size(); ++k) {
        {
            std::lock_guard<std::mutex> g(g_plan_mu);
            e->args = cands[k];
        }
        const float t = time_it([&] { return run_fused(s, tf32, transposed, x, wp, y, OH, OW, stream); });
        if (t < best) { best = t; best_k = k; }
    }
    float t_unf = 1e30f;
    if (ident) {
        t_unf = time_it([&] { return run_gemm(M, s->f, s->c, tf32, x, wp, y, s->f, !tf32, stream); });
    } else if (unfused_ok && aligned16(ws)) {
        t_unf = time_it([&] {
            ollie_status r = run_gemm(M, s->r * s->s * s->f, s->c, tf32, x, wp, ws, ldT_of(s), false, stream);
            if (r != OLLIE_OK) return r;
            return run_offset_add(s, transposed, (const float *)ws, ldT_of(s), !tf32, y, OH, OW, stream);
        });
    }
    float t_red = 1e30f;
    const bool red_ok = red_supported(s, transposed) && ws && ws_bytes >= red_acc_bytes(s, OH, OW) && aligned16(ws);
    if (red_ok)
        t_red = time_it([&] { return run_gemm_red(s, transposed, tf32, x, wp, (float *)ws, y, OH, OW, stream, nullptr); });
    float t_rs = 1e30f, t_rd = 1e30f;     // the two row-streaming forms (ysum, direct)
    if (rowstream_supported(s, tf32, transposed, OH, OW, 0))
        t_rs = time_it([&] { return run_rowstream(s, tf32, transposed, x, wp, y, OH, OW, stream, nullptr, 0); });
    if (rowstream_supported(s, tf32, transposed, OH, OW, 1))
        t_rd = time_it([&] { return run_rowstream(s, tf32, transposed, x, wp, y, OH, OW, stream, nullptr, 1); });
    float t_sm = 1e30f;                   // the CUDA-core program for tiny layers
    if (small_supported(s, transposed, OH, OW))
        t_sm = time_it([&] { return run_small(s, tf32, transposed, x, wp, y, OH, OW, stream, nullptr); });
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const bool any_timed = best < 1e29f || t_unf < 1e29f || t_red < 1e29f || t_rs < 1e29f || t_rd < 1e29f || t_sm < 1e29f;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        if (!cands.empty()) e->args = cands[best_k >= 0 ? best_k : 0];
        // record a decision only when some plan actually ran and was timed: a failed tuning leaves
        // AUTO to the cost model instead of pinning it to an unmeasured plan
        if (any_timed) {
            const float t_min = std::min(std::min(std::min(std::min(best, t_unf), std::min(t_red, t_rs)), t_rd), t_sm);
            // the CUDA-core plan has no tensor-memory / TMA setup: within 15% of the best warm burst it
            // is also the fastest from a cold L2 (motivating example: 4.3 vs 8.7 us flushed, rowstream
            // 4.0 vs 4.2 us warm), so it wins those ties
            if (t_sm == t_min || t_sm <= 1.15f * t_min) e->tuned = OLLIE_PLAN_SMALL;
            else if (t_rd == t_min) e->tuned = OLLIE_PLAN_ROWSTREAM_DIRECT;
            else if (t_rs == t_min) e->tuned = OLLIE_PLAN_ROWSTREAM_YSUM;
            else if (t_red == t_min) e->tuned = 3;
            else e->tuned = (t_unf == t_min || best_k < 0) ? 2 : 1;
        }
    }
    if (best_us) *best_us = 1e3f * std::min(std::min(std::min(std::min(best, t_unf), std::min(t_red, t_rs)), t_rd), t_sm);
    if (!any_timed) return fail(OLLIE_E_UNSUPPORTED, "no runnable plan to tune");
    if (tune_file) {
        if (FILE *fp = fopen(tune_file, "a")) {
            const int t = e->tuned;
            fprintf(fp, "%s %s %d\n", key,
                    t == 1 ? "f" : t == 2 ? "u" : t == 3 ? "r" : t == OLLIE_PLAN_ROWSTREAM_DIRECT ? "d" :
                    t == OLLIE_PLAN_SMALL ? "c" : "s",
                    t == 1 ? best_k : 0);
            fclose(fp);
        }
    }
    // leave y holding the chosen plan's result
    return derived_layer(s, dtype, x, wp, y, ws, ws_bytes, OLLIE_PLAN_AUTO, stream, transposed);
}


// ------------------------------------------------------------------------ NEXT-4 G2BMM
static int g_g2_dbg = 0;
// Debug hook (not part of include/ollie.h): G2BMM epilogue ablations (bit 0 skip stores, bit 1 skip staging).
extern "C" void ollie_debug_g2bmm_flags(int f) { g_g2_dbg = f; }
template <bool TF32, int CS>
static ollie_status launch_g2bmm_t(const CUtensorMap &ta, const CUtensorMap &tb, const G2Args &g, size_t smem,
                                   cudaStream_t stream) {
    auto kern = g2bmm_kernel<TF32, CS>;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_done[dev & 63]) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done[dev & 63] = true;
    }
    const int grid = (int)std::min<int64_t>(g.num_items, num_sms());
    CUDA_TRY(launch(kern, dim3(grid), dim3(g2_threads(CS)), smem, stream, ta, tb, g));
    return OLLIE_OK;
}

extern "C" ollie_status ollie_g2bmm(int64_t batch, int64_t L, int64_t K, int64_t W, int64_t d, ollie_dtype dtype,
                                    const void *A, const void *B, void *out, int64_t ldo, int form,
                                    ollie_stream_t stream_) {
    if (batch <= 0 || L <= 0 || K <= 0 || W < 0 || d < 1) return fail(OLLIE_E_INVALID, "G2BMM: batch, L, K > 0, W >= 0, d >= 1");
    if (dtype != OLLIE_BF16 && dtype != OLLIE_TF32) return fail(OLLIE_E_UNSUPPORTED, "G2BMM dtype must be BF16 or TF32");
    if (form != OLLIE_G2BMM_DERIVED && form != OLLIE_G2BMM_DIRECT) return fail(OLLIE_E_INVALID, "unknown G2BMM form %d", form);
    if (!A || !B || !out) return fail(OLLIE_E_INVALID, "null pointer");
    if (ldo < 2 * W + 1) return fail(OLLIE_E_INVALID, "ldo < 2W + 1");
    if (batch > INT32_MAX || L > INT32_MAX || W > (INT32_MAX - 1) / 2)
        return fail(OLLIE_E_UNSUPPORTED, "G2BMM extents exceed int32");
    const bool tf32 = dtype == OLLIE_TF32;
    const int es = tf32 ? 4 : 2;
    if (K * es != 128) return fail(OLLIE_E_UNSUPPORTED, "G2BMM implemented for K*sizeof(elem) == 128 (K = 64 bf16 / 32 tf32)");
    if (!aligned16(A) || !aligned16(B)) return fail(OLLIE_E_ALIGN, "A / B must be 16-byte aligned");
    // the epilogue picks 16-byte (ldo % 8 == 0) or 4-byte stores from the pitch: the base must match
    if (!aligned16(out)) return fail(OLLIE_E_ALIGN, "out must be 16-byte aligned");
    if (batch * L * (2 * W + 1) >= (1ll << 40) || L >= (1ll << 30)) return fail(OLLIE_E_UNSUPPORTED, "G2BMM extents too large");
    // derived: tiles over one residue class (rows r + d*u, stride d), band columns dense (cs = 1);
    // direct: contiguous rows, band columns d apart (cs = d)
    const bool derived = form == OLLIE_G2BMM_DERIVED || d == 1;
    const int stride = derived ? (int)d : 1;
    const int cs = derived ? 1 : (int)d;
    if (cs > 4) return fail(OLLIE_E_UNSUPPORTED, "direct G2BMM form implemented for d <= 4 (use the derived form)");
    if (stride > 8) return fail(OLLIE_E_UNSUPPORTED, "G2BMM derived form implemented for d <= 8 (TMA element stride)");
    G2Args g{};
    g.batch = (int)batch; g.L = (int)L; g.W = (int)W; g.d = (int)d;
    g.stride = stride; g.cs = cs;
    g.nw = (int)(2 * W + 1);
    g.nwb = (g.nw + 31) / 32;
    const int last_col = 96 + cs * 32 * (g.nwb - 1) + 32 * (cs + 1);
    g.nchunks = (last_col + G2_BN - 1) / G2_BN;
    g.rpb = 128;                              // rows per TMA box: a power of two with rpb * stride <= 256
    while (g.rpb * stride > 256) g.rpb /= 2;
    g.nres = derived ? (int)d : 1;
    const int64_t rows_per_res = derived ? ceil_div(L, d) : L;
    g.tiles_r = (int)ceil_div(rows_per_res, 128);
    if (batch * g.nres * (int64_t)g.tiles_r > INT32_MAX) return fail(OLLIE_E_UNSUPPORTED, "G2BMM work items exceed int32");
    g.num_items = (int)(batch * g.nres * g.tiles_r);
    g.ldo = ldo;
    g.out = out;
    g.dbg = g_g2_dbg;
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
    const CUtensorMapDataType dt = tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta, tb;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)L, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)(K * es), (cuuint64_t)(L * K * es)};
    cuuint32_t box[3] = {(cuuint32_t)K, (cuuint32_t)(g.rpb * stride), 1};   // rpb rows, element stride `stride`
    cuuint32_t estr[3] = {1, (cuuint32_t)stride, 1};
    for (int t = 0; t < 2; ++t) {
        CUresult r = enc(t == 0 ? &ta : &tb, dt, 3, const_cast<void *>(t == 0 ? A : B), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(OLLIE_E_CUDA, "cuTensorMapEncodeTiled (G2BMM) failed (%d)", (int)r);
    }
    const size_t smem = 1024 + 128 * 128 + G2_NBUF * G2_BN * 128 + (size_t)g2_epi_warps(cs) * 32 * g2_stage_pitch(cs) * 4 + 512;
    cudaStream_t stream = (cudaStream_t)stream_;
    ollie_status st;
    switch (cs) {
        case 1: st = tf32 ? launch_g2bmm_t<true, 1>(ta, tb, g, smem, stream) : launch_g2bmm_t<false, 1>(ta, tb, g, smem, stream); break;
        case 2: st = tf32 ? launch_g2bmm_t<true, 2>(ta, tb, g, smem, stream) : launch_g2bmm_t<false, 2>(ta, tb, g, smem, stream); break;
        case 3: st = tf32 ? launch_g2bmm_t<true, 3>(ta, tb, g, smem, stream) : launch_g2bmm_t<false, 3>(ta, tb, g, smem, stream); break;
        default: st = tf32 ? launch_g2bmm_t<true, 4>(ta, tb, g, smem, stream) : launch_g2bmm_t<false, 4>(ta, tb, g, smem, stream); break;
    }
    return st == OLLIE_OK ? ok() : st;
}
