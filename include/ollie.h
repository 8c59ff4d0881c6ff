/*
 * ollie.h -- C ABI of libollie, the B200 (sm_100a) runtime of the programs Ollie's
 * expression derivation produces for Conv2d / ConvTranspose2d (arXiv 2208.02025).
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n (assembled copy P:670-1704),
 * "S:n" = SPEC.md line n, "SURVEY" = /root/repo/SURVEY.md.
 *
 * The hot path:
 *   a0  weight DLT, evaluated once at "compile time"  (Eq. layout-K)
 *   a1  input layout-A  A'[t1*W+t2, c] = A[t1,t2,c]   (Eq. layout-A) -- the identity
 *       on NHWC memory, eliminated without a launch
 *   a2  merged Matmul T[m, (i,j,f)] = sum_c X[m,c] * W'[(i,j,f), c]
 *   a3  OffsetAdd eOperator (E7)
 *   a4  ConvTranspose selective addition
 *   a5  fused eOperator pair (chain rule)
 *   a7  generic scoped eOperator L_x Sum_y f(T[tau(x,y)])
 *   a8  OffsetAdd / selective add fused into the GEMM epilogue (instance of P:955-965)
 *
 * Conventions (apply to every entry point):
 *  - Ownership: every data pointer is a CALLER-OWNED CUDA DEVICE pointer.  The library
 *    never allocates or frees device memory, never retains a pointer after the call
 *    returns, and never synchronises the device.  Descriptor structs are read during
 *    the call only (host memory, caller-owned).
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  All device
 *    work of a call is enqueued on it, asynchronously.
 *  - Errors: status codes only; no C++ exception crosses the ABI.  All validation
 *    happens BEFORE any launch, so a call that fails validation has no side effect.
 *    ollie_last_error() returns a thread-local, human-readable detail string.
 *  - Threading: calls are stateless and reentrant; ordering is by `stream` only.
 *  - Layouts: activations are NHWC (the paper's HWC "A[t1,t2,c]");
 *    Conv2d weights are PyTorch [f][c][r][s], ConvTranspose2d weights [c][f][r][s];
 *    the prepared (merged) weight is W'[(i*S+j)*F+f][c] (K-major: the transpose of the
 *    paper's K'[c, r*S*F+s*F+f]); the intermediate T is [n*h*w][r*s*f] with columns in
 *    (i, j, f) order.
 *  - dtypes: OLLIE_BF16 -- x, w, w_prep, y are bf16, accumulation fp32, T fp32;
 *            OLLIE_TF32 -- x, w, w_prep, y are fp32 in memory, TF32 tensor-core MMA,
 *                          fp32 accumulation (the paper's fp32, reading Q1/Q14).
 *  - Alignment: x rows (c * sizeof(elem)) must be a multiple of 16 bytes and every
 *    base pointer 16-byte aligned (TMA rule), else OLLIE_E_ALIGN; channel-pad the
 *    activation first with an eOperator.
 */
#ifndef OLLIE_H_
#define OLLIE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OLLIE_ABI_VERSION 1

typedef void *ollie_stream_t; /* a cudaStream_t */

typedef enum {
    OLLIE_OK = 0,
    OLLIE_E_INVALID = -1,     /* bad shape / range / arity / undeclared iterator       */
    OLLIE_E_UNSUPPORTED = -2, /* valid but not implemented (dtype combination, plan)         */
    OLLIE_E_WORKSPACE = -3,   /* ws too small or NULL when the unfused plan needs T           */
    OLLIE_E_OOB = -4,         /* an index map reads outside the pad band              */
    OLLIE_E_ALIGN = -5,       /* base pointer / row stride violates the 16-byte TMA rule      */
    OLLIE_E_CUDA = -6         /* CUDA launch / runtime error; detail in ollie_last_error()    */
} ollie_status;

typedef enum {
    OLLIE_BF16 = 0, /* bfloat16 storage                                   */
    OLLIE_TF32 = 1, /* fp32 storage, TF32 tensor-core operands             */
    OLLIE_FP32 = 2  /* fp32 storage, fp32 arithmetic (eOperators, T, y)    */
} ollie_dtype;

/* The problem statement of a layer (SPEC OpNode attrs "strides, dilation,
 * pads").  Offsets follow PyTorch: kernel tap i reads input row oh*stride - pad
 * + i*dilation (reading Q2 of DESIGN.md: the paper's centred r in [-1,1] is i - pad). */
typedef struct {
    int64_t n, c, h, w;     /* input: batch, channels, height, width                 */
    int64_t f, r, s;        /* output channels, kernel height (R), kernel width (S)  */
    int32_t pad, stride, dilation;
    int32_t output_padding; /* ConvTranspose2d only (PyTorch semantics, reading Q9)  */
} ollie_conv_shape;

/* Plans of the derived layer:
 *   AUTO     -- measured choice (first call per shape: ollie_autotune_derived) or the cost model;
 *               the choice is process-wide, so re-query ollie_workspace_bytes(AUTO) after tuning --
 *               a call whose ws cannot hold the tuned plan's T / accumulator runs FUSED instead
 *   FUSED    -- a8: OffsetAdd / selective add fused into the GEMM, T only in TMEM / smem
 *   UNFUSED  -- the literal two-kernel program: merged GEMM writes T (workspace), then a3 / a4
 *   GEMM_RED -- merged GEMM over full n*h*w rows whose epilogue adds every T element into its
 *               output pixel as fp32 L2 reductions (red.global.add.v4.f32; "the L2 reduction",
 *               P:1580), then Y = epilogue(acc): the workspace holds the fp32 accumulator
 *               [n][OH][OW][f] (zeroed by the call); f % 4 == 0; summation order is not fixed
 *               (fp32 atomics: results are deterministic only up to rounding, reading Q12).
 *   ROWSTREAM -- a8 for narrow outputs: summation splitting of the r*s taps into kernel
 *               columns (accumulated by the tensor core from column-shifted A operands) and kernel
 *               rows (on the MMA's N, N = r*f; their OffsetAdd done in the epilogue by adding the
 *               TMEM accumulators of consecutive input rows); a ConvTranspose2d first becomes the
 *               stride-1 program over the union of its output residue classes' input offsets,
 *               classes on N too (expression splitting; the epilogue writes the classes
 *               interleaved -- the fused pair of P:1437-1438).  Each input row is streamed through
 *               shared memory once.  Plannable for dilation 1, Conv2d stride 1 or any
 *               ConvTranspose2d stride, c*sizeof(elem) <= 128, w <= 512, f <= 64 and
 *               r' * stride^2 * f <= 64 with stride^2 * f in {4, 8, 12, 16} (r', s' <= 16 the
 *               stride-1 program's kernel, its column padding <= 8); else OLLIE_E_UNSUPPORTED.
 *               No workspace.  This is the "ysum" form (OLLIE_PLAN_ROWSTREAM_YSUM).
 *               The "direct" form (OLLIE_PLAN_ROWSTREAM_DIRECT, Conv2d only) puts only the f
 *               output channels on N and every one of the r*s taps on an A-row shift over the r
 *               input rows resident in shared memory: one TMEM accumulator per OUTPUT row, no
 *               epilogue sum (the OffsetAdd of all r*s offsets done by the tensor core,
 *               P:992-996 applied to both tap dimensions).  Plannable for Conv2d stride 1,
 *               dilation 1, f <= 64, s <= 9, the same channel / width limits.
 *               OLLIE_PLAN_ROWSTREAM runs the planner's form: direct when r*s*ceil(c*es/32)
 *               <= 12 MMAs per M-tile, else ysum (else direct).
 *   SMALL    -- a8 on CUDA cores for layers of at most 2^22 multiply-adds (the paper's motivating
 *               example): one thread per output element evaluates the fused program
 *               Y[m, f] = Sum_{i,j} Sum_c X[m + Delta_ij, c] W'[(i,j,f), c] (traversal merging of
 *               OffsetAdd o Matmul; ConvTranspose2d: the selected taps of each output,
 *               P:1575-1580) in fp32, taps in (i, j) order, channels in order -- a single launch with
 *               no tensor-memory setup, for problems whose tensor-core kernels are launch-latency
 *               bound.  TF32 layers are computed in full fp32 (within the TF32 bar).  No workspace;
 *               OLLIE_E_UNSUPPORTED above the size limit.  AUTO measures it for such layers. */
enum { OLLIE_PLAN_AUTO = 0, OLLIE_PLAN_FUSED = 1, OLLIE_PLAN_UNFUSED = 2, OLLIE_PLAN_GEMM_RED = 3,
       OLLIE_PLAN_ROWSTREAM = 4, OLLIE_PLAN_ROWSTREAM_YSUM = 5, OLLIE_PLAN_ROWSTREAM_DIRECT = 6,
       OLLIE_PLAN_SMALL = 7 };

/* ---------------------------------------------------------------------------------
 * Versioning and errors
 * --------------------------------------------------------------------------------- */
int         ollie_abi_version(void);
const char *ollie_status_string(ollie_status st);
const char *ollie_last_error(void); /* thread-local detail of the last failing call ("" if none) */

/* Output spatial size of the layer (Conv2d if transposed == 0, else ConvTranspose2d).
 * Returns OLLIE_E_INVALID for a non-positive size. */
ollie_status ollie_output_hw(const ollie_conv_shape *shape, int transposed, int64_t *oh, int64_t *ow);

/* ---------------------------------------------------------------------------------
 * a0 -- compile-time weight DLT (Eq. layout-K; compile-time expression
 * evaluation):   w_prep[(i*S+j)*F+f][c] = W[f][c][i][j]   (Conv2d)
 *                             w_prep[(i*S+j)*F+f][c] = W[c][f][i][j]   (ConvTranspose2d)
 * w (input) and w_prep (output, ollie_prepared_weight_bytes() bytes) are device
 * buffers of `dtype` elements (BF16 or TF32).  Pure indexing: bit-exact.
 * --------------------------------------------------------------------------------- */
size_t       ollie_prepared_weight_bytes(const ollie_conv_shape *shape, ollie_dtype dtype);
ollie_status ollie_prepare_weight_conv2d(const ollie_conv_shape *shape, ollie_dtype dtype,
                                         const void *w_fcrs, void *w_prep, ollie_stream_t stream);
ollie_status ollie_prepare_weight_convtranspose2d(const ollie_conv_shape *shape, ollie_dtype dtype,
                                                  const void *w_cfrs, void *w_prep, ollie_stream_t stream);

/* Workspace for the unfused plan: T fp32 [n*h*w][ldT] with ldT = r*s*f rounded up to a
 * multiple of 4 (16-byte rows).  Returns 0 when `plan` resolves to the fused plan. */
size_t ollie_workspace_bytes(const ollie_conv_shape *shape, ollie_dtype dtype, int plan, int transposed);

/* ---------------------------------------------------------------------------------
 * The derived layer: a1 (eliminated) + a2 merged GEMM + a3 OffsetAdd (Conv2d) or a4
 * selective addition (ConvTranspose2d), unfused (T through `ws`) or fused (a8, T lives
 * only in TMEM / shared memory).
 *   x_nhwc : [n][h][w][c]            dtype elements (device)
 *   w_prep : [r*s*f][c]              from ollie_prepare_weight_* (device); read-only for the
 *                                    layer's lifetime: the fused kernel loads it before waiting
 *                                    on the previous kernel of the stream (programmatic dependent
 *                                    launch), which the weight DLT allows by never triggering early
 *   y_nhwc : [n][OH][OW][f]          dtype elements, fully overwritten (device)
 *   ws     : ollie_workspace_bytes() bytes (device), may be NULL if that is 0
 *   plan   : OLLIE_PLAN_AUTO / FUSED / UNFUSED / GEMM_RED / ROWSTREAM
 * ConvTranspose2d requires dilation == 1 (the configured workloads); else UNSUPPORTED.
 * --------------------------------------------------------------------------------- */
ollie_status ollie_conv2d_derived(const ollie_conv_shape *shape, ollie_dtype dtype,
                                  const void *x_nhwc, const void *w_prep, void *y_nhwc,
                                  void *ws, size_t ws_bytes, int plan, ollie_stream_t stream);
ollie_status ollie_convtranspose2d_derived(const ollie_conv_shape *shape, ollie_dtype dtype,
                                           const void *x_nhwc, const void *w_prep, void *y_nhwc,
                                           void *ws, size_t ws_bytes, int plan, ollie_stream_t stream);

/* ---------------------------------------------------------------------------------
 * NEXT-3 -- element-wise epilogue fused into the kernel that writes Y ("OffsetAdd ...
 * fused with following element-wise operators"; reading Q19):
 *     v = acc + bias[f] + residual[n][oh][ow][f];     Y = act(v)
 *   bias     : fp32 [f] (device) or NULL
 *   residual : [n][OH][OW][f] in Y's storage dtype (device) or NULL; may alias y_nhwc
 *   act      : OLLIE_ACT_NONE, OLLIE_ACT_RELU (max(v, 0)) or OLLIE_ACT_PRELU
 *              (v > 0 ? v : alpha[f] * v)
 *   alpha    : fp32 [f] PReLU slopes (device), required for OLLIE_ACT_PRELU
 * Arithmetic is fp32 on the fp32 accumulator, then the usual RNE store; every plan applies it
 * (fused epilogue, OffsetAdd / selective-add kernel, or the identity plan's GEMM epilogue).
 * Errors: E_INVALID for an unknown act or PReLU without alpha (before any launch).
 * ollie_*_derived_ex(..., epilogue = NULL, ...) == ollie_*_derived(...).
 * --------------------------------------------------------------------------------- */
enum { OLLIE_ACT_NONE = 0, OLLIE_ACT_RELU = 1, OLLIE_ACT_PRELU = 2 };
typedef struct {
    const float *bias;
    const void *residual;
    int32_t act;
    const float *alpha;
} ollie_epilogue;

ollie_status ollie_conv2d_derived_ex(const ollie_conv_shape *shape, ollie_dtype dtype,
                                     const void *x_nhwc, const void *w_prep, void *y_nhwc,
                                     void *ws, size_t ws_bytes, int plan,
                                     const ollie_epilogue *epilogue, ollie_stream_t stream);
ollie_status ollie_convtranspose2d_derived_ex(const ollie_conv_shape *shape, ollie_dtype dtype,
                                              const void *x_nhwc, const void *w_prep, void *y_nhwc,
                                              void *ws, size_t ws_bytes, int plan,
                                              const ollie_epilogue *epilogue, ollie_stream_t stream);

/* Introspection: writes a one-line description of the plan `plan` resolves to for this layer
 * (kernel choice, tile geometry, f-slice, stages) into buf (NUL-terminated, truncated to len).
 * Host-only; no launch. */
ollie_status ollie_plan_describe(const ollie_conv_shape *shape, ollie_dtype dtype, int plan, int transposed,
                                 char *buf, size_t len);

/* Plan selection by measurement (the paper keeps the candidate with the best measured
 * performance): times the planner's fused candidates (best few by its cost model), the
 * row-streaming plan when the layer admits it and, when ws can hold T, the unfused plan, on `stream` (synchronizing it), and makes
 * OLLIE_PLAN_AUTO use the fastest for this (shape, dtype, direction) from then on, process-wide.
 * x / w_prep / y / ws as for ollie_conv2d_derived; y ends up holding the layer's result.
 * best_us (may be NULL) receives the winner's time in microseconds.  Not for capture into a
 * CUDA graph. */
ollie_status ollie_autotune_derived(const ollie_conv_shape *shape, ollie_dtype dtype, int transposed,
                                    const void *x_nhwc, const void *w_prep, void *y_nhwc, void *ws,
                                    size_t ws_bytes, ollie_stream_t stream, float *best_us);
/* Same, measuring every candidate from an evicted L2: flush_buf (caller-owned device memory, >= 2x
 * the L2 size for a full eviction) is rewritten by cudaMemsetAsync before each timed launch, and each
 * candidate's time is the mean of 5 such single launches.  For workloads whose layers start cold (a
 * flushed benchmark step; weights evicted by the rest of a network).  flush_buf NULL / flush_bytes 0:
 * OLLIE_E_INVALID. */
ollie_status ollie_autotune_derived_cold(const ollie_conv_shape *shape, ollie_dtype dtype, int transposed,
                                         const void *x_nhwc, const void *w_prep, void *y_nhwc, void *ws,
                                         size_t ws_bytes, void *flush_buf, size_t flush_bytes,
                                         ollie_stream_t stream, float *best_us);

/* a2 standalone (the merged Matmul of P:1342-1352 on tcgen05 tensor cores):
 *   T[m][n] = sum_k A[m][k] * B[n][k]      A [M][K], B [N][K] in `dtype` (BF16 / TF32),
 *   T fp32 with row stride ldT elements (ldT >= N, ldT % 4 == 0), 16-byte aligned, else
 *   OLLIE_E_ALIGN.  K % 8 (bf16) or K % 4 (tf32) must be 0 (16-byte rows). */
ollie_status ollie_merged_gemm(int64_t M, int64_t N, int64_t K, ollie_dtype dtype,
                               const void *A, const void *B, float *T, int64_t ldT,
                               ollie_stream_t stream);

/* a3 / a4 standalone eOperator.  T is fp32 [n*h*w][ldT] (ldT >= r*s*f; pass r*s*f for a
 * dense T), columns in (i, j, f) order.  transposed == 0: OffsetAdd (Conv2d semantics);
 * transposed == 1: ConvTranspose selective addition (dilation 1).  y is [n][OH][OW][f]
 * in y_dtype (OLLIE_BF16 rounds fp32 sums RNE; OLLIE_FP32 / OLLIE_TF32 store fp32).
 * Spatial bounds are checked per dimension (reading Q5). */
ollie_status ollie_offset_add(const ollie_conv_shape *shape, int transposed, const float *T,
                              int64_t ldT, ollie_dtype y_dtype, void *y_nhwc, ollie_stream_t stream);

/* im2col ("tap folding") layout eOperator of the Conv2d `shape` describes (stride, dilation, pad;
 * the output grid OH x OW is the conv's): variable substitution of E1 that moves the taps
 * into the Matmul's reduction index, so operator matching sees a plain Matmul:
 *     out[b][oy][ox][k] = x[b][oy*stride - pad + i*dil][ox*stride - pad + j*dil][ch],
 *     k = (i*s + j)*c + ch < r*s*c;  0 outside the image and for r*s*c <= k < kp.
 * Used for layers with few input channels (FSRCNN's c = 1 feature extraction), which then run as a
 * 1x1 conv over kp-wide pixels.  x_nhwc [n][h][w][c], out [n][OH][OW][kp], device, `dtype` elements
 * (BF16, or TF32 / FP32 for 4-byte storage); kp >= r*s*c with kp*sizeof(elem) % 16 == 0 and out
 * 16-byte aligned, else OLLIE_E_INVALID / OLLIE_E_ALIGN.  Pure indexing: bit-exact. */
ollie_status ollie_tap_fold(const ollie_conv_shape *shape, ollie_dtype dtype, const void *x_nhwc, int64_t kp,
                            void *out, ollie_stream_t stream);

/* ---------------------------------------------------------------------------------
 * a5-a7 -- scoped index-expression eOperator (SPEC IndexExpr / TensorDecl / Scope /
 * Compute; general format L_x Sum_y f(T[tau(x,y)])).
 *
 * Iterators of a scope are numbered 0..n_trav-1 (traversal, in declared order = the
 * output layout) then n_trav..n_trav+n_sum-1 (summation, order-free,
 * P:855-857).  An index is  c0 + sum_t coef_t * atom_t  with atom = iterator,
 * floordiv(iterator, div) or mod(iterator, div) (div > 0; floor division and
 * non-negative remainder).  Reads inside a tensor's pad band return 0
 * (P:871-874); reads outside it are rejected statically (interval arithmetic over the
 * iterator ranges) with OLLIE_E_OOB, so an accepted eOp never reads out of bounds.
 * scope[0] is the evaluated (outer) scope; scope[1], if n_scopes == 2, is a nested
 * instantiated scope referenced as tensor -1 and evaluated inline (chain rule /
 * expression fusion): its element at coordinate v (v = its traversal
 * iterator values) is its body summed over its summation space, 0 in its pad band.
 * The output is dense, shape = scope[0]'s traversal range widths.
 * --------------------------------------------------------------------------------- */
#define OLLIE_MAX_DIMS 8
#define OLLIE_MAX_TERMS 8
#define OLLIE_MAX_ACCESS 8
#define OLLIE_MAX_INSTR 32
#define OLLIE_MAX_INPUTS 8

enum { OLLIE_ATOM_ITER = 0, OLLIE_ATOM_FLOORDIV = 1, OLLIE_ATOM_MOD = 2 };
enum { OLLIE_OP_PUSH_ACCESS = 0, OLLIE_OP_PUSH_CONST = 1, OLLIE_OP_ADD = 2, OLLIE_OP_MUL = 3,
       OLLIE_OP_SUB = 4, OLLIE_OP_NEG = 5, OLLIE_OP_MAX = 6, OLLIE_OP_MIN = 7 };

typedef struct { int32_t iter; int32_t kind; int64_t div; int64_t coef; } ollie_term;
typedef struct { int32_t nterms; ollie_term term[OLLIE_MAX_TERMS]; int64_t c0; } ollie_index;
typedef struct { int32_t tensor; /* >= 0 input id; -1 = scope[1] */
                 int32_t ndim; ollie_index idx[OLLIE_MAX_DIMS]; } ollie_access;
typedef struct { int32_t ndim; int64_t shape[OLLIE_MAX_DIMS];
                 int64_t pad_lo[OLLIE_MAX_DIMS], pad_hi[OLLIE_MAX_DIMS];
                 ollie_dtype dtype; } ollie_tensor;
typedef struct { int32_t op; int32_t arg; float cval; } ollie_instr; /* postfix body f */
typedef struct {
    int32_t n_trav; int64_t trav_lo[OLLIE_MAX_DIMS], trav_hi[OLLIE_MAX_DIMS];
    int32_t n_sum;  int64_t sum_lo[OLLIE_MAX_DIMS],  sum_hi[OLLIE_MAX_DIMS];
    int32_t n_acc;  ollie_access acc[OLLIE_MAX_ACCESS];
    int32_t n_ins;  ollie_instr body[OLLIE_MAX_INSTR];
    int64_t pad_lo[OLLIE_MAX_DIMS], pad_hi[OLLIE_MAX_DIMS]; /* zero band, scope[1] only */
} ollie_scope;
typedef struct {
    int32_t n_in; ollie_tensor in[OLLIE_MAX_INPUTS];
    ollie_dtype out_dtype;   /* OLLIE_BF16 or OLLIE_FP32; inputs likewise */
    int32_t n_scopes; ollie_scope scope[2];
} ollie_eop;

typedef struct {
    int32_t is_identity;    /* output == input[0] byte for byte            */
    int32_t pure_indexing;  /* single access, no summation, no arithmetic: bit-exact copy */
    int64_t out_elems;
    int64_t bytes_in, bytes_out; /* algorithmic bytes of one evaluation (0 if identity)  */
} ollie_eop_info;

/* Validate + classify; no launch. */
ollie_status ollie_eop_analyze(const ollie_eop *eop, ollie_eop_info *info);
/* Evaluate.  inputs[k] are device pointers to dense tensors of eop->in[k]; output is a
 * device pointer to the dense output.  An identity eOp whose output aliases input 0
 * launches nothing; a non-aliased identity is one device-to-device copy. */
ollie_status ollie_eop_eval(const ollie_eop *eop, const void *const *inputs, void *output,
                            ollie_stream_t stream);

/* ---------------------------------------------------------------------------------
 * NEXT-4 -- G2BMM, general-to-band matrix multiplication (iterator mapping table, P:1109-1118;
 * LongFormer dilated attention; band width / dilation reading R4 in DESIGN.md):
 *     out[b][m][w] = sum_k A[b][m][k] * B[b][m + d*(w - W)][k],   w in [0, 2W],
 * and 0 where the B row m + d*(w - W) lies outside [0, L).
 *   A, B : [batch][L][K] dtype elements, 16-byte aligned (device); K*sizeof(elem) == 128
 *          (K = 64 bf16 / 32 tf32), else E_UNSUPPORTED
 *   out  : [batch][L][ldo], ldo >= 2W+1, 16-byte aligned (else E_ALIGN); bf16 (BF16) or fp32
 *          (TF32); columns >= 2W+1 untouched.  batch, L, 2W+1 and the work items must fit int32.
 *   form : OLLIE_G2BMM_DERIVED -- the paper's dilated -> non-dilated rewrite: tiles of one
 *          residue class m = r + d*u, a dense band product per class (TMA element stride d);
 *          OLLIE_G2BMM_DIRECT -- dilated tiles over contiguous rows (band columns d apart), d <= 4.
 * fp32 accumulation; errors before any launch.
 * --------------------------------------------------------------------------------- */
enum { OLLIE_G2BMM_DERIVED = 0, OLLIE_G2BMM_DIRECT = 1 };
ollie_status ollie_g2bmm(int64_t batch, int64_t L, int64_t K, int64_t W, int64_t d, ollie_dtype dtype,
                         const void *A, const void *B, void *out, int64_t ldo, int form, ollie_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* OLLIE_H_ */
