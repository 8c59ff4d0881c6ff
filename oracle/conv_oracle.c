/*
 * conv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU oracle for the derived-convolution hot
 * path of Ollie (arXiv 2208.02025).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (libollie) never links, calls or imports it, and it shares no code,
 * headers or constants with the CUDA path.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n (the assembled copy,
 * P:670-1704); "S:n" = SPEC.md line n.  Every loop nest below is written in the
 * order of the definition it follows; no blocking, fusion or reordering.
 *
 * Layouts (the paper's HWC activations, "A[t1,t2,c]"):
 *   x      : NHWC  [n][h][w][c]
 *   y      : NHWC  [n][OH][OW][f]
 *   w_fcrs : PyTorch Conv2d weight          [f][c][r][s]
 *   w_cfrs : PyTorch ConvTranspose2d weight [c][f][r][s]
 *   wp     : merged weight, K-major          [(i*S+j)*F+f][c]   (transpose of Eq. layout-K)
 *   T      : merged-GEMM intermediate        [n*h*w][(i*S+j)*F+f]
 *
 * Readings of the paper used here: cross-correlation (Q3),
 * zero padding (Q20), PyTorch (i, pad, stride, dilation) offsets (Q2),
 * per-dimension bounds on the 5-D view of T (Q5), PyTorch ConvTranspose2d
 * semantics incl. output_padding (Q9).
 *
 * Pins: tests/test_oracle_conv.py (brute force im2col, torch fp64 library,
 * closed forms, the S:502 worked example, adjointness, derivation identity).
 */
#include <stdint.h>
#include <stddef.h>

typedef int64_t i64;

/* Output size of Conv2d, standard definition. */
i64 oracle_conv_out_size(i64 in, i64 k, i64 pad, i64 stride, i64 dil) {
    return (in + 2 * pad - dil * (k - 1) - 1) / stride + 1;
}

/* Output size of ConvTranspose2d (reading Q9). */
i64 oracle_convt_out_size(i64 in, i64 k, i64 pad, i64 stride, i64 dil, i64 opad) {
    return (in - 1) * stride - 2 * pad + dil * (k - 1) + opad + 1;
}

/*
 * O1 -- Conv2d by its definition (E1: L_{h,w,f} Sum_{c,r,s} A[h+r,w+s,c] K[r,s,f,c];
 * padding reads are 0):
 *   Y[b,oh,ow,f] = sum_c sum_i sum_j X[b, oh*st-p+i*d, ow*st-p+j*d, c] * W[f,c,i,j]
 */
void oracle_conv2d(i64 N, i64 C, i64 H, i64 W, i64 F, i64 R, i64 S,
                   i64 pad, i64 st, i64 dil,
                   const double *x, const double *w, double *y) {
    i64 OH = oracle_conv_out_size(H, R, pad, st, dil);
    i64 OW = oracle_conv_out_size(W, S, pad, st, dil);
    #pragma omp parallel for collapse(2) schedule(static)
    for (i64 b = 0; b < N; b++)
        for (i64 oh = 0; oh < OH; oh++)
            for (i64 ow = 0; ow < OW; ow++)
                for (i64 f = 0; f < F; f++) {
                    double acc = 0.0;
                    for (i64 c = 0; c < C; c++)
                        for (i64 i = 0; i < R; i++)
                            for (i64 j = 0; j < S; j++) {
                                i64 ih = oh * st - pad + i * dil;
                                i64 iw = ow * st - pad + j * dil;
                                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue; /* padding = 0 */
                                acc += x[((b * H + ih) * W + iw) * C + c] *
                                       w[((f * C + c) * R + i) * S + j];
                            }
                    y[((b * OH + oh) * OW + ow) * F + f] = acc;
                }
}

/*
 * O2 -- ConvTranspose2d in scatter form (the definition; reading Q9, PyTorch semantics):
 *   for every (b, ih, iw, c, i, j, f): oh = ih*st - p + i*d, ow = iw*st - p + j*d;
 *   if in range: Y[b,oh,ow,f] += X[b,ih,iw,c] * W[c,f,i,j]
 * Parallel over images only (scatter targets are private to an image).
 */
void oracle_convtranspose2d(i64 N, i64 C, i64 H, i64 W, i64 F, i64 R, i64 S,
                            i64 pad, i64 st, i64 dil, i64 opad,
                            const double *x, const double *w, double *y) {
    i64 OH = oracle_convt_out_size(H, R, pad, st, dil, opad);
    i64 OW = oracle_convt_out_size(W, S, pad, st, dil, opad);
    #pragma omp parallel for schedule(static)
    for (i64 b = 0; b < N; b++) {
        for (i64 k = 0; k < OH * OW * F; k++) y[b * OH * OW * F + k] = 0.0;
        for (i64 ih = 0; ih < H; ih++)
            for (i64 iw = 0; iw < W; iw++)
                for (i64 c = 0; c < C; c++)
                    for (i64 i = 0; i < R; i++)
                        for (i64 j = 0; j < S; j++)
                            for (i64 f = 0; f < F; f++) {
                                i64 oh = ih * st - pad + i * dil;
                                i64 ow = iw * st - pad + j * dil;
                                if (oh < 0 || oh >= OH || ow < 0 || ow >= OW) continue;
                                y[((b * OH + oh) * OW + ow) * F + f] +=
                                    x[((b * H + ih) * W + iw) * C + c] *
                                    w[((c * F + f) * R + i) * S + j];
                            }
    }
}

/*
 * O5 -- plain matmul, C[m,n] = sum_k A[m,k] * B[n,k]  (B stored K-major, i.e. the
 * Matmul of P:1342-1352 with K'^T as the second operand).
 */
void oracle_gemm_nt(i64 M, i64 Nn, i64 K, const double *A, const double *B, double *Cm) {
    #pragma omp parallel for schedule(static)
    for (i64 m = 0; m < M; m++)
        for (i64 n = 0; n < Nn; n++) {
            double acc = 0.0;
            for (i64 k = 0; k < K; k++) acc += A[m * K + k] * B[n * K + k];
            Cm[m * Nn + n] = acc;
        }
}

/*
 * a0 -- weight DLT (compile-time expression evaluation) written from
 * Eq. layout-K: K'[c, r*S*F + s*F + f] = K[r,s,f,c], stored transposed
 * (K-major) as wp[(i*S+j)*F+f][c].
 *   Conv2d   : K[r,s,f,c] = W[f,c,r,s]
 *   ConvT    : K[r,s,f,c] = W[c,f,r,s]
 */
void oracle_weight_dlt_conv2d(i64 F, i64 C, i64 R, i64 S, const double *w_fcrs, double *wp) {
    for (i64 i = 0; i < R; i++)
        for (i64 j = 0; j < S; j++)
            for (i64 f = 0; f < F; f++)
                for (i64 c = 0; c < C; c++)
                    wp[((i * S + j) * F + f) * C + c] = w_fcrs[((f * C + c) * R + i) * S + j];
}

void oracle_weight_dlt_convt(i64 C, i64 F, i64 R, i64 S, const double *w_cfrs, double *wp) {
    for (i64 i = 0; i < R; i++)
        for (i64 j = 0; j < S; j++)
            for (i64 f = 0; f < F; f++)
                for (i64 c = 0; c < C; c++)
                    wp[((i * S + j) * F + f) * C + c] = w_cfrs[((c * F + f) * R + i) * S + j];
}

/*
 * O3 step a3 -- OffsetAdd (E7):
 *   Y[b,oh,ow,f] = sum_{i<R} sum_{j<S} T[b, oh*st-p+i*d, ow*st-p+j*d, (i*S+j)*F+f]
 * Terms whose spatial index leaves [0,H)x[0,W) are zero; the test is made per
 * spatial dimension on the 5-D view of T (reading Q5), never on the flattened m.
 */
void oracle_offset_add(i64 N, i64 H, i64 W, i64 F, i64 R, i64 S,
                       i64 pad, i64 st, i64 dil, const double *T, double *y) {
    i64 OH = oracle_conv_out_size(H, R, pad, st, dil);
    i64 OW = oracle_conv_out_size(W, S, pad, st, dil);
    i64 NT = R * S * F;
    #pragma omp parallel for collapse(2) schedule(static)
    for (i64 b = 0; b < N; b++)
        for (i64 oh = 0; oh < OH; oh++)
            for (i64 ow = 0; ow < OW; ow++)
                for (i64 f = 0; f < F; f++) {
                    double acc = 0.0;
                    for (i64 i = 0; i < R; i++)
                        for (i64 j = 0; j < S; j++) {
                            i64 t1 = oh * st - pad + i * dil;
                            i64 t2 = ow * st - pad + j * dil;
                            if (t1 < 0 || t1 >= H || t2 < 0 || t2 >= W) continue;
                            acc += T[((b * H + t1) * W + t2) * NT + (i * S + j) * F + f];
                        }
                    y[((b * OH + oh) * OW + ow) * F + f] = acc;
                }
}

/*
 * O3 step a4 -- ConvTranspose selective addition:
 *   Y[b,oh,ow,f] = sum over (i,j) with st | (oh+p-i*d) and st | (ow+p-j*d) of
 *                  T[b, (oh+p-i*d)/st, (ow+p-j*d)/st, (i*S+j)*F+f],
 * counting only input indices inside [0,H)x[0,W).
 */
void oracle_selective_add(i64 N, i64 H, i64 W, i64 F, i64 R, i64 S,
                          i64 pad, i64 st, i64 dil, i64 opad, const double *T, double *y) {
    i64 OH = oracle_convt_out_size(H, R, pad, st, dil, opad);
    i64 OW = oracle_convt_out_size(W, S, pad, st, dil, opad);
    i64 NT = R * S * F;
    #pragma omp parallel for collapse(2) schedule(static)
    for (i64 b = 0; b < N; b++)
        for (i64 oh = 0; oh < OH; oh++)
            for (i64 ow = 0; ow < OW; ow++)
                for (i64 f = 0; f < F; f++) {
                    double acc = 0.0;
                    for (i64 i = 0; i < R; i++)
                        for (i64 j = 0; j < S; j++) {
                            i64 a = oh + pad - i * dil;
                            i64 c = ow + pad - j * dil;
                            if (a < 0 || c < 0) continue;          /* negative: no input index */
                            if (a % st != 0 || c % st != 0) continue; /* not selected */
                            i64 ih = a / st, iw = c / st;
                            if (ih >= H || iw >= W) continue;
                            acc += T[((b * H + ih) * W + iw) * NT + (i * S + j) * F + f];
                        }
                    y[((b * OH + oh) * OW + ow) * F + f] = acc;
                }
}

/* NEXT-4 G2BMM, general-to-band matrix multiplication (iterator mapping table, P:1109-1118;
 * LongFormer dilated attention), the definition written out (reading R4):
 *   out[b][m][w] = sum_k A[b][m][k] * B[b][m + d*(w - W)][k],  w in [0, 2W],
 * and 0 when the B row m + d*(w - W) lies outside [0, L).  A, B: [batch][L][K]; out: [batch][L][2W+1]. */
void oracle_g2bmm(i64 batch, i64 L, i64 K, i64 W, i64 d, const double *A, const double *B, double *out) {
    const i64 NW = 2 * W + 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (i64 b = 0; b < batch; b++)
        for (i64 m = 0; m < L; m++)
            for (i64 w = 0; w < NW; w++) {
                const i64 j = m + d * (w - W);
                double acc = 0.0;
                if (j >= 0 && j < L)
                    for (i64 k = 0; k < K; k++) acc += A[(b * L + m) * K + k] * B[(b * L + j) * K + k];
                out[(b * L + m) * NW + w] = acc;
            }
}

/* Number of OpenMP threads the oracle will use (reported as cpu_baseline.cores). */
#ifdef _OPENMP
#include <omp.h>
int oracle_num_threads(void) { return omp_get_max_threads(); }
/* Thread count for later calls (bench.py's single-thread cpu_baseline figure); arithmetic unchanged. */
void oracle_set_num_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
#else
int oracle_num_threads(void) { return 1; }
void oracle_set_num_threads(int n) { (void)n; }
#endif
