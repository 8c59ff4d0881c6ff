"""Hand-written eOperator expressions (plain-data spec, schema in DESIGN.md) used by the
oracle pins and the GPU parity tests.  Test-side only: they are written from the
paper's formulas independently of the product's own builders
(paper_2208_02025_b200/eops.py), so each side checks the other.
"""


def I(it, coef=1):
    return [coef, it, "id", 1]


def D(it, d, coef=1):
    return [coef, it, "div", d]


def M(it, d, coef=1):
    return [coef, it, "mod", d]


def idx(*terms, const=0):
    return {"terms": [list(t) for t in terms], "const": const}


def copy_body():
    return [["acc", 0]]


def transpose_nchw_to_nhwc(n, c, h, w):
    """DLT: out[n,h,w,c] = in[n,c,h,w]."""
    return {"inputs": [{"shape": [n, c, h, w]}],
            "scopes": [{"trav": [[0, n], [0, h], [0, w], [0, c]], "sum": [],
                        "access": [{"tensor": 0, "index": [idx(I(0)), idx(I(3)), idx(I(1)), idx(I(2))]}],
                        "body": copy_body()}]}


def layout_a(h, w, c):
    """Eq. layout-A: A'[t1*W+t2, c] = A[t1, t2, c] -> identity on HWC memory."""
    return {"inputs": [{"shape": [h, w, c]}],
            "scopes": [{"trav": [[0, h * w], [0, c]], "sum": [],
                        "access": [{"tensor": 0, "index": [idx(D(0, w)), idx(M(0, w)), idx(I(1))]}],
                        "body": copy_body()}]}


def channel_pad(n, h, w, c, cp):
    """Channel-pad layout eOperator (H3): out[n,h,w,k] = in[n,h,w,k], zero for k >= c."""
    return {"inputs": [{"shape": [n, h, w, c], "pad": [[0, 0], [0, 0], [0, 0], [0, cp - c]]}],
            "scopes": [{"trav": [[0, n], [0, h], [0, w], [0, cp]], "sum": [],
                        "access": [{"tensor": 0, "index": [idx(I(0)), idx(I(1)), idx(I(2)), idx(I(3))]}],
                        "body": copy_body()}]}


def offset_add(n, h, w, f, r, s, pad, stride=1, dil=1):
    """E7 over T viewed as [n, h, w, r*s*f]:
    L_{b,oh,ow,f} Sum_{i,j} T[b, oh*st-p+i*d, ow*st-p+j*d, (i*S+j)*F+f], zero pad band on h, w."""
    oh = (h + 2 * pad - dil * (r - 1) - 1) // stride + 1
    ow = (w + 2 * pad - dil * (s - 1) - 1) // stride + 1
    hi_h = max(0, (oh - 1) * stride - pad + (r - 1) * dil - (h - 1))
    hi_w = max(0, (ow - 1) * stride - pad + (s - 1) * dil - (w - 1))
    return {"inputs": [{"shape": [n, h, w, r * s * f], "pad": [[0, 0], [pad, hi_h], [pad, hi_w], [0, 0]]}],
            "scopes": [{"trav": [[0, n], [0, oh], [0, ow], [0, f]], "sum": [[0, r], [0, s]],
                        # iterators: 0 b, 1 oh, 2 ow, 3 f, 4 i, 5 j
                        "access": [{"tensor": 0, "index": [
                            idx(I(0)),
                            idx(I(1, stride), I(4, dil), const=-pad),
                            idx(I(2, stride), I(5, dil), const=-pad),
                            idx(I(4, s * f), I(5, f), I(3))]}],
                        "body": copy_body()}]}


def selective_add(n, h, w, f, r, s, pad, stride, opad=0):
    """Strided ConvT selective addition, dilation 1, as one eOperator over
    T viewed as [n, h, w, r, s, f].  The traversal runs over t = o + pad, so the selected
    kernel rows are i = stride*k + t % stride reading input row t // stride - k; kernel
    rows beyond r fall in the zero pad band of the r / s dims."""
    oh = (h - 1) * stride - 2 * pad + (r - 1) + opad + 1
    ow = (w - 1) * stride - 2 * pad + (s - 1) + opad + 1
    kr = -(-r // stride)
    ks = -(-s // stride)
    # index ranges: t//st - k in [ -kr+1 + pad//st, (oh-1+pad)//st ]
    lo_h = max(0, kr - 1 - pad // stride)
    lo_w = max(0, ks - 1 - pad // stride)
    hi_h = max(0, (oh - 1 + pad) // stride - (h - 1))
    hi_w = max(0, (ow - 1 + pad) // stride - (w - 1))
    return {"inputs": [{"shape": [n, h, w, r, s, f],
                        "pad": [[0, 0], [lo_h, hi_h], [lo_w, hi_w], [0, kr * stride - r],
                                [0, ks * stride - s], [0, 0]]}],
            "scopes": [{"trav": [[0, n], [pad, oh + pad], [pad, ow + pad], [0, f]],
                        "sum": [[0, kr], [0, ks]],
                        # iterators: 0 b, 1 th, 2 tw, 3 f, 4 kh, 5 kw
                        "access": [{"tensor": 0, "index": [
                            idx(I(0)),
                            idx(D(1, stride), I(4, -1)),
                            idx(D(2, stride), I(5, -1)),
                            idx(I(4, stride), M(1, stride)),
                            idx(I(5, stride), M(2, stride)),
                            idx(I(3))]}],
                        "body": copy_body()}]}


def fused_pad_then_offset_add(n, h, w, f, r, s, pad, extra):
    """Fused eOperator pair: the inner scope widens T's last dim
    with `extra` zero channels per pixel (a layout eOp); the outer OffsetAdd reads it."""
    nt = r * s * f
    inner = {"trav": [[0, n], [0, h], [0, w], [0, nt + extra]], "sum": [],
             "access": [{"tensor": 0, "index": [idx(I(0)), idx(I(1)), idx(I(2)), idx(I(3))]}],
             "body": [["acc", 0], ["const", 2.0], ["mul"]],
             "pad": [[0, 0], [pad, pad], [pad, pad], [0, 0]]}
    outer = offset_add(n, h, w, f, r, s, pad)["scopes"][0]
    outer = dict(outer)
    outer["access"] = [dict(outer["access"][0], tensor=-1)]
    return {"inputs": [{"shape": [n, h, w, nt], "pad": [[0, 0], [0, 0], [0, 0], [0, extra]]}],
            "scopes": [outer, inner]}


def affine_mix(n, c, h, w):
    """A non-identity affine eOp with summation and arithmetic in the body:
    out[b, y, x] = Sum_k ((2*in0[b, k, y, x] - in1[y, x]) * 0.5 + max(in1[y,x], 0))"""
    return {"inputs": [{"shape": [n, c, h, w]}, {"shape": [h, w]}],
            "scopes": [{"trav": [[0, n], [0, h], [0, w]], "sum": [[0, c]],
                        "access": [{"tensor": 0, "index": [idx(I(0)), idx(I(3)), idx(I(1)), idx(I(2))]},
                                   {"tensor": 1, "index": [idx(I(1)), idx(I(2))]}],
                        "body": [["const", 2.0], ["acc", 0], ["mul"], ["acc", 1], ["sub"],
                                 ["const", 0.5], ["mul"], ["acc", 1], ["const", 0.0], ["max"], ["add"]]}]}
