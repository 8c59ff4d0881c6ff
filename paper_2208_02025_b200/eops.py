"""Product-side builders of the layout eOperators the hot path needs, as plain-data specs
(schema: DESIGN.md "eOperator spec"; turned into the C struct by ollie.make_eop).

 - channel_pad: the pad layout eOperator that widens NHWC rows to a 16-byte multiple
   for TMA, zero-filled from the tensor's pad band.
 - nchw_to_nhwc: the DLT eOperator of Fig. post-opt for NCHW callers.
 - layout_a: Eq. layout-A, the identity on NHWC memory (eliminated,
   P:1440-1443).
"""
from __future__ import annotations


def _it(i, coef=1):
    return [coef, i, "id", 1]


def _ix(*terms, const=0):
    return {"terms": [list(t) for t in terms], "const": const}


def channel_pad(n: int, h: int, w: int, c: int, cp: int) -> dict:
    """out[b, y, x, k] = in[b, y, x, k] for k < c, 0 for c <= k < cp."""
    assert cp >= c
    return {"inputs": [{"shape": [n, h, w, c], "pad": [[0, 0], [0, 0], [0, 0], [0, cp - c]]}],
            "scopes": [{"trav": [[0, n], [0, h], [0, w], [0, cp]], "sum": [],
                        "access": [{"tensor": 0, "index": [_ix(_it(0)), _ix(_it(1)), _ix(_it(2)), _ix(_it(3))]}],
                        "body": [["acc", 0]]}]}


def nchw_to_nhwc(n: int, c: int, h: int, w: int) -> dict:
    """out[b, y, x, k] = in[b, k, y, x]."""
    return {"inputs": [{"shape": [n, c, h, w]}],
            "scopes": [{"trav": [[0, n], [0, h], [0, w], [0, c]], "sum": [],
                        "access": [{"tensor": 0, "index": [_ix(_it(0)), _ix(_it(3)), _ix(_it(1)), _ix(_it(2))]}],
                        "body": [["acc", 0]]}]}


def layout_a(h: int, w: int, c: int) -> dict:
    """A'[t1*W + t2, c] = A[t1, t2, c]."""
    return {"inputs": [{"shape": [h, w, c]}],
            "scopes": [{"trav": [[0, h * w], [0, c]], "sum": [],
                        "access": [{"tensor": 0, "index": [_ix([1, 0, "div", w]), _ix([1, 0, "mod", w]),
                                                           _ix(_it(1))]}],
                        "body": [["acc", 0]]}]}


# --------------------------------------------------------------------------- NEXT-1
# Dilated -> non-dilated derivation: with pad = dil * k, output row d*u + a of a dilation-d conv
# reads input rows d*(u + i - k) + a only, i.e. residue class a of the input, densely.  So the
# dilated conv is  batch_to_space o dense_conv(pad k) o space_to_batch  with the d*d residue
# classes of rows and cols stacked on the batch dimension (expression splitting by residue,
# P:927-934, plus two layout DLT eOperators).
def space_to_batch(n: int, h: int, w: int, c: int, d: int) -> dict:
    """out[(a*d + b)*n + img, u, v, k] = in[img, d*u + a, d*v + b, k]   (zero past h / w).

    Traversal [a, b, img, u, v, k] (the same memory as [d*d*n, hs, ws, c]): every index is
    affine.  Rows / cols past the image read the zero pad band."""
    hs, ws = -(-h // d), -(-w // d)
    return {"inputs": [{"shape": [n, h, w, c], "pad": [[0, 0], [0, hs * d - h], [0, ws * d - w], [0, 0]]}],
            "scopes": [{"trav": [[0, d], [0, d], [0, n], [0, hs], [0, ws], [0, c]], "sum": [],
                        "access": [{"tensor": 0, "index": [_ix(_it(2)), _ix(_it(3, d), _it(0)), _ix(_it(4, d), _it(1)),
                                                           _ix(_it(5))]}],
                        "body": [["acc", 0]]}]}


def batch_to_space(n: int, hs: int, ws: int, f: int, d: int, oh: int, ow: int) -> dict:
    """out[img, y, x, k] = in[((y mod d)*d + (x mod d))*n + img, y div d, x div d, k].

    When oh == d*hs and ow == d*ws the traversal [img, u, a, v, b, k] (memory of [n, oh, ow, f])
    keeps every index affine; otherwise the floordiv / mod form crops to [n, oh, ow, f]."""
    if oh == d * hs and ow == d * ws:
        return {"inputs": [{"shape": [d * d * n, hs, ws, f]}],
                "scopes": [{"trav": [[0, n], [0, hs], [0, d], [0, ws], [0, d], [0, f]], "sum": [],
                            "access": [{"tensor": 0, "index": [_ix(_it(2, d * n), _it(4, n), _it(0)), _ix(_it(1)),
                                                               _ix(_it(3)), _ix(_it(5))]}],
                            "body": [["acc", 0]]}]}
    return {"inputs": [{"shape": [d * d * n, hs, ws, f]}],
            "scopes": [{"trav": [[0, n], [0, oh], [0, ow], [0, f]], "sum": [],
                        "access": [{"tensor": 0, "index": [_ix([d * n, 1, "mod", d], [n, 2, "mod", d], _it(0)),
                                                           _ix([1, 1, "div", d]), _ix([1, 2, "div", d]), _ix(_it(3))]}],
                        "body": [["acc", 0]]}]}
