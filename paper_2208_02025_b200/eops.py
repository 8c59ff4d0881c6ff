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
