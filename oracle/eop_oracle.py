"""Literal eOperator interpreter -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Evaluates a scoped tensor-algebra expression in the paper's general 1-scope format


    L_{x in X} Sum_{y in Y} f( T[ tau(x, y) ] )

with SPEC's lowering semantics: one loop per traversal iterator in the
declared order (the order IS the output layout), inner loops over the
summation iterators, zero-valued reads in the declared pad band
and a hard error for reads outside it (OutOfBoundsRead).  Index functions are
affine combinations of iterators plus floordiv / mod atoms.
A second scope (scopes[1]) is a nested instantiated scope read by the outer body
(expression fusion / chain rule); it is evaluated either inline per read
or memoised once -- both must agree.

Pure Python, fp64, for small cases only.

The expression is a plain-data dict (schema in DESIGN.md "eOperator spec"):

    {"inputs": [{"shape": [...], "pad": [[lo, hi], ...]}, ...],
     "scopes": [{"trav": [[lo, hi], ...], "sum": [[lo, hi], ...],
                 "access": [{"tensor": k, "index": [IDX, ...]}, ...],
                 "body": [["acc", a] | ["const", v] | ["add"] | ["mul"] | ["sub"]
                          | ["neg"] | ["max"] | ["min"], ...],      # postfix
                 "pad": [[lo, hi], ...]},                            # scopes[1] only
                ...]}
    IDX = {"terms": [[coef, iter, kind, div], ...], "const": c0}
          kind in {"id", "div", "mod"}; iter numbers the scope's traversal iterators
          first (0..nt-1) then its summation iterators (nt..nt+ns-1).
    tensor k >= 0 is inputs[k]; k == -1 is scopes[1].
"""
from __future__ import annotations

import itertools

import numpy as np


class OutOfBoundsRead(Exception):
    """a read outside the declared pad band."""


class InvalidExpression(Exception):
    """UndeclaredIterator / ArityMismatch / EmptyRange / ShapeMismatch."""


def _eval_index(idx, it_vals):
    """tau: sum of coef * atom + const; atoms: iterator, floordiv(iterator, d), mod(iterator, d)."""
    v = idx.get("const", 0)
    for coef, it, kind, div in idx["terms"]:
        if it < 0 or it >= len(it_vals):
            raise InvalidExpression("UndeclaredIterator")
        a = it_vals[it]
        if kind == "id":
            pass
        elif kind == "div":
            if div <= 0:
                raise InvalidExpression("non-positive divisor")
            a = a // div          # floor division
        elif kind == "mod":
            if div <= 0:
                raise InvalidExpression("non-positive divisor")
            a = a % div           # non-negative remainder
        else:
            raise InvalidExpression(f"unknown atom kind {kind}")
        v += coef * a
    return v


def _check_scope(sc):
    for lo, hi in list(sc["trav"]) + list(sc.get("sum", [])):
        if not lo < hi:
            raise InvalidExpression("EmptyRange")


class _Evaluator:
    def __init__(self, expr, inputs, memoize):
        self.expr = expr
        self.inputs = [np.asarray(t, dtype=np.float64) for t in inputs]
        ins = expr["inputs"]
        if len(ins) != len(self.inputs):
            raise InvalidExpression("ShapeMismatch: number of inputs")
        for decl, arr in zip(ins, self.inputs):
            if tuple(decl["shape"]) != tuple(arr.shape):
                raise InvalidExpression(f"ShapeMismatch {decl['shape']} vs {arr.shape}")
        for sc in expr["scopes"]:
            _check_scope(sc)
        self.memo = None
        if memoize and len(expr["scopes"]) > 1:
            inner = expr["scopes"][1]
            shape = [hi - lo for lo, hi in inner["trav"]]
            self.memo = np.zeros(shape, np.float64)
            for x in itertools.product(*[range(lo, hi) for lo, hi in inner["trav"]]):
                pos = tuple(v - lo for v, (lo, _) in zip(x, inner["trav"]))
                self.memo[pos] = self._scope_value(1, x)

    def _read(self, tensor, coords):
        if tensor >= 0:
            decl = self.expr["inputs"][tensor]
            shape = decl["shape"]
            pad = decl.get("pad") or [[0, 0]] * len(shape)
            if len(coords) != len(shape):
                raise InvalidExpression("ArityMismatch")
            inside = True
            for v, d, (plo, phi) in zip(coords, shape, pad):
                if v < -plo or v >= d + phi:
                    raise OutOfBoundsRead(f"input {tensor} at {coords}")
                if v < 0 or v >= d:
                    inside = False
            return float(self.inputs[tensor][tuple(coords)]) if inside else 0.0
        if tensor != -1 or len(self.expr["scopes"]) < 2:
            raise InvalidExpression("unknown tensor reference")
        inner = self.expr["scopes"][1]
        trav = inner["trav"]
        pad = inner.get("pad") or [[0, 0]] * len(trav)
        if len(coords) != len(trav):
            raise InvalidExpression("ArityMismatch")
        inside = True
        for v, (lo, hi), (plo, phi) in zip(coords, trav, pad):
            if v < lo - plo or v >= hi + phi:
                raise OutOfBoundsRead(f"scope 1 at {coords}")
            if v < lo or v >= hi:
                inside = False
        if not inside:
            return 0.0
        if self.memo is not None:
            return float(self.memo[tuple(v - lo for v, (lo, _) in zip(coords, trav))])
        return self._scope_value(1, tuple(coords))

    def _body(self, sc, it_vals):
        stack = []
        for ins in sc["body"]:
            op = ins[0]
            if op == "acc":
                acc = sc["access"][ins[1]]
                coords = [_eval_index(ix, it_vals) for ix in acc["index"]]
                stack.append(self._read(acc["tensor"], coords))
            elif op == "const":
                stack.append(float(ins[1]))
            elif op == "neg":
                stack.append(-stack.pop())
            elif op in ("add", "mul", "sub", "max", "min"):
                b = stack.pop()
                a = stack.pop()
                stack.append({"add": a + b, "mul": a * b, "sub": a - b,
                              "max": max(a, b), "min": min(a, b)}[op])
            else:
                raise InvalidExpression(f"unknown op {op}")
        if len(stack) != 1:
            raise InvalidExpression("malformed body")
        return stack[0]

    def _scope_value(self, k, x):
        """Value of scope k at traversal point x: Sum_y f(T[tau(x, y)])."""
        sc = self.expr["scopes"][k]
        sums = sc.get("sum", [])
        if not sums:
            return self._body(sc, tuple(x))
        total = 0.0
        for y in itertools.product(*[range(lo, hi) for lo, hi in sums]):
            total += self._body(sc, tuple(x) + tuple(y))
        return total


def eop_eval(expr, inputs, memoize: bool = False) -> np.ndarray:
    """Evaluate scopes[0]; output shape = its traversal range widths, in traversal order."""
    ev = _Evaluator(expr, inputs, memoize)
    outer = expr["scopes"][0]
    shape = [hi - lo for lo, hi in outer["trav"]]
    out = np.zeros(shape, np.float64)
    for x in itertools.product(*[range(lo, hi) for lo, hi in outer["trav"]]):
        pos = tuple(v - lo for v, (lo, _) in zip(x, outer["trav"]))
        out[pos] = ev._scope_value(0, x)
    return out


def eop_bounds_ok(expr) -> bool:
    """Brute force: does every access of every scope stay inside its pad band?"""
    for k, sc in enumerate(expr["scopes"]):
        rngs = [range(lo, hi) for lo, hi in list(sc["trav"]) + list(sc.get("sum", []))]
        for it_vals in itertools.product(*rngs):
            for acc in sc["access"]:
                coords = [_eval_index(ix, it_vals) for ix in acc["index"]]
                t = acc["tensor"]
                if t >= 0:
                    decl = expr["inputs"][t]
                    shape = decl["shape"]
                    pad = decl.get("pad") or [[0, 0]] * len(shape)
                    lims = [(-plo, d + phi) for d, (plo, phi) in zip(shape, pad)]
                else:
                    inner = expr["scopes"][1]
                    pad = inner.get("pad") or [[0, 0]] * len(inner["trav"])
                    lims = [(lo - plo, hi + phi) for (lo, hi), (plo, phi) in zip(inner["trav"], pad)]
                if len(coords) != len(lims):
                    return False
                for v, (a, b) in zip(coords, lims):
                    if v < a or v >= b:
                        return False
    return True


def eop_is_identity(expr) -> bool:
    """Identity eOperator test of P:1440-1443, literally: squash input and output to 1-D
    and check, element by element, that output element o reads input element o."""
    if len(expr["scopes"]) != 1 or len(expr["inputs"]) != 1:
        return False
    sc = expr["scopes"][0]
    if sc.get("sum") or sc["body"] != [["acc", 0]] or len(sc["access"]) != 1:
        return False
    acc = sc["access"][0]
    if acc["tensor"] != 0:
        return False
    shape_in = list(expr["inputs"][0]["shape"])
    shape_out = [hi - lo for lo, hi in sc["trav"]]
    if int(np.prod(shape_in)) != int(np.prod(shape_out)):
        return False
    strides = [int(np.prod(shape_in[d + 1:])) for d in range(len(shape_in))]
    for o, x in enumerate(itertools.product(*[range(lo, hi) for lo, hi in sc["trav"]])):
        coords = [_eval_index(ix, x) for ix in acc["index"]]
        if len(coords) != len(shape_in):
            return False
        for v, d in zip(coords, shape_in):
            if v < 0 or v >= d:
                return False
        if sum(v * st for v, st in zip(coords, strides)) != o:
            return False
    return True
