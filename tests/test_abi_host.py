"""CPU-only checks of the boundary (no GPU compute): libollie.so loads, exports every
function include/ollie.h declares, and its host logic (shape validation, workspace
sizing, eOperator validation / interval bounds / identity detection) agrees with the
oracle's independent definitions."""
import ctypes
import os
import re
import subprocess

import pytest

import oracle
from tests import eop_cases as ec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ollie.h")


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import build
    build.build()
    from paper_2208_02025_b200 import ollie
    return ollie


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ollie_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(O):
    names = _declared()
    assert len(names) >= 14
    lib = ctypes.CDLL(O.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", O.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), f"{n} not a defined text symbol"
    assert set(names) == set(O.EXPORTED)


def test_abi_version_and_strings(O):
    assert O.abi_version() == 1
    assert O.status_string(O.E_OOB) == "OLLIE_E_OOB"
    assert O.status_string(O.OK) == "OLLIE_OK"


@pytest.mark.parametrize("h,r,pad,st,dil,tr,op", [(56, 3, 1, 1, 1, False, 0), (64, 3, 2, 1, 2, False, 0),
                                                  (56, 3, 1, 2, 1, False, 0), (2, 4, 1, 2, 1, True, 0),
                                                  (256, 9, 4, 2, 1, True, 1), (7, 1, 0, 1, 1, False, 0)])
def test_output_size_matches_oracle(O, h, r, pad, st, dil, tr, op):
    shp = O.conv_shape(2, 16, h, h + 1, 8, r, r, pad, st, dil, op)
    oh, ow = O.output_hw(shp, tr)
    if tr:
        assert (oh, ow) == (oracle.convt_out_size(h, r, pad, st, dil, op), oracle.convt_out_size(h + 1, r, pad, st, dil, op))
    else:
        assert (oh, ow) == (oracle.conv_out_size(h, r, pad, st, dil), oracle.conv_out_size(h + 1, r, pad, st, dil))


def test_invalid_shapes(O):
    for bad in (O.conv_shape(0, 16, 8, 8, 8, 3, 3, 1), O.conv_shape(1, 16, 8, 8, 8, 3, 3, -1),
                O.conv_shape(1, 16, 2, 2, 8, 5, 5, 0), O.conv_shape(1, 16, 8, 8, 8, 3, 3, 1, 0)):
        with pytest.raises(O.OllieError) as ei:
            O.output_hw(bad, False)
        assert ei.value.status == O.E_INVALID
    with pytest.raises(O.OllieError):
        O.output_hw(O.conv_shape(1, 16, 4, 4, 8, 4, 4, 1, 2, 1, 2), True)   # output_padding >= stride


def test_workspace_sizes(O):
    shp = O.conv_shape(16, 64, 56, 56, 64, 3, 3, 1)
    assert O.workspace_bytes(shp, O.BF16, O.PLAN_UNFUSED) == 16 * 56 * 56 * 576 * 4
    one = O.conv_shape(4, 56, 9, 9, 12, 1, 1, 0)
    assert O.workspace_bytes(one, O.BF16, O.PLAN_UNFUSED) == 0           # identity OffsetAdd eliminated
    odd = O.conv_shape(1, 56, 5, 5, 1, 9, 9, 4, 2, 1, 1)
    assert O.workspace_bytes(odd, O.BF16, O.PLAN_UNFUSED, True) == 25 * 84 * 4   # ldT = 81 -> 84
    assert O.prepared_weight_bytes(shp, O.BF16) == 576 * 64 * 2


def _spec_cases():
    return {
        "transpose": ec.transpose_nchw_to_nhwc(2, 3, 4, 5),
        "layout_a": ec.layout_a(3, 4, 5),
        "layout_a_deg": ec.transpose_nchw_to_nhwc(1, 1, 4, 5),
        "channel_pad": ec.channel_pad(1, 2, 2, 3, 4),
        "offset_add": ec.offset_add(2, 4, 5, 2, 3, 3, 1),
        "offset_add_s2d2": ec.offset_add(1, 9, 8, 3, 3, 3, 2, 2, 2),
        "selective_add": ec.selective_add(2, 2, 3, 2, 4, 4, 1, 2),
        "selective_add_9": ec.selective_add(1, 3, 3, 1, 9, 9, 4, 2, 1),
        "fused_pair": ec.fused_pad_then_offset_add(1, 4, 5, 2, 3, 3, 1, 3),
        "affine_mix": ec.affine_mix(2, 3, 2, 4),
    }


@pytest.mark.parametrize("name", sorted(_spec_cases()))
def test_eop_analysis_agrees_with_oracle(O, name):
    spec = _spec_cases()[name]
    e = O.make_eop(spec, [O.FP32] * len(spec["inputs"]), O.FP32)
    assert oracle.eop_bounds_ok(spec)
    info = O.eop_analyze(e)
    assert info["is_identity"] == oracle.eop_is_identity(spec)
    assert info["pure_indexing"] == (len(spec["scopes"]) == 1 and not spec["scopes"][0]["sum"]
                                     and spec["scopes"][0]["body"] == [["acc", 0]])


def test_eop_identity_reshape_variants(O):
    # [2,3,4] viewed as [6,4] (m = a*3 + b): identity; swapped div/mod: not identity
    ok = {"inputs": [{"shape": [2, 3, 4]}],
          "scopes": [{"trav": [[0, 6], [0, 4]], "sum": [],
                      "access": [{"tensor": 0, "index": [ec.idx(ec.D(0, 3)), ec.idx(ec.M(0, 3)), ec.idx(ec.I(1))]}],
                      "body": [["acc", 0]]}]}
    bad = {"inputs": [{"shape": [3, 2, 4]}],
           "scopes": [{"trav": [[0, 6], [0, 4]], "sum": [],
                       "access": [{"tensor": 0, "index": [ec.idx(ec.M(0, 3)), ec.idx(ec.D(0, 3)), ec.idx(ec.I(1))]}],
                       "body": [["acc", 0]]}]}
    for spec, want in ((ok, True), (bad, False)):
        assert oracle.eop_is_identity(spec) is want
        assert O.eop_analyze(O.make_eop(spec, [O.FP32], O.FP32))["is_identity"] is want
    # identity needs matching dtypes: bf16 -> fp32 is a conversion, not an identity
    assert not O.eop_analyze(O.make_eop(ok, [O.BF16], O.FP32))["is_identity"]


def test_eop_errors(O):
    oob = ec.offset_add(1, 4, 4, 1, 3, 3, 1)
    oob["inputs"][0]["pad"] = [[0, 0]] * 4
    assert not oracle.eop_bounds_ok(oob)
    with pytest.raises(O.OllieError) as ei:
        O.eop_analyze(O.make_eop(oob))
    assert ei.value.status == O.E_OOB
    empty = ec.layout_a(2, 2, 2)
    empty["scopes"][0]["trav"][1] = [3, 3]
    undeclared = ec.layout_a(2, 2, 2)
    undeclared["scopes"][0]["access"][0]["index"][2] = ec.idx(ec.I(5))
    arity = ec.layout_a(2, 2, 2)
    arity["scopes"][0]["access"][0]["index"].pop()
    underflow = ec.layout_a(2, 2, 2)
    underflow["scopes"][0]["body"] = [["acc", 0], ["add"]]
    for spec in (empty, undeclared, arity, underflow):
        with pytest.raises(O.OllieError) as ei:
            O.eop_analyze(O.make_eop(spec))
        assert ei.value.status == O.E_INVALID
