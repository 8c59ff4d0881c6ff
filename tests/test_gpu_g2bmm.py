"""GPU parity of NEXT-4 G2BMM (both forms) against the fp64 oracle: integer mode bit-exact (bf16 RNE
of exact fp32 sums), random within the bf16 / TF32 bars; ragged L (not a multiple of the tile,
shorter than a tile), W = 0, every d up to 4, a padded output pitch, and the LongFormer config at
full size compared on every row."""
import numpy as np
import pytest
import torch

import oracle
import ollie_synth as syn
from tests.test_gpu_parity import TOL, _max_rel, _round_like

pytestmark = pytest.mark.gpu

CASES = [
    syn.G2("tiny", 1, 37, 64, 3, 1),
    syn.G2("d2", 2, 300, 64, 16, 2),
    syn.G2("d3_ragged", 1, 517, 64, 33, 3),
    syn.G2("d4_w256", 1, 1300, 64, 256, 4),
    syn.G2("w0", 2, 200, 64, 0, 2),
    syn.G2("short_L", 3, 20, 64, 40, 4),
    syn.G2("tf32", 1, 400, 32, 20, 2, dtype="tf32"),
]


@pytest.fixture(scope="module")
def O():
    from paper_2208_02025_b200 import ollie
    return ollie


def _run(O, g, a, b, form, ldo=None):
    nw = 2 * g.W + 1
    ldo = ldo or nw
    out = torch.full((g.batch, g.L, ldo), float("nan"), dtype=torch.float32 if g.dtype == "tf32" else torch.bfloat16,
                     device="cuda")
    O.g2bmm(g.batch, g.L, g.K, g.W, g.d, O.TF32 if g.dtype == "tf32" else O.BF16, a.cuda(), b.cuda(), out, ldo, form)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), nw


@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("g", CASES, ids=[c.name for c in CASES])
def test_g2bmm_integer_exact(O, g, form):
    a, b = syn.g2bmm_inputs(g, 700, exact_int=True)
    got, nw = _run(O, g, a, b, form)
    assert np.array_equal(got[..., :nw], _round_like(oracle.g2bmm(a, b, g.W, g.d), g.dtype))


@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("g", CASES, ids=[c.name for c in CASES])
def test_g2bmm_random_tolerance(O, g, form):
    a, b = syn.g2bmm_inputs(g, 701)
    got, nw = _run(O, g, a, b, form)
    assert _max_rel(got[..., :nw], oracle.g2bmm(a, b, g.W, g.d)) <= TOL[g.dtype]


@pytest.mark.parametrize("ldo", [48, 39, 34])          # 16-byte rows; odd pitches (edge-chunk stores)
def test_g2bmm_padded_pitch_leaves_padding(O, ldo):
    g = CASES[1]
    a, b = syn.g2bmm_inputs(g, 702, exact_int=True)
    got, nw = _run(O, g, a, b, 0, ldo=ldo)
    assert np.array_equal(got[..., :nw], _round_like(oracle.g2bmm(a, b, g.W, g.d), g.dtype))
    assert np.isnan(got[..., nw:]).all()


@pytest.mark.parametrize("g", CASES, ids=[c.name for c in CASES])
def test_g2bmm_aligned_pitch_vector_path(O, g):
    a, b = syn.g2bmm_inputs(g, 703, exact_int=True)
    nw = 2 * g.W + 1
    got, _ = _run(O, g, a, b, 0, ldo=(nw + 7) // 8 * 8)
    assert np.array_equal(got[..., :nw], _round_like(oracle.g2bmm(a, b, g.W, g.d), g.dtype))


def test_g2bmm_longformer_full_size(O):
    g = syn.G2_CONFIGS["longformer"][0]
    a, b = syn.g2bmm_inputs(g, 1000)
    got, nw = _run(O, g, a, b, 0)
    assert _max_rel(got, oracle.g2bmm(a, b, g.W, g.d)) <= TOL[g.dtype]


def test_g2bmm_errors(O):
    x = torch.zeros(1, 10, 48, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(1, 10, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as e:
        O.g2bmm(1, 10, 48, 1, 1, O.BF16, x, x, y)
    assert e.value.status == O.E_UNSUPPORTED
    with pytest.raises(O.OllieError) as e:
        O.g2bmm(1, 10, 48, 1, 0, O.BF16, x, x, y)
    assert e.value.status == O.E_INVALID


# with a narrow band (nwb < epilogue warps per TMEM quadrant) some epilogue warps
# read no window; they must still release every TMEM chunk, or a CTA that wraps the 4-buffer ring
# (more than ~2 items per CTA) waits forever.  Many items per CTA, small W, both forms.
@pytest.mark.parametrize("form,W,d", [(0, 8, 4), (0, 15, 2), (1, 7, 2), (1, 3, 4)])
def test_g2bmm_small_band_many_items_per_cta(O, form, W, d):
    g = syn.G2("many_items", 8, 10000, 64, W, d)
    a, b = syn.g2bmm_inputs(g, 703, exact_int=True)
    got, nw = _run(O, g, a, b, form)
    rows = np.r_[0:300, 4900:5300, 9700:10000]                 # sampled rows, every tile position kind
    full = oracle.g2bmm(a, b, g.W, g.d)
    assert np.array_equal(got[:, rows, :nw], _round_like(full[:, rows], g.dtype))


def test_g2bmm_misaligned_out_is_status(O):
    g = CASES[0]
    a, b = syn.g2bmm_inputs(g, 704, exact_int=True)
    buf = torch.zeros(g.batch * g.L * 7 + 1, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(O.OllieError) as ei:
        O.g2bmm(g.batch, g.L, g.K, g.W, g.d, O.BF16, a.cuda(), b.cuda(), buf[1:], 7)
    assert ei.value.status == O.E_ALIGN


def test_merged_gemm_misaligned_T_is_status(O):
    a = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(32, 64, dtype=torch.bfloat16, device="cuda")
    T = torch.zeros(64 * 32 + 1, dtype=torch.float32, device="cuda")
    with pytest.raises(O.OllieError) as ei:
        O.merged_gemm(64, 32, 64, O.BF16, a, b, T[1:], 32)
    assert ei.value.status == O.E_ALIGN
