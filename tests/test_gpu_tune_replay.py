"""Autotune record / replay (OLLIE_TUNE_FILE, ollie.cu ollie_autotune_derived): the first autotune of a
shape appends its decision to the file; a later autotune of the same shape replays it without
measuring (profiler runs use this to execute the timed bench's plans).  Both runs must match the
oracle bit for bit in integer mode."""
import numpy as np
import pytest
import torch

import ollie_synth as syn
from tests.test_gpu_parity import _dev, _oracle_layer, _round_like

pytestmark = pytest.mark.gpu

LAYERS = [syn.Layer("tr_conv", 2, 64, 14, 14, 64, 3, 3, pad=1),
          syn.Layer("tr_convt", 2, 64, 5, 5, 32, 4, 4, pad=1, stride=2, transposed=True)]


@pytest.mark.parametrize("lay", LAYERS, ids=lambda l: l.name)
def test_tune_record_then_replay(lay, tmp_path, monkeypatch):
    from paper_2208_02025_b200 import DerivedConv
    f = tmp_path / "tune.txt"
    monkeypatch.setenv("OLLIE_TUNE_FILE", str(f))
    x, w = syn.layer_inputs(lay, 11, exact_int=True)
    ref = _round_like(_oracle_layer(lay, x, w), lay.dtype)
    outs = []
    for _ in range(2):   # first: measure + record; second: replay the recorded line
        conv = DerivedConv.from_layer(lay).prepare(_dev(w))
        y = conv(_dev(x))
        torch.cuda.synchronize()
        outs.append(y.float().cpu().numpy())
    lines = f.read_text().split("\n")
    lines = [ln for ln in lines if ln]
    assert len(lines) == 1, lines                      # recorded once, replayed the second time
    key, decision, idx = lines[0].split()
    assert key.split(",")[:5] == [str(v) for v in (lay.n, lay.c, lay.h, lay.w, lay.f)]
    assert decision in ("f", "u", "r") and int(idx) >= 0
    for got in outs:
        assert np.array_equal(got, ref)
