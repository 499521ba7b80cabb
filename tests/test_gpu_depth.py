"""Depth: the full 20-block 1.3B-width model (h=1536, 12 heads, ffn 9216, w=60, C_in=144, C_out=70)
on a 60x120 grid (two windows per layout; odd blocks shifted by 30 with the seam mask) against the
oracle's forward, with init_parameters_random(2024, 0.01) weights. The golden output was produced
by tests/golden/make_depth20.py (float32 oracle, ~8 CPU minutes); the device regenerates the same
weights with swf_init_params (the reference counter RNG, model.hpp:185-223)."""
import os

import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.util import rel_err_per_channel

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "depth20_c2w_60x120.npz")
CFG = dict(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=20, blocks_per_layer=1, window_px=60,
           in_channels=144, out_channels=70, time_dim=1536)
H, W = 60, 120


@pytest.mark.parametrize("prec,tol", [(swf.PREC_BF16, 2e-2), (swf.PREC_FP32, 1e-4)])
def test_depth20_c2_widths_vs_oracle(prec, tol):
    g = np.load(GOLDEN)
    assert list(g["meta"]) == [H, W, 2024, 2025]
    dn = swf.Denoiser(swf.ModelConfig(**CFG), H, W, precision=prec)
    dn.init_params(2024, mode=1, scale=float(g["scale"]))
    x = o.random_field(144, H * W, 2025).astype(np.float32)
    y = dn.forward(x, float(g["t"]))
    dn.close()
    assert rel_err_per_channel(y, g["y"]) <= tol
