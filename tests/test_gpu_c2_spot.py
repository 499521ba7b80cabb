"""Full-size parity at the C2 shape (720x1440 grid, h=1536, 12 heads, d=128, ffn 9216, w=60), per
block: a 2-block model (shift 0, then shift 30) runs on the whole grid on the GPU, and the residual
stream is read back after the encode, after block 0 and after block 1 (swf_forward_hidden). Each
block's increment dx = x_out - x_in of selected windows is recomputed by the oracle's
block_window_forward (swin.hpp:306-325) from the GPU's own block input, so errors do not compound
and the comparison sees the block itself, not the identity path. A window's block output depends
only on that window's input (test_swin_core.cpp:224-239).

Windows: an interior window and a bottom-row window of each layout; on the shifted block the
bottom-row window is the seam-masked one (window.hpp:107-122) and is assembled from four block-0
windows. Weights: init_parameters_random(seed, 0.01) -- every branch live (zeroing W_out or W_down
moves the increments by far more than the 2e-2 bar; the negative controls below prove it)."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.util import rel_err_per_channel

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
H, W, w = 720, 1440, 60
NX = W // w
CFG = dict(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=1, blocks_per_layer=2, window_px=60,
           in_channels=144, out_channels=70, time_dim=1536)
WINDOWS = [(5, 7), (11, 3)]  # interior; bottom row (seam-masked under the shift)
T = 0.7


def _rms_norm(x, g):
    r = np.sqrt((x.astype(np.float64) ** 2).mean(axis=1, keepdims=True) + 1e-8)
    return (x / r) * g


@pytest.fixture(scope="module")
def c2():
    oc, sc = o.ModelConfig(**CFG), swf.ModelConfig(**CFG)
    p = o.init_params(oc, 2024, random=True, scale=0.01, dtype=np.float32)
    names = [n for n, _, _ in o.param_shapes(oc)]
    x = np.random.default_rng(5).standard_normal((H * W, 144)).astype(np.float32)
    perm = [o.window_perm(H, W, w, s).reshape(-1, w * w) for s in (0, w // 2)]
    pix = [np.concatenate([perm[b][wy * NX + wx] for wy, wx in WINDOWS]) for b in (0, 1)]
    allpix = np.concatenate(pix)
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16)
    dn.load_params(p)
    hid = [dn.forward_hidden(x, T, nb, allpix) for nb in (0, 1, 2)]
    y = dn.forward(x, T)
    dn.close()
    n0 = pix[0].size
    gpu = {
        "x0_b0": hid[0][:n0], "x1_b0": hid[1][:n0],  # block 0 windows: input / output
        "x0_b1": hid[1][n0:], "x1_b1": hid[2][n0:],  # block 1 windows
        "y": y, "x_final": hid[2][n0:],
    }
    # oracle increments from the GPU's own block inputs
    ref = {}
    for b in (0, 1):
        xin = gpu[f"x0_b{b}"].reshape(len(WINDOWS), w * w, -1)
        ref[b] = [o.block_window(oc, p, T, H, W, b, wy, wx, xin[i]) - xin[i] for i, (wy, wx) in enumerate(WINDOWS)]
    return dict(oc=oc, sc=sc, p=p, names=names, x=x, pix=pix, gpu=gpu, ref=ref, allpix=allpix)


def _increment_errors(c, blocks):
    """Per-window per-channel errors of GPU increments against the oracle's: blocks = {b: (x_in, x_out)}
    with the rows of that block's windows (WINDOWS order)."""
    errs = {}
    for b, (xi, xo) in blocks.items():
        d = (xo - xi).reshape(len(WINDOWS), w * w, -1)
        for i, win in enumerate(WINDOWS):
            errs[(b, win)] = rel_err_per_channel(d[i], c["ref"][b][i])
    return errs


def test_c2_encode(c2):
    p, names = c2["p"], c2["names"]
    arr = o.split_params(c2["oc"], p)
    Wenc = arr[0].reshape(144, 1536).astype(np.float64)  # col-major (h x C_in) -> [in][out]
    pix = c2["pix"][0]
    ref = c2["x"][pix].astype(np.float64) @ Wenc + arr[1]
    assert rel_err_per_channel(c2["gpu"]["x0_b0"], ref) <= TOL_BF16


def test_c2_block_increments(c2):
    """Block 0 (unshifted) and block 1 (shifted, seam-masked bottom row) increments vs the oracle."""
    g = c2["gpu"]
    errs = _increment_errors(c2, {0: (g["x0_b0"], g["x1_b0"]), 1: (g["x0_b1"], g["x1_b1"])})
    bad = {k: v for k, v in errs.items() if v > TOL_BF16}
    assert not bad, errs
    # the increments are not vanishing: the block changes the stream by O(0.01-0.1) per element
    for b in (0, 1):
        for dref in c2["ref"][b]:
            assert np.abs(dref).max() > 1e-2


def test_c2_decode(c2):
    arr = o.split_params(c2["oc"], c2["p"])
    names = c2["names"]
    g = arr[names.index("decode.g")]
    Wd = arr[names.index("decode.w")].reshape(1536, 70).astype(np.float64)
    ref = _rms_norm(c2["gpu"]["x_final"].astype(np.float64), g) @ Wd + arr[names.index("decode.b")]
    got = c2["gpu"]["y"][c2["pix"][1]]
    assert rel_err_per_channel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("kill", ["out.w", "down.w", "ada.w"])
def test_c2_negative_controls(c2, kill):
    """The increments test has teeth: a GPU model with one block array zeroed (attention output
    projection, FFN down projection, or the AdaLN modulation weights) must fail it against the intact
    oracle."""
    p2 = c2["p"].copy()
    arrs = o.split_params(c2["oc"], p2)
    for b in (0, 1):
        arrs[c2["names"].index(f"block{b}.{kill}")][:] = 0
    dn = swf.Denoiser(c2["sc"], H, W, precision=swf.PREC_BF16)
    dn.load_params(p2)
    hid = [dn.forward_hidden(c2["x"], T, nb, c2["allpix"]) for nb in (0, 1)]
    dn.close()
    n0 = c2["pix"][0].size
    # block 0's input (the encode) is untouched, so its increments face the intact oracle's directly
    errs = _increment_errors(c2, {0: (hid[0][:n0], hid[1][:n0])})
    assert min(errs.values()) > 5 * TOL_BF16, errs
