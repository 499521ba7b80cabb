"""Single-process multi-GPU groups (swf_set_topology_devices): one host call drives every rank of a
WP x SP topology -- rank r on device_ids[r], several ranks per device when the box has fewer GPUs
(the driver's 1-GPU box runs all of them on cuda:0) -- with in-process peer mapping instead of IPC
and no torch.distributed. The group's outputs must equal the single-device outputs BITWISE
(ownership only permutes independent windows / rows; the GEMM K order does not depend on M) and
match the oracle (window.hpp / topology.hpp semantics: simulator.hpp:431-530, 781-824)."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.util import rel_err_per_channel

pytestmark = pytest.mark.gpu

C1 = dict(hidden_dim=128, n_heads=4, ffn_dim=256, n_layers=2, window_px=8, in_channels=8, out_channels=3,
          time_dim=128)
MID = dict(hidden_dim=256, n_heads=2, ffn_dim=512, n_layers=3, window_px=12, in_channels=16, out_channels=6,
           time_dim=256)
MID4 = dict(hidden_dim=512, n_heads=4, ffn_dim=1024, n_layers=2, window_px=12, in_channels=16, out_channels=6,
            time_dim=256)
GRIDS = {"C1": (C1, 32, 64), "MID": (MID, 48, 96), "MID4": (MID4, 48, 96)}
# (wp_a, wp_b, sp, ownership)
TOPOS = [(1, 2, 1, swf.OWN_CONTIGUOUS), (1, 2, 1, swf.OWN_ROUND_ROBIN), (2, 2, 1, swf.OWN_CONTIGUOUS),
         (1, 1, 2, swf.OWN_CONTIGUOUS), (1, 2, 2, swf.OWN_CONTIGUOUS), (2, 4, 1, swf.OWN_CONTIGUOUS),
         (2, 2, 2, swf.OWN_ROUND_ROBIN)]


def ngpus():
    import torch
    return torch.cuda.device_count()


def devices(world):
    n = max(1, ngpus())
    return [r % n for r in range(world)]


def setup(name, seed=7):
    d, H, W = GRIDS[name]
    oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
    p = o.init_params(oc, seed, random=True, scale=0.03, dtype=np.float32)
    x = o.random_field(oc.in_channels, H * W, seed + 1).astype(np.float32)
    return oc, sc, p, x, H, W


@pytest.fixture(scope="module")
def singles():
    out = {}
    for name in GRIDS:
        oc, sc, p, x, H, W = setup(name)
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16)
        dn.load_params(p)
        out[name] = (dn.forward(x, 0.9), o.forward(oc, p, x, np.float32(0.9), H, W))
        dn.close()
    return out


@pytest.mark.parametrize("topo", TOPOS, ids=lambda t: f"wp{t[0]}x{t[1]}_sp{t[2]}_own{t[3]}")
@pytest.mark.parametrize("name", list(GRIDS))
def test_group_forward_bitwise(singles, name, topo):
    wa, wb, sp, own = topo
    oc, sc, p, x, H, W = setup(name)
    if oc.n_heads % sp or oc.window_px % sp or (H // oc.window_px) % wa or (W // oc.window_px) % wb:
        pytest.skip("topology does not divide this model / grid (build_topology constraints)")
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16, topology=topo, devices=devices(wa * wb * sp))
    assert dn.group_size() == wa * wb * sp
    dn.load_params(p)
    y = dn.forward(x, 0.9)
    y2 = dn.forward(x, 0.9)  # repeated calls exercise the start-of-forward barrier and epochs
    dn.close()
    single, ref = singles[name]
    assert np.array_equal(y, y2)
    assert np.array_equal(y, single)
    assert rel_err_per_channel(y, ref) <= 2e-2


def test_group_forecast_and_rollout_bitwise():
    """Sampler entry points (graph-captured solve with barriers inside) on a WP 1x2 group."""
    oc, sc, p, _, H, W = setup("C1", 300)
    x0 = o.random_field(3, H * W, 301).astype(np.float32)
    forc = [o.random_field(2, H * W, 302 + k).astype(np.float32) for k in range(2)]
    dc = swf.DiffusionConfig(solver_steps=3, churn=0.5)
    res = {}
    for grp in (False, True):
        kw = dict(topology=(1, 2, 1, swf.OWN_CONTIGUOUS), devices=devices(2)) if grp else {}
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16, **kw)
        dn.load_params(p)
        res[grp] = ([dn.forecast_step(x0, forc[0], dc, 11, o.key_derive(41, k, 0)) for k in range(3)],
                    dn.rollout_ensemble(x0, forc, 2, 2, dc, 11, 77))
        dn.close()
    for a, b in zip(res[False][0], res[True][0]):
        assert np.array_equal(a, b)
    assert np.array_equal(res[False][1], res[True][1])


def test_group_nan_raises_same_error_on_every_rank():
    """A NaN inside one rank's windows: the flags are OR-reduced across ranks at the barriers, so the
    group (every rank) raises NumericsError naming the input (check_finite, swin.hpp:295-300)."""
    oc, sc, p, x, H, W = setup("C1")
    owner = swf.plan_owners(H, W, 8, 1, 2)
    perm = o.window_perm(H, W, 8, 0).reshape(-1, 64)
    pix = int(perm[int(np.argmax(owner == 1))][5])  # a pixel of a window rank 1 owns
    x[pix, 2] = np.nan
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16, topology=(1, 2, 1, swf.OWN_CONTIGUOUS), devices=devices(2))
    dn.load_params(p)
    with pytest.raises(swf.NumericsError, match="input"):
        dn.forward(x, 0.5)
    x[pix, 2] = 0.0  # the group recovers: the next call succeeds
    assert np.isfinite(dn.forward(x, 0.5)).all()


def test_group_backward_fp32_matches_single():
    """FP32 validation-mode backward on a WP 1x2 group: per-rank partial gradients summed in rank
    order equal the single-device gradients within fp32 summation-order noise."""
    oc, sc, p, x, H, W = setup("C1", 77)
    R = o.random_field(3, H * W, 79).astype(np.float32)
    out = {}
    for grp in (False, True):
        kw = dict(topology=(1, 2, 1, swf.OWN_CONTIGUOUS), devices=devices(2)) if grp else {}
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32, **kw)
        dn.load_params(p)
        out[grp] = dn.backward(x, 0.8, R)
        dn.close()
    g1, d1 = out[False]
    g2, d2 = out[True]
    assert float(np.abs(g1 - g2).max()) <= 1e-5 * float(np.abs(g1).max())
    assert np.array_equal(d1, d2) or float(np.abs(d1 - d2).max()) <= 1e-5 * float(np.abs(d1).max())


def test_group_c4_width_sp2_vs_oracle():
    """Wide-layer slice of the 40B shape (BASELINE configs[3]): h = 6144, 48 heads (d = 128), sequence
    parallel SP = 2 inside 12 x 12 windows (heads and window rows split over the two ranks, the
    all-to-alls fused into the QKV / attention epilogues), 2 blocks (shift 0, 6 with the seam mask) on
    a 12 x 24 grid, weights generated on the device with the reference init (swf_init_params)."""
    d = dict(hidden_dim=6144, n_heads=48, ffn_dim=6144, n_layers=2, window_px=12, in_channels=16,
             out_channels=6, time_dim=128)
    H, W = 12, 24
    oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
    x = o.random_field(16, H * W, 9).astype(np.float32)
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16, topology=(1, 1, 2, swf.OWN_CONTIGUOUS), devices=devices(2))
    dn.init_params(2024, mode=1, scale=0.004)
    y = dn.forward(x, 0.9)
    dn.close()
    one = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16)
    one.init_params(2024, mode=1, scale=0.004)
    y1 = one.forward(x, 0.9)
    one.close()
    assert np.array_equal(y, y1)
    p = o.init_params(oc, 2024, random=True, scale=0.004, dtype=np.float32)
    ref = o.forward(oc, p, x, np.float32(0.9), H, W)
    assert rel_err_per_channel(y, ref) <= 2e-2


def test_group_train_step_matches_single():
    """reference_train_step (simulator.hpp:50-86) on a WP 1x2 single-process group: the ranks' partial
    losses / gradients over their own windows are summed by the group, no process group needed."""
    d = dict(hidden_dim=64, n_heads=4, ffn_dim=128, n_layers=2, window_px=8, in_channels=8, out_channels=3,
             time_dim=64)
    H, W = 32, 64
    oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
    p = o.init_params(oc, 57, random=True, scale=0.05, dtype=np.float32)
    data = swf.DataSet(*[[o.random_field(c, H * W, 900 + 3 * i + j).astype(np.float32) for i in range(3)]
                         for j, c in ((0, 3), (1, 2), (2, 3))])
    w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
    res = {}
    for grp in (False, True):
        kw = dict(topology=(1, 2, 1, swf.OWN_CONTIGUOUS), devices=devices(2)) if grp else {}
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32, **kw)
        dn.load_params(p)
        res[grp] = dn.train_step(data, 3, 2, 2, w, swf.DiffusionConfig(), 31)
        dn.close()
    a, b = res[False], res[True]
    assert np.allclose(a.mb_losses, b.mb_losses, rtol=1e-6, atol=0)
    assert float(np.abs(a.grads - b.grads).max()) <= 1e-5 * float(np.abs(a.grads).max())
