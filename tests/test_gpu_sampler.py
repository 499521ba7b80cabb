"""Device-resident sampler vs the oracle beyond the identity / churn-free case: the churn rotation
(diffusion.hpp:255-268), non-identity Standardizers (grid.hpp:127-132 via forecast_step,
diffusion.hpp:295-319) and rollout_ensemble (diffusion.hpp:323-339, mirroring
test_trigflow.cpp:372-406), in the FP32 validation mode (1e-4) and on the BF16 path (2e-2)."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.util import rel_err_per_channel

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-4
TOL_BF16 = 2e-2
TINY = dict(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=8, out_channels=3,
            time_dim=16)  # tiny_config with 3 + 3 + 2 channels (test_trigflow.cpp:372-380)
C1 = dict(hidden_dim=128, n_heads=4, ffn_dim=256, n_layers=2, window_px=8, in_channels=8, out_channels=3,
          time_dim=128)


def cfgs(d):
    return o.ModelConfig(**d), swf.ModelConfig(**d)


def stats(seed):
    """Non-identity Standardizers: (mean, std) of state (3), residual (3), forcing (2)."""
    rng = np.random.default_rng(seed)
    mk = lambda n: (rng.normal(0.0, 2.0, n), rng.uniform(0.3, 3.0, n))
    return mk(3), mk(3), mk(2)


def dev_stats(st, dtype):
    (sm, ss), (rm, rsd), (fm, fs) = st
    return [a.astype(dtype) for a in (sm, ss, rm, rsd, fm, fs)]


@pytest.mark.parametrize("churn", [0.5, 1.0])
def test_forecast_step_churn_fp32_mode(churn):
    oc, sc = cfgs(TINY)
    p = o.init_params(oc, 200, random=True, scale=0.05)
    x0 = o.random_field(3, 144, 201)
    forc = o.random_field(2, 144, 202)
    ev = o.key_derive(31, 0, 0)
    # 9 steps: churn is active on steps 3..5 (ChurnSchedule: S/3 <= k < 2S/3, not the last)
    ref, fe = o.forecast_step(oc, p, 12, 12, x0, forc, 7, ev, steps=9, churn=churn)
    ref0, _ = o.forecast_step(oc, p, 12, 12, x0, forc, 7, ev, steps=9, churn=0.0)
    dn = swf.Denoiser(sc, 12, 12, precision=swf.PREC_FP32)
    dn.load_params(p)
    got = dn.forecast_step(x0.astype(np.float32), forc.astype(np.float32),
                           swf.DiffusionConfig(solver_steps=9, churn=churn), 7, ev)
    assert fe == 18
    assert rel_err_per_channel(got, ref) <= TOL_FP32
    # the churn changes the result well beyond the tolerance (the comparison sees the rotation)
    assert rel_err_per_channel(ref0, ref) > 20 * TOL_FP32


def test_forecast_step_standardizers_fp32_mode():
    oc, sc = cfgs(TINY)
    p = o.init_params(oc, 210, random=True, scale=0.05)
    st = stats(3)
    x0 = 2.0 + 3.0 * o.random_field(3, 144, 211)
    forc = -1.0 + 0.5 * o.random_field(2, 144, 212)
    ev = o.key_derive(32, 0, 0)
    ref, _ = o.forecast_step(oc, p, 12, 12, x0, forc, 9, ev, st=st[0], rs=st[1], fo=st[2], steps=4)
    dn = swf.Denoiser(sc, 12, 12, precision=swf.PREC_FP32)
    dn.load_params(p)
    got = dn.forecast_step(x0.astype(np.float32), forc.astype(np.float32), swf.DiffusionConfig(solver_steps=4), 9,
                           ev, stds=dev_stats(st, np.float32))
    # compare the sampled residual (out - x_prev) in physical units, per channel
    assert rel_err_per_channel(got - x0, ref - x0) <= TOL_FP32
    ident, _ = o.forecast_step(oc, p, 12, 12, x0, forc, 9, ev, steps=4)
    assert rel_err_per_channel(ident - x0, ref - x0) > 0.1  # the statistics matter


def test_forecast_step_churn_standardizers_bf16_c1():
    oc, sc = cfgs(C1)
    p = o.init_params(oc, 300, random=True, scale=0.02, dtype=np.float32)
    st = stats(4)
    x0 = (1.0 + 2.0 * o.random_field(3, 2048, 301)).astype(np.float32)
    forc = o.random_field(2, 2048, 302).astype(np.float32)
    ev = o.key_derive(41, 1, 0)
    st32 = tuple(tuple(a.astype(np.float32) for a in pair) for pair in st)
    ref, _ = o.forecast_step(oc, p, 32, 64, x0, forc, 11, ev, st=st32[0], rs=st32[1], fo=st32[2], steps=6, churn=0.5)
    dn = swf.Denoiser(sc, 32, 64, precision=swf.PREC_BF16)
    dn.load_params(p)
    got = dn.forecast_step(x0, forc, swf.DiffusionConfig(solver_steps=6, churn=0.5), 11, ev,
                           stds=dev_stats(st, np.float32))
    assert rel_err_per_channel(got - x0, ref - x0) <= TOL_BF16


def test_rollout_ensemble_fp32_mode():
    """test_trigflow.cpp:372-406 on the device: 2 members x 3 steps equal the oracle's rollout; member 0
    equals chained forecast_step calls with events key_derive(31, 0, k) bitwise; members differ."""
    oc, sc = cfgs(TINY)
    p = o.init_params(oc, 200, random=True, scale=0.05)
    x0 = o.random_field(3, 144, 201)
    forcings = [o.random_field(2, 144, 202)] * 3
    st = stats(5)
    ref = o.rollout_ensemble(oc, p, 12, 12, x0, forcings, 2, 3, 7, 31, st=st[0], rs=st[1], fo=st[2], steps=4)
    dn = swf.Denoiser(sc, 12, 12, precision=swf.PREC_FP32)
    dn.load_params(p)
    dc = swf.DiffusionConfig(solver_steps=4)
    ens = dn.rollout_ensemble(x0.astype(np.float32), [f.astype(np.float32) for f in forcings], 2, 3, dc, 7, 31,
                              stds=dev_stats(st, np.float32))
    assert ens.shape == (2, 3, 144, 3)
    for m in range(2):
        for k in range(3):
            assert rel_err_per_channel(ens[m, k] - x0, ref[m, k] - x0) <= TOL_FP32, (m, k)
    x = x0.astype(np.float32)
    for k in range(3):
        x = dn.forecast_step(x, forcings[k].astype(np.float32), dc, 7, o.key_derive(31, 0, k),
                             stds=dev_stats(st, np.float32))
        assert np.array_equal(x, ens[0, k]), k
    assert np.abs(ens[0, 0] - ens[1, 0]).max() > 0.0


def test_rollout_ensemble_bf16_c1_graph_replay():
    """BF16 rollout (2 members x 2 steps, churn on): the sampler graph captured on the second
    forecast serves every later member / step; the result matches the oracle rollout."""
    oc, sc = cfgs(C1)
    p = o.init_params(oc, 320, random=True, scale=0.02, dtype=np.float32)
    x0 = o.random_field(3, 2048, 321).astype(np.float32)
    forcings = [o.random_field(2, 2048, 322 + k).astype(np.float32) for k in range(2)]
    ref = o.rollout_ensemble(oc, p, 32, 64, x0, forcings, 2, 2, 13, 77, steps=3, churn=0.5)
    dn = swf.Denoiser(sc, 32, 64, precision=swf.PREC_BF16)
    dn.load_params(p)
    ens = dn.rollout_ensemble(x0, forcings, 2, 2, swf.DiffusionConfig(solver_steps=3, churn=0.5), 13, 77)
    for m in range(2):
        for k in range(2):
            assert rel_err_per_channel(ens[m, k] - x0, ref[m, k] - x0) <= TOL_BF16, (m, k)
