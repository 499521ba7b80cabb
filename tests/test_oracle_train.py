"""CPU: the training-loss oracle and the data-parallel train_step host logic.

* latitude weights, noise draw and weighted loss against the reference's own known answers
  (test_grid_data.cpp:50-85, test_trigflow.cpp:57-68, 114-146);
* the oracle's diffusion_loss_sample gradient against central differences end to end, restating
  test_trigflow.cpp:148-196 (same config, seeds, kappa and t_key);
* train.train_step's sample assignment / reduction: one process running dp replicas equals
  dp = 2 gloo ranks (world_size 2) and the reference loop written out by hand.
"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o

TRIG_CFG = dict(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=8, out_channels=3,
                time_dim=16)  # test_trigflow.cpp:29-40


def test_latitude_weights_known_answers():
    for lw in (o.latitude_weights, swf.latitude_weights):
        assert np.allclose(lw(2), [1.0, 1.0], rtol=0, atol=1e-12)
        w = lw(4)
        c675, c225 = np.cos(np.radians(67.5)), np.cos(np.radians(22.5))
        mean = (2 * c675 + 2 * c225) / 4
        assert abs(w[0] - c675 / mean) <= 1e-12 and abs(w[1] - c225 / mean) <= 1e-12
        assert abs(w[0] / w[1] - np.tan(np.radians(22.5))) <= 1e-12
        for h in (4, 8, 30, 128):
            w = lw(h)
            assert abs(w.mean() - 1.0) < 1e-9 and w.min() > 0 and w[h // 2] > w[0]


def test_noise_draw_known_answers():
    assert abs(o.noise_draw_from_u(0.0) - 0.19739555984988078) <= 1e-12  # test_trigflow.cpp:60-63
    assert abs(o.noise_draw_from_u(1.0) - np.arctan(500.0)) <= 1e-15


def test_weighted_loss_known_answers():
    err = np.full((4, 3), 0.7)  # 2x2 grid, 3 variables, uniform weights: |V| e^2
    loss, _ = o.weighted_sq_loss(err, np.ones(2), np.ones(3), 2)
    assert abs(loss - 3 * 0.49) <= 1e-15
    e = o.random_field(3, 16, 11)
    l1, _ = o.weighted_sq_loss(e, np.ones(4), np.ones(3), 4)
    l2, _ = o.weighted_sq_loss(e, np.ones(4), 2 * np.ones(3), 4)
    assert l2 == 2.0 * l1  # exact homogeneity in kappa
    with pytest.raises(ValueError):
        o.weighted_sq_loss(err, np.ones(2), np.ones(2), 2)


def test_loss_gradient_matches_central_differences():
    oc = o.ModelConfig(**TRIG_CFG)
    p = o.init_params(oc, 55, random=True)
    H = W = 12
    xp, x0, fo = (o.random_field(c, H * W, k) for c, k in ((3, 61), (3, 62), (2, 63)))
    z = o.random_field(3, H * W, 64)
    alpha, kappa = np.ones(H), np.array([1.0, 0.6, 1.7])
    loss, g = o.loss_sample(oc, p, H, W, xp, x0, fo, alpha, kappa, 4242, z)
    assert loss > 0
    rng = np.random.default_rng(65)
    eps, checked = 1e-3, 0
    while checked < 50:
        i = int(rng.integers(0, p.size))
        q = p.copy()
        q[i] += eps
        lp, _ = o.loss_sample(oc, q, H, W, xp, x0, fo, alpha, kappa, 4242, z)
        q[i] -= 2 * eps
        lm, _ = o.loss_sample(oc, q, H, W, xp, x0, fo, alpha, kappa, 4242, z)
        fd = (lp - lm) / (2 * eps)
        if abs(fd) < 1e-7 and abs(g[i]) < 1e-7:
            continue
        assert abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-8) < 1e-4, i
        checked += 1


class OracleEngine:
    """The train_step engine interface over the oracle (test infrastructure only)."""

    def __init__(self, oc, params, H, W):
        self.oc, self.p, self.H, self.W = oc, params, H, W
        self.acc = np.zeros_like(params)

    def train_reset(self):
        self.acc[:] = 0

    def train_accumulate(self, x_prev, x0, forc, w, dc, run_seed, sid):
        z = o.noise_field(run_seed, sid, self.oc.out_channels, self.H, self.W, self.oc.window_px, dc.sigma_d)
        loss, g = o.loss_sample(self.oc, self.p, self.H, self.W, x_prev, x0, forc, w.alpha_row, w.kappa,
                                o.key_derive(run_seed, 0x74, sid), z, dc.sigma_d, dc.sigma_min, dc.sigma_max)
        self.acc += g
        return loss

    def train_grads_device(self):
        return None

    def train_read(self, scale):
        return self.acc * scale


def _dataset(H, W, n=3):
    k = 900
    st, fo, rs = [], [], []
    for i in range(n):
        st.append(o.random_field(3, H * W, k + 3 * i))
        fo.append(o.random_field(2, H * W, k + 3 * i + 1))
        rs.append(o.random_field(3, H * W, k + 3 * i + 2))
    return swf.DataSet(st, fo, rs)


def _setup():
    oc = o.ModelConfig(**TRIG_CFG)
    p = o.init_params(oc, 56, random=True, scale=0.1)
    return oc, p, 12, 12, _dataset(12, 12), swf.LossWeights.make(12, [1.0, 0.6, 1.7]), swf.DiffusionConfig()


def test_train_step_single_rank_matches_reference_loop():
    oc, p, H, W, data, w, dc = _setup()
    res = swf.train.train_step(OracleEngine(oc, p, H, W), data, 5, 2, 2, w, dc, 31)
    acc, losses = np.zeros_like(p), []
    for d in range(2):
        for g in range(2):
            sid = 5 + d * 2 + g
            i = sid % 3
            z = o.noise_field(31, sid, 3, H, W, 6)
            l_, gr = o.loss_sample(oc, p, H, W, data.states[i], data.residuals[i], data.forcings[i], w.alpha_row,
                                   w.kappa, o.key_derive(31, 0x74, sid), z)
            acc += gr
            losses.append(l_)
    assert res.mb_losses == losses
    assert abs(res.loss - sum(losses) / 4) <= 1e-15 * max(1.0, abs(res.loss))
    assert np.array_equal(res.grads, acc * 0.25)


def _dp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oc, p, H, W, data, w, dc = _setup()
        res = swf.train.train_step(OracleEngine(oc, p, H, W), data, 5, world, 2, w, dc, 31, group=dist.group.WORLD)
        if rank == 0:
            q.put((res.loss, res.mb_losses, res.grads))
    finally:
        dist.destroy_process_group()


def test_train_step_dp2_gloo_matches_single_rank():
    oc, p, H, W, data, w, dc = _setup()
    ref = swf.train.train_step(OracleEngine(oc, p, H, W), data, 5, 2, 2, w, dc, 31)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    loss, mbl, grads = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert mbl == ref.mb_losses
    assert abs(loss - ref.loss) <= 1e-12 * abs(ref.loss)
    # replica sums meet in fp32 on the wire (the device accumulator's type)
    assert np.abs(grads - ref.grads).max() <= 1e-6 * np.abs(ref.grads).max()


def test_train_step_rejects_bad_arguments():
    oc, p, H, W, data, w, dc = _setup()
    eng = OracleEngine(oc, p, H, W)
    with pytest.raises(ValueError):
        swf.train.train_step(eng, swf.DataSet([], [], []), 0, 1, 1, w, dc, 1)
    with pytest.raises(ValueError):
        swf.train.train_step(eng, data, 0, 1, 0, w, dc, 1)
    with pytest.raises(ValueError):
        swf.LossWeights.make(4, [1.0, 0.0])
    eng.wp_world = 2  # a window-parallel replica cannot run without its process group
    with pytest.raises(ValueError):
        swf.train.train_step(eng, data, 0, 1, 1, w, dc, 1)
