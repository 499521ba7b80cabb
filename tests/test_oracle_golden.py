"""Pins the CPU oracle (oracle/swf_oracle.cpp) on the reference's own frozen values.

Each test cites the reference test it restates (proj/tests/*.cpp).
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as o

TINY = o.ModelConfig(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=4,
                     out_channels=2, time_dim=16)  # test_swin_core.cpp:16-27


def test_forward_golden_probe():
    # test_swin_core.cpp:415-422 -- y(1,77) = 1.2440901490316572 at 1e-12 (f64)
    p = o.init_params(TINY, 2024, random=True, scale=0.25)
    x = o.random_field(TINY.in_channels, 144, 2025)
    y = o.forward(TINY, p, x, 0.62831853071795862, 12, 12)
    assert y[77, 1] == pytest.approx(1.2440901490316572, rel=1e-12)


def test_forward_golden_probe_f32_close():
    p = o.init_params(TINY, 2024, random=True, scale=0.25, dtype=np.float32)
    x = o.random_field(TINY.in_channels, 144, 2025).astype(np.float32)
    y = o.forward(TINY, p, x, np.float32(0.62831853071795862), 12, 12)
    assert y[77, 1] == pytest.approx(1.2440901490316572, rel=1e-4)


def test_param_count_golden():
    # test_swin_core.cpp:157-173
    c = o.ModelConfig(1536, 12, 9216, 10, 2, 30, 144, 70)
    assert o.param_count_formula(c) == 1324144198
    # formula == allocation (test_swin_core.cpp:146-155)
    for cfg in (TINY, o.ModelConfig(16, 4, 48, 2, 2, 6, 4, 2, 16)):
        assert sum(r * c for _, r, c in o.param_shapes(cfg)) == o.param_count_formula(cfg)


def test_zero_params_zero_output():
    # test_swin_core.cpp:175-186
    p = np.zeros(o.param_count_formula(TINY))
    arr = o.split_params(TINY, p)
    names = [n for n, _, _ in o.param_shapes(TINY)]
    for a, n in zip(arr, names):
        if n.endswith(".g"):
            a[:] = 1.0
    x = o.random_field(4, 144, 7)
    assert np.abs(o.forward(TINY, p, x, 0.5, 12, 12)).max() == 0.0


def test_nan_input_rejected():
    # test_swin_core.cpp:188-194
    p = o.init_params(TINY, 1, random=True)
    x = o.random_field(4, 144, 8)
    x[5, 1] = np.nan
    with pytest.raises(o.NumericsError):
        o.forward(TINY, p, x, 0.5, 12, 12)


def test_bad_grid_is_config_error():
    p = o.init_params(TINY, 1, random=True)
    with pytest.raises(o.ConfigError):
        o.forward(TINY, p, o.random_field(4, 13 * 12, 8), 0.5, 13, 12)


def test_window_locality_bitwise():
    # test_swin_core.cpp:224-239
    cfg = o.ModelConfig(16, 4, 32, 1, 1, 6, 4, 2, 16)
    p = o.init_params(cfg, 4, random=True)
    H, W = 12, 18
    x = o.random_field(4, H * W, 10)
    perm = o.window_perm(H, W, 6, 0).reshape(H // 6 * (W // 6), 36)
    xz = np.zeros_like(x)
    win = 1 * (W // 6) + 2
    xz[perm[win]] = x[perm[win]]
    y = o.forward(cfg, p, x, 0.4, H, W)
    yz = o.forward(cfg, p, xz, 0.4, H, W)
    assert np.array_equal(y[perm[win]], yz[perm[win]])


def test_permutation_equivariance():
    # test_swin_core.cpp:196-222
    cfg = o.ModelConfig(16, 4, 32, 1, 1, 6, 4, 2, 16)
    p = o.init_params(cfg, 3, random=True)
    H = W = 12
    x = o.random_field(4, H * W, 9)
    perm = o.window_perm(H, W, 6, 0).reshape(4, 36)
    xp = x.copy()
    xp[perm[0]], xp[perm[3]] = x[perm[3]], x[perm[0]]
    y = o.forward(cfg, p, x, 0.3, H, W)
    yp = o.forward(cfg, p, xp, 0.3, H, W)
    assert np.abs(yp[perm[0]] - y[perm[3]]).max() < 1e-12
    assert np.abs(yp[perm[3]] - y[perm[0]]).max() < 1e-12
    assert np.array_equal(y[perm[1]], yp[perm[1]])


def test_time_embedding_distinct():
    # test_swin_core.cpp:315-326
    p = o.init_params(TINY, 32, random=True)
    _, s1 = o.time_embed(TINY, p, 0.3)
    _, s2 = o.time_embed(TINY, p, 0.9)
    assert np.abs(s1[0, :16] - s2[0, :16]).max() > 1e-8
