"""Oracle backward (swin.hpp:370-467) pinned like the reference's own tests: central finite differences
of the oracle forward (itself pinned to the golden probe) on 50 random parameters and 12 input
elements, determinism, and dead paths (test_swin_core.cpp:328-413)."""
import numpy as np

from oracle import pyoracle as o

TINY = o.ModelConfig(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=4,
                     out_channels=2, time_dim=16)


def _input(C, H, W, seed):
    return o.gaussian_fill(seed, H * W * C).reshape(H * W, C)  # x.data()[i] = gaussian(seed, i), col-major


def _R(H, W, seed):
    return o.gaussian_fill(seed, H * W * TINY.out_channels).reshape(H * W, TINY.out_channels)


def test_param_gradients_match_central_differences():  # test_swin_core.cpp:328-366
    p = o.init_params(TINY, 77, random=True)
    H = W = 12
    x, R, t = _input(4, H, W, 78), _R(H, W, 79), 0.8
    g, _ = o.backward(TINY, p, x, t, H, W, R)
    rng = np.random.default_rng(80)
    eps, checked = 1e-3, 0
    while checked < 50:
        i = int(rng.integers(0, p.size))
        orig = p[i]
        p[i] = orig + eps
        lp = float((R * o.forward(TINY, p, x, t, H, W)).sum())
        p[i] = orig - eps
        lm = float((R * o.forward(TINY, p, x, t, H, W)).sum())
        p[i] = orig
        fd, an = (lp - lm) / (2 * eps), g[i]
        if abs(fd) < 1e-7 and abs(an) < 1e-7:
            continue
        assert abs(fd - an) / max(abs(fd), abs(an), 1e-8) < 1e-4, (i, fd, an)
        checked += 1


def test_input_gradient_matches_central_differences():  # :368-393
    p = o.init_params(TINY, 90, random=True)
    H, W = 6, 12
    x, R = _input(4, H, W, 91), _R(H, W, 92)
    _, din = o.backward(TINY, p, x, 0.5, H, W, R)
    rng = np.random.default_rng(93)
    eps = 1e-4
    for _ in range(12):
        i = np.unravel_index(int(rng.integers(0, x.size)), x.shape)
        orig = x[i]
        x[i] = orig + eps
        lp = float((R * o.forward(TINY, p, x, 0.5, H, W)).sum())
        x[i] = orig - eps
        lm = float((R * o.forward(TINY, p, x, 0.5, H, W)).sum())
        x[i] = orig
        fd, an = (lp - lm) / (2 * eps), din[i]
        assert abs(fd - an) / max(abs(fd), abs(an), 1e-8) < 1e-5, (i, fd, an)


def test_deterministic_and_dead_paths():  # :395-413
    p = o.init_params(TINY, 100, random=True)
    x = _input(4, 12, 12, 101)
    R = np.ones((144, 2))
    R[:, 1] = 0.0
    g1, _ = o.backward(TINY, p, x, 0.7, 12, 12, R)
    g2, _ = o.backward(TINY, p, x, 0.7, 12, 12, R)
    assert np.array_equal(g1, g2)
    shapes = o.param_shapes(TINY)
    off = {}
    pos = 0
    for name, r, c in shapes:
        off[name] = (pos, r, c)
        pos += r * c
    names = [n for n, _, _ in shapes]
    wd = [n for n in names if "decode" in n and ("w" in n.split(".")[-1])][0]
    bd = [n for n in names if "decode" in n and n.endswith("b")][0]
    a, r, c = off[wd]
    w_dec = g1[a:a + r * c].reshape(c, r).T  # col-major r x c
    assert np.abs(w_dec[1]).max() == 0.0
    a, r, c = off[bd]
    assert g1[a + 1] == 0.0
