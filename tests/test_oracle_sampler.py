"""Sampler KATs (proj/tests/test_trigflow.cpp)."""
import math

import numpy as np
import pytest

from oracle import pyoracle as o


def test_t_endpoints():
    # test_trigflow.cpp:58-81
    assert o.t_of_sigma(0.2) == pytest.approx(0.19739555984988078, rel=1e-12)
    assert o.t_of_sigma(500.0) == pytest.approx(1.5687963294615568, rel=1e-12)


def test_two_evals_per_step():
    # test_trigflow.cpp:239-252
    x = o.random_field(2, 9, 80).ravel()
    assert o.solve_gaussian(x)[1] == 20
    assert o.solve_gaussian(x, steps=5)[1] == 10


def test_pinned_contraction():
    # test_trigflow.cpp:296-306
    out, _ = o.solve_gaussian(np.ones(1))
    assert out[0] == pytest.approx(0.968827, rel=1e-4)


def test_churn_determinism():
    # test_trigflow.cpp:254-269
    x = o.random_field(2, 16, 81).ravel()
    a, _ = o.solve_gaussian(x, 0.4, 0.7, 1.0, churn_key=1)
    b, _ = o.solve_gaussian(x, 0.4, 0.7, 1.0, churn_key=2)
    assert np.array_equal(a, b)
    c1, _ = o.solve_gaussian(x, 0.4, 0.7, 1.0, churn=1.0, churn_key=7)
    c2, _ = o.solve_gaussian(x, 0.4, 0.7, 1.0, churn=1.0, churn_key=7)
    c3, _ = o.solve_gaussian(x, 0.4, 0.7, 1.0, churn=1.0, churn_key=8)
    assert np.array_equal(c1, c2)
    assert np.abs(c1 - c3).max() > 0 and np.abs(c1 - a).max() > 0


def test_second_order_convergence():
    # test_trigflow.cpp:308-341 (exact endpoint via fine RK4 of the same linear ODE)
    mu, s0, sd = 0.8, 0.5, 1.0
    x0 = o.random_field(1, 8, 84).ravel()

    def vel(x, t):
        c, s = math.cos(t), math.sin(t)
        den = c * c * s0 * s0 + s * s * sd * sd
        dev = x - c * mu
        return c * (s * sd * sd / den) * dev - s * (mu + (c * s0 * s0 / den) * dev)

    t0, t1 = o.t_of_sigma(500.0), o.t_of_sigma(0.2)
    n = 20000
    dt = (t1 - t0) / n
    x, t = x0.copy(), t0
    for _ in range(n):
        k1 = vel(x, t)
        k2 = vel(x + 0.5 * dt * k1, t + 0.5 * dt)
        k3 = vel(x + 0.5 * dt * k2, t + 0.5 * dt)
        k4 = vel(x + dt * k3, t + dt)
        x = x + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        t += dt
    e10 = np.linalg.norm(o.solve_gaussian(x0, mu, s0, sd, steps=10)[0] - x)
    e20 = np.linalg.norm(o.solve_gaussian(x0, mu, s0, sd, steps=20)[0] - x)
    slope = math.log2(e10 / e20)
    assert 1.7 < slope < 2.3


def test_divergence_raises():
    # test_trigflow.cpp:343-350
    with pytest.raises(o.NumericsError):
        o.solve_affine(o.random_field(1, 4, 85).ravel(), 1e155, 1e155)


def test_forecast_step_runs_and_counts_evals():
    cfg = o.ModelConfig(16, 4, 32, 2, 1, 6, 8, 3, 16)
    p = o.init_params(cfg, 200, random=True, scale=0.05)
    x0 = o.random_field(3, 144, 201)
    forc = o.random_field(2, 144, 202)
    out, fe = o.forecast_step(cfg, p, 12, 12, x0, forc, 7, o.key_derive(31, 0, 0), steps=4)
    assert fe == 8 and np.isfinite(out).all()
