"""The reference's ops leaves (swin.hpp:49-234) through the C-ABI on the device, against float64
numpy restatements of the reference formulas: linear_cols (:49-54), prenorm_modulate /
prenorm_plain (:72-85, 111-123, eps 1e-8 inside the sqrt), swiglu_fwd (:228-234)."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from tests.util import rel_err_per_channel

pytestmark = pytest.mark.gpu


def rng(seed):
    return np.random.default_rng(seed)


@pytest.mark.parametrize("prec,tol", [(swf.PREC_FP32, 1e-5), (swf.PREC_BF16, 2e-2)])
@pytest.mark.parametrize("out,inp,n", [(384, 128, 300), (70, 1536, 257), (1536, 144, 1000)])
def test_linear_cols(prec, tol, out, inp, n):
    r = rng(out + inp)
    W = r.standard_normal((inp, out)).astype(np.float32) / np.sqrt(inp)  # col-major out x in = [in][out]
    X = r.standard_normal((n, inp)).astype(np.float32)
    Y = swf.ops.linear_cols(W, out, inp, X, precision=prec)
    ref = X.astype(np.float64) @ W.astype(np.float64)
    assert rel_err_per_channel(Y, ref) <= tol


@pytest.mark.parametrize("modulated", [True, False])
def test_prenorm_modulate(modulated):
    r = rng(3)
    n, h = 500, 256
    X = (3.0 * r.standard_normal((n, h))).astype(np.float32)
    g, a, b, gate = (r.standard_normal(h).astype(np.float32) for _ in range(4))
    Y = swf.ops.prenorm_modulate(X, g, *((a, b, gate) if modulated else (None, None, None)))
    x = X.astype(np.float64)
    u = x / np.sqrt((x ** 2).mean(axis=1, keepdims=True) + 1e-8) * g
    ref = gate * (u * (1 + a) + b) if modulated else u
    assert rel_err_per_channel(Y, ref) <= 1e-5
    X[7, 3] = np.inf
    with pytest.raises(swf.NumericsError):
        swf.ops.prenorm_modulate(X, g)


@pytest.mark.parametrize("prec,tol", [(swf.PREC_FP32, 1e-5), (swf.PREC_BF16, 2e-2)])
def test_swiglu_fwd(prec, tol):
    r = rng(5)
    n, h, f = 400, 128, 384
    Wg = r.standard_normal((h, f)).astype(np.float32) / np.sqrt(h)
    Wu = r.standard_normal((h, f)).astype(np.float32) / np.sqrt(h)
    Wd = r.standard_normal((f, h)).astype(np.float32) / np.sqrt(f)
    X = r.standard_normal((n, h)).astype(np.float32)
    Y = swf.ops.swiglu_fwd(Wg, Wu, Wd, h, f, X, precision=prec)
    x = X.astype(np.float64)
    g, u = x @ Wg, x @ Wu
    ref = (g / (1 + np.exp(-g)) * u) @ Wd
    assert rel_err_per_channel(Y, ref) <= tol
