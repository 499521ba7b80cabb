"""f3 on the tensor cores: the BF16 training mode (swf_set_backward_precision(BF16)) runs every
linear layer of the training forward, of the backward's recomputation and of the backward itself as
tcgen05 BF16 GEMMs (data gradients with K-major operands, weight gradients with MN-major operands and
K = tokens); attention and the norms stay FP32. The GEMM against float64 products of the same bf16-rounded operands,
the gradients against the oracle backward (block_window_backward / swiglu_bwd / head_attention_bwd,
swin.hpp:370-467), which tests/test_oracle_backward.py pins by central finite differences."""
import numpy as np
import pytest

import paper_2509_13523_b200 as swf
from oracle import pyoracle as o

pytestmark = pytest.mark.gpu

# fp32 accumulation of bf16 x bf16 products (exact in fp32) over K terms: ~sqrt(K) * 2^-24 of |C|
TOL_GEMM = 2e-4
# bf16 operands (8-bit mantissa, 2^-9 relative rounding) through the backward's chain of GEMMs, per
# parameter array relative to its max |grad| -- the same bar as the BF16 forward
TOL_GRAD_BF16 = 2e-2

TINY = dict(hidden_dim=16, n_heads=4, ffn_dim=32, n_layers=2, window_px=6, in_channels=4, out_channels=2,
            time_dim=16)
C1 = dict(hidden_dim=128, n_heads=4, ffn_dim=256, n_layers=2, window_px=8, in_channels=8, out_channels=3,
          time_dim=128)
MID = dict(hidden_dim=256, n_heads=2, ffn_dim=512, n_layers=2, window_px=12, in_channels=16, out_channels=6,
           time_dim=256)


def bf16(a):
    """Round-to-nearest-even to bf16, returned as float64."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("M,N,K", [(300, 200, 100), (1000, 384, 2048), (256, 64, 16), (129, 1000, 777), (200, 70, 96)])
@pytest.mark.parametrize("mn", [False, True])
def test_gemm_bf16_general(M, N, K, mn):
    rng = np.random.default_rng(M * 7 + N + K + mn)
    pad = lambda n: (n + 7) // 8 * 8  # noqa: E731  (16-byte operand rows)
    if mn:
        A = rng.standard_normal((K, pad(M))).astype(np.float32)
        B = rng.standard_normal((K, pad(N))).astype(np.float32)
        ref = bf16(A).T @ bf16(B)
    else:
        A = rng.standard_normal((M, pad(K))).astype(np.float32)
        B = rng.standard_normal((N, pad(K))).astype(np.float32)
        A[:, K:] = 0.0
        B[:, K:] = 0.0
        ref = bf16(A) @ bf16(B).T
    got = swf.ops.gemm_bf16(A, B, mn)
    scale = float(np.abs(ref).max())
    assert float(np.abs(got - ref).max()) <= TOL_GEMM * scale
    C0 = rng.standard_normal(ref.shape).astype(np.float32)  # accumulate: C += op(A) op(B)
    acc = swf.ops.gemm_bf16(A, B, mn, C=C0, accumulate=True)
    assert float(np.abs(acc - (C0 + ref)).max()) <= TOL_GEMM * (scale + 4.0)


@pytest.mark.parametrize("cfg,H,W", [(TINY, 12, 12), (C1, 32, 64), (MID, 24, 48)])
def test_backward_bf16_matches_oracle(cfg, H, W):
    oc, sc = o.ModelConfig(**cfg), swf.ModelConfig(**cfg)
    # weight scale 0.03: at the FP32 tests' 0.1 the MID network is chaotic -- perturbing only the input
    # by 2^-9 (one bf16 rounding) moves the f64 oracle's own gradients by up to 33% (tools/bwd_err_probe.py)
    p = o.init_params(oc, 77, random=True, scale=0.03, dtype=np.float64)
    x = o.random_field(oc.in_channels, H * W, 78)
    R = o.random_field(oc.out_channels, H * W, 79)
    gref, dref = o.backward(oc, p, x, 0.8, H, W, R)
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32)
    dn.load_params(p.astype(np.float32))
    g32, _ = dn.backward(x.astype(np.float32), 0.8, R.astype(np.float32))
    dn.set_backward_precision(swf.PREC_BF16)
    g, din = dn.backward(x.astype(np.float32), 0.8, R.astype(np.float32))
    g2, _ = dn.backward(x.astype(np.float32), 0.8, R.astype(np.float32))
    dn.close()
    assert np.array_equal(g, g2)  # deterministic (no atomics in the tensor-core path either)
    assert not np.array_equal(g, g32)  # the BF16 path ran
    off = 0
    for name, r, c in o.param_shapes(oc):
        a, b = g[off:off + r * c], gref[off:off + r * c]
        off += r * c
        scale = max(float(np.abs(b).max()), 1e-30)
        assert float(np.abs(a - b).max()) / scale <= TOL_GRAD_BF16, name
    scale = np.maximum(np.abs(dref).max(axis=0), 1e-30)
    assert float((np.abs(din - dref).max(axis=0) / scale).max()) <= TOL_GRAD_BF16


def test_backward_bf16_c2_widths_matches_fp32_mode():
    """C2 widths (h 1536, 12 heads, d 128, f 9216, 60 x 60 windows: s = 3600, 15 key tiles per GEMM with a
    partial last one, the shifted block's windows all seam-masked) on a 60 x 120 grid, 2 blocks: the BF16
    training mode (P / dS built in the tensor-core GEMMs' epilogues from the forward kernel's row
    log2-sum-exp) against the FP32 validation mode, which the tests above pin to the oracle at the
    small widths; per parameter array and for the input gradient."""
    cfg = swf.ModelConfig(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=1, blocks_per_layer=2,
                          window_px=60, in_channels=144, out_channels=70, time_dim=1536)
    H, W = 60, 120
    rng = np.random.default_rng(11)
    x = rng.standard_normal((H * W, cfg.in_channels)).astype(np.float32)
    R = rng.standard_normal((H * W, cfg.out_channels)).astype(np.float32)
    dn = swf.Denoiser(cfg, H, W, precision=swf.PREC_FP32)
    dn.init_params(2024, mode=1, scale=0.01)
    g32, d32 = dn.backward(x, 0.8, R)
    dn.set_backward_precision(swf.PREC_BF16)
    g, din = dn.backward(x, 0.8, R)
    dn.close()
    assert not np.array_equal(g, g32)  # the BF16 path ran
    off = 0
    for name, r, c in swf.param_arrays(cfg):
        a, b = g[off:off + r * c], g32[off:off + r * c]
        off += r * c
        scale = max(float(np.abs(b).max()), 1e-30)
        assert float(np.abs(a - b).max()) / scale <= TOL_GRAD_BF16, name
    assert off == g.size
    scale = np.maximum(np.abs(d32).max(axis=0), 1e-30)
    assert float((np.abs(din - d32).max(axis=0) / scale).max()) <= TOL_GRAD_BF16


def test_train_step_bf16_backward():
    """reference_train_step in the BF16 training mode (the forward's and the backward's linears on the
    tensor cores, attention / norms in FP32): losses and accumulated gradients within the BF16 bar of
    the FP32 validation mode's."""
    oc, sc = o.ModelConfig(**C1), swf.ModelConfig(**C1)
    H, W = 32, 64
    p = o.init_params(oc, 57, random=True, scale=0.03, dtype=np.float32)
    data = swf.DataSet(*[[o.random_field(c, H * W, 900 + 3 * i + j).astype(np.float32) for i in range(3)]
                         for j, c in ((0, 3), (1, 2), (2, 3))])
    w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
    res = {}
    for prec in (swf.PREC_FP32, swf.PREC_BF16):
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32)
        dn.load_params(p)
        dn.set_backward_precision(prec)
        res[prec] = dn.train_step(data, 3, 2, 2, w, swf.DiffusionConfig(), 31)
        dn.close()
    a, b = res[swf.PREC_FP32], res[swf.PREC_BF16]
    assert np.allclose(a.mb_losses, b.mb_losses, rtol=TOL_GRAD_BF16, atol=0)
    assert not np.array_equal(a.mb_losses, b.mb_losses)  # the forward's linears ran in BF16
    off = 0
    for name, r, c in o.param_shapes(oc):
        x, y = a.grads[off:off + r * c], b.grads[off:off + r * c]
        off += r * c
        assert float(np.abs(x - y).max()) <= TOL_GRAD_BF16 * max(float(np.abs(x).max()), 1e-30), name


def test_train_step_bf16_wp_group_matches_single():
    """The BF16 training mode on a window-parallel group (WP 1x2, one process, ranks on devices
    [0, 1 % n]): per-rank partial gradients over their own windows, summed by the group, equal the
    single-device BF16 training mode's within fp32 summation-order noise; losses identical."""
    import torch
    oc, sc = o.ModelConfig(**C1), swf.ModelConfig(**C1)
    H, W = 32, 64
    p = o.init_params(oc, 58, random=True, scale=0.03, dtype=np.float32)
    data = swf.DataSet(*[[o.random_field(c, H * W, 700 + 3 * i + j).astype(np.float32) for i in range(3)]
                         for j, c in ((0, 3), (1, 2), (2, 3))])
    w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
    n = max(1, torch.cuda.device_count())
    res = {}
    for grp in (False, True):
        kw = dict(topology=(1, 2, 1, swf.OWN_CONTIGUOUS), devices=[0, 1 % n]) if grp else {}
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32, **kw)
        dn.load_params(p)
        dn.set_backward_precision(swf.PREC_BF16)
        res[grp] = dn.train_step(data, 3, 2, 2, w, swf.DiffusionConfig(), 31)
        dn.close()
    a, b = res[False], res[True]
    assert np.allclose(a.mb_losses, b.mb_losses, rtol=1e-5, atol=0)
    assert float(np.abs(a.grads - b.grads).max()) <= 1e-3 * float(np.abs(a.grads).max())


def test_backward_precision_config_errors():
    cfg = dict(TINY, hidden_dim=12, n_heads=3, ffn_dim=24)  # rows of 12 bf16 = 24 B: not 16-byte aligned
    dn = swf.Denoiser(swf.ModelConfig(**cfg), 12, 12, precision=swf.PREC_FP32)
    with pytest.raises(swf.ConfigError):
        dn.set_backward_precision(swf.PREC_BF16)
    with pytest.raises(swf.ConfigError):
        dn.set_backward_precision(7)
    dn.close()
