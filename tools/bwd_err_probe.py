"""Per-array error of the BF16 training mode's gradients against the f64 oracle (development probe):
worst arrays and the input-gradient error per config. usage: python tools/bwd_err_probe.py [scale]"""
import numpy as np, sys
sys.path.insert(0, '.')
import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.test_gpu_bwd_tc import TINY, C1, MID
for cfg, H, W in [(TINY, 12, 12), (C1, 32, 64), (MID, 24, 48)]:
    oc, sc = o.ModelConfig(**cfg), swf.ModelConfig(**cfg)
    p = o.init_params(oc, 77, random=True, scale=float(sys.argv[1]) if len(sys.argv) > 1 else 0.03, dtype=np.float64)
    x = o.random_field(oc.in_channels, H * W, 78)
    R = o.random_field(oc.out_channels, H * W, 79)
    gref, dref = o.backward(oc, p, x, 0.8, H, W, R)
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32)
    dn.load_params(p.astype(np.float32))
    dn.set_backward_precision(swf.PREC_BF16)
    g, din = dn.backward(x.astype(np.float32), 0.8, R.astype(np.float32))
    off = 0; errs = []
    for name, r, c in o.param_shapes(oc):
        a, b = g[off:off + r * c], gref[off:off + r * c]; off += r * c
        errs.append((float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-30), name))
    errs.sort(reverse=True)
    scale = np.maximum(np.abs(dref).max(axis=0), 1e-30)
    print(cfg['hidden_dim'], 'worst', [f"{n}:{e:.2e}" for e, n in errs[:6]], 'din', float((np.abs(din - dref).max(axis=0) / scale).max()))
