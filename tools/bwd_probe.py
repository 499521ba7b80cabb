import numpy as np, sys
sys.path.insert(0, '.')
import paper_2509_13523_b200 as swf
from oracle import pyoracle as o
from tests.test_gpu_parity import MID, cfgs
oc, sc = cfgs(MID)
H, W = 24, 48
p = o.init_params(oc, 77, random=True, scale=0.1, dtype=np.float64)
x = o.random_field(oc.in_channels, H * W, 78); R = o.random_field(oc.out_channels, H * W, 79)
gref, dref = o.backward(oc, p, x, 0.8, H, W, R)
g32, d32 = o.backward(oc, p.astype(np.float32), x.astype(np.float32), np.float32(0.8), H, W, R.astype(np.float32))
dn = swf.Denoiser(sc, H, W, precision=swf.PREC_FP32); dn.load_params(p.astype(np.float32))
g, din = dn.backward(x.astype(np.float32), 0.8, R.astype(np.float32))
off = 0
for name, r, c in o.param_shapes(oc):
    a, b, f = g[off:off+r*c], gref[off:off+r*c], g32[off:off+r*c]; off += r*c
    s = max(np.abs(b).max(), 1e-30)
    print(f"{name:22s} gpu {np.abs(a-b).max()/s:.2e}  orc32 {np.abs(f-b).max()/s:.2e}  gpu-vs-orc32 {np.abs(a-f).max()/s:.2e}")
