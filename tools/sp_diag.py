"""SP=2 single-process group diagnostics (two ranks, devices [0, 0 or 1]): times each call and prints
the error on failure. Usage: SWF_ATTN=split|default python tools/sp_diag.py <cfg>"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

cfgs = {
    "MID": (dict(hidden_dim=256, n_heads=2, ffn_dim=512, n_layers=3, window_px=12, in_channels=16, out_channels=6,
                 time_dim=256), 48, 96),
    "C4W": (dict(hidden_dim=6144, n_heads=48, ffn_dim=6144, n_layers=2, window_px=12, in_channels=16, out_channels=6,
                 time_dim=128), 12, 24),
    "C4W1": (dict(hidden_dim=6144, n_heads=48, ffn_dim=6144, n_layers=1, window_px=12, in_channels=16,
                  out_channels=6, time_dim=128), 12, 24),
    "H1K": (dict(hidden_dim=1024, n_heads=8, ffn_dim=1024, n_layers=2, window_px=12, in_channels=16, out_channels=6,
                 time_dim=128), 12, 24),
}
name = sys.argv[1]
d, H, W = cfgs[name]
sc = swf.ModelConfig(**d)
x = o.random_field(16, H * W, 9).astype(np.float32)
how = sys.argv[2] if len(sys.argv) > 2 else "init"
topo = {"sp2": (1, 1, 2, swf.OWN_CONTIGUOUS), "wp2": (1, 2, 1, swf.OWN_CONTIGUOUS)}[sys.argv[3] if len(sys.argv) > 3 else "sp2"]
for devs in ([0, 0],):
    t0 = time.time()
    dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16, topology=topo, devices=devs)
    if how == "init":
        dn.init_params(2024, mode=1, scale=0.004)
    else:
        dn.load_params(o.init_params(o.ModelConfig(**d), 2024, random=True, scale=0.004, dtype=np.float32))
    print(f"{name} {how} {topo} attn={os.environ.get('SWF_ATTN', 'default')} params {time.time() - t0:.1f}s",
          flush=True)
    try:
        t0 = time.time()
        y = dn.forward(x, 0.9)
        print(f"  forward ok {time.time() - t0:.2f}s finite={np.isfinite(y).all()}", flush=True)
    except Exception as e:
        print(f"  forward FAILED after {time.time() - t0:.1f}s: {e}", flush=True)
    dn.close()
