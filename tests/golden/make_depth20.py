"""Generates tests/golden/depth20_c2w_60x120.npz: the oracle forward (float32 restatement of
swin.hpp:327-368) of the 1.3B-width 20-block model (h=1536, 12 heads, ffn 9216, w=60, C_in=144,
C_out=70) with init_parameters_random(seed=2024, scale=0.01) on a 60x120 grid (one window row, two
windows; blocks alternate shift 0 / 30, the shifted windows seam-masked), input random_field(144,
7200, key=2025), t = 0.7. The GPU test regenerates the same weights on the device
(swf_init_params mode 1) and compares. Run: python tests/golden/make_depth20.py (~5-10 min CPU)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as o  # noqa: E402

CFG = dict(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=20, blocks_per_layer=1, window_px=60,
           in_channels=144, out_channels=70, time_dim=1536)
H, W, SEED, SCALE, XKEY, T = 60, 120, 2024, 0.01, 2025, 0.7

if __name__ == "__main__":
    oc = o.ModelConfig(**CFG)
    t0 = time.time()
    p = o.init_params(oc, SEED, random=True, scale=SCALE, dtype=np.float32)
    x = o.random_field(144, H * W, XKEY).astype(np.float32)
    print(f"params {p.size} in {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    y = o.forward(oc, p, x, np.float32(T), H, W)
    print(f"forward in {time.time() - t0:.1f}s rms(y)={np.sqrt((y ** 2).mean()):.4f}", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "depth20_c2w_60x120.npz"),
                        y=y, cfg=np.array(list(CFG.values())),
                        meta=np.array([H, W, SEED, XKEY]), scale=SCALE, t=T)
