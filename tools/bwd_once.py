"""One BF16-training-mode backward at C2 widths on a reduced grid (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2509_13523_b200 as swf  # noqa: E402

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (120, 240)
cfg = swf.ModelConfig(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=1, blocks_per_layer=2, window_px=60,
                      in_channels=144, out_channels=70, time_dim=1536)
rng = np.random.default_rng(5)
x = rng.standard_normal((H * W, cfg.in_channels)).astype(np.float32)
R = rng.standard_normal((H * W, cfg.out_channels)).astype(np.float32)
dn = swf.Denoiser(cfg, H, W, precision=swf.PREC_FP32)
dn.init_params(2024, mode=1, scale=0.01)
dn.set_backward_precision(swf.PREC_BF16)
g, _ = dn.backward(x, 0.8, R)
print("ok", float(np.abs(g).max()))
