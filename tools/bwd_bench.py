"""Backward timing, FP32 validation mode vs BF16 tensor-core linears (swf_set_backward_precision):
C2 widths (h 1536, 12 heads, f 9216, w 60) on a reduced grid, 2 blocks; prints ms per backward call.
usage: python tools/bwd_bench.py [H W reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2509_13523_b200 as swf  # noqa: E402

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (120, 240)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = swf.ModelConfig(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=1, blocks_per_layer=2, window_px=60,
                      in_channels=144, out_channels=70, time_dim=1536)
rng = np.random.default_rng(5)
x = rng.standard_normal((H * W, cfg.in_channels)).astype(np.float32)
R = rng.standard_normal((H * W, cfg.out_channels)).astype(np.float32)
dn = swf.Denoiser(cfg, H, W, precision=swf.PREC_FP32)
dn.init_params(2024, mode=1, scale=0.01)
res = {}
for name, prec in (("fp32", swf.PREC_FP32), ("bf16_tc", swf.PREC_BF16)):
    dn.set_backward_precision(prec)
    g, _ = dn.backward(x, 0.8, R)  # warm-up (allocations)
    t0 = time.perf_counter()
    for _ in range(reps):
        g, _ = dn.backward(x, 0.8, R)
    ms = (time.perf_counter() - t0) / reps * 1e3
    res[name] = (ms, g)
    print(f"{name}: {ms:.1f} ms per backward (forward with saved activations + backward, {H}x{W}, 2 blocks)", flush=True)
a, b = res["fp32"][1], res["bf16_tc"][1]
print(f"max |g_bf16 - g_fp32| / max |g_fp32| = {float(np.abs(a - b).max() / np.abs(a).max()):.3e}")
print(f"speed-up {res['fp32'][0] / res['bf16_tc'][0]:.2f}x")
