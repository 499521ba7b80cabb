"""Sampler CUDA-graph A/B: wall time per forecast_step (10 solver steps = 20 denoiser evaluations)
with the eager launch sequence vs the captured graph, on small grids where launch overhead shows.
usage: python tools/graph_ab.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402

CFGS = [("C1 32x64 d128 2 blocks", dict(hidden_dim=128, n_heads=4, ffn_dim=256, n_layers=2, window_px=8,
                                        in_channels=8, out_channels=3, time_dim=128), 32, 64),
        ("72x144 d512 8 blocks w36", dict(hidden_dim=512, n_heads=4, ffn_dim=1024, n_layers=8, window_px=36,
                                          in_channels=8, out_channels=3, time_dim=256), 72, 144)]
for name, d, H, W in CFGS:
    sc = swf.ModelConfig(**d)
    rng = np.random.default_rng(0)
    x0 = rng.standard_normal((H * W, 3)).astype(np.float32)
    fo = rng.standard_normal((H * W, 2)).astype(np.float32)
    dc = swf.DiffusionConfig(solver_steps=10)
    res = {}
    for graphs in (False, True):
        dn = swf.Denoiser(sc, H, W, precision=swf.PREC_BF16)
        dn.init_params(7, mode=1, scale=0.02)
        dn.set_graphs(graphs)
        for k in range(3):
            dn.forecast_step(x0, fo, dc, 1, k)
        n = 20
        t0 = time.perf_counter()
        for k in range(n):
            y = dn.forecast_step(x0, fo, dc, 1, 100 + k)
        res[graphs] = (time.perf_counter() - t0) / n * 1e3
        launches = dn.kernel_launches()
        dn.close()
    print(f"{name}: eager {res[False]:.3f} ms/forecast_step, graph {res[True]:.3f} ms "
          f"({res[False] / res[True]:.2f}x), 20 evals each", flush=True)
