"""HBM-bound kernels of the C2 sampler / forward path (for ncu): one forecast_step (1 solver step = 2
denoiser evaluations, churn on) through the C-ABI host-buffer call on the 720x1440 grid, after one
warm-up call. Run under ncu with the metrics gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum and a kernel filter for the elementwise / gather kernels (tools/gpurun/gpu_hbm.sh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_13523_b200 as swf  # noqa: E402

cfg = swf.ModelConfig(**bench.CFG)
dn = swf.Denoiser(cfg, bench.H, bench.W, precision=swf.PREC_BF16)
dn.init_params(bench.SEED, mode=1, scale=bench.WEIGHT_SCALE)
rng = np.random.default_rng(1)
x0 = rng.standard_normal((bench.H * bench.W, 70), dtype=np.float32)
fo = rng.standard_normal((bench.H * bench.W, 4), dtype=np.float32)
dc = swf.DiffusionConfig(solver_steps=2, churn=0.5)
for k in range(2):
    y = dn.forecast_step(x0, fo, dc, 7, 100 + k)
print("hbm_probe ok", float(np.abs(y).mean()))
