"""Kernel isolation benchmark at the C2 shape: one forward, then each kernel class replayed
back-to-back (steady clocks) with nvidia-smi clocks sampled; prints ms and TFLOP/s per class."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_13523_b200 as swf  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
classes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["attention", "qkv_gemm", "out_gemm", "gateup_gemm",
                                                             "down_gemm", "rms_adaln"]
cfg = swf.ModelConfig(**bench.CFG)
dn = swf.Denoiser(cfg, bench.H, bench.W, precision=swf.PREC_BF16)
dn.init_params(bench.SEED, mode=1, scale=bench.WEIGHT_SCALE)
x = bench.synthetic_input(dn, bench.CFG)
d_in = torch.from_numpy(x).cuda()
d_out = torch.empty(bench.H * bench.W * bench.CFG["out_channels"], device="cuda")
try:
    dn.forward_device(d_in.data_ptr(), bench.T_STEP, d_out.data_ptr())
    dn.sync()
except swf.NumericsError as e:  # development builds that skip work (e.g. SWF_ATTN_NOSOFTMAX)
    print("forward:", e, flush=True)
M = dn.local_tokens()
cf = bench.class_flops(bench.CFG, M)
res = {}
try:  # board energy counter (mJ): under the 1 kW cap, energy per launch decides the clock
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
    energy_mj = lambda: pynvml.nvmlDeviceGetTotalEnergyConsumption(_h)  # noqa: E731
except Exception:
    energy_mj = None
for k in classes:
    e0 = energy_mj() if energy_mj else None
    with bench.ClockSampler(0) as clk:
        ms = dn.bench_kernel(k, block=1, reps=reps)
    e1 = energy_mj() if energy_mj else None
    res[k] = {"ms": ms, "tflops": cf[k] / (ms / 1e3) / 1e12 if k in cf else None, "clocks": clk.summary()}
    if e0 is not None:
        res[k]["J_per_launch"] = (e1 - e0) / 1e3 / reps  # includes the untimed warm-up launch share
    if k == "rms_adaln":
        res[k]["GBps"] = M * bench.CFG["hidden_dim"] * 6 / (ms / 1e3) / 1e9
    print(k, json.dumps(res[k]), flush=True)
