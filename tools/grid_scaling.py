"""Member batching proxy (f1): C2 model forward on the 720x1440 grid and on a 1440x1440 grid (twice the
tokens, i.e. two ensemble members batched along M). Device time per forward (CUDA events on the context
stream, 3 warm-up + 5 timed) and pixels/s; equal pixels/s means batching members along M cannot speed
the ensemble up (one member already fills the GPU)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_13523_b200 as swf  # noqa: E402

out = {}
for H, W in ((720, 1440), (1440, 1440)):
    dn = swf.Denoiser(swf.ModelConfig(**bench.CFG), H, W, precision=swf.PREC_BF16)
    dn.init_params(bench.SEED, mode=1, scale=bench.WEIGHT_SCALE)
    x = torch.randn(H * W * bench.CFG["in_channels"], device="cuda") * 0.5
    y = torch.empty(H * W * bench.CFG["out_channels"], device="cuda")
    st = torch.cuda.ExternalStream(dn.stream)
    for _ in range(3):
        dn.forward_device(x.data_ptr(), bench.T_STEP, y.data_ptr())
    dn.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(0) as clk:
        e0.record(st)
        for _ in range(5):
            dn.forward_device(x.data_ptr(), bench.T_STEP, y.data_ptr())
        e1.record(st)
        e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[f"{H}x{W}"] = {"ms_per_forward": ms, "pixels_per_s": H * W / (ms / 1e3), "clocks": clk.summary()}
    print(json.dumps({f"{H}x{W}": out[f"{H}x{W}"]}), flush=True)
    dn.close()
    del x, y
    torch.cuda.empty_cache()
r = out["1440x1440"]["pixels_per_s"] / out["720x1440"]["pixels_per_s"]
print(json.dumps({"throughput_ratio_2x_tokens": r}))
