"""Two processes on one GPU (gloo): every rank computes the same microbatch losses of the FP32 training
path; prints them per rank (SWF_DIAG_SERIAL=1: the ranks take turns)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(0)
if world > 1:
    dist.init_process_group("gloo")
d = dict(hidden_dim=64, n_heads=4, ffn_dim=128, n_layers=2, window_px=8, in_channels=8, out_channels=3, time_dim=64)
H, W = 32, 64
oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
p = o.init_params(oc, 57, random=True, scale=0.05, dtype=np.float32)
data = [[o.random_field(c, H * W, 900 + 3 * i + j).astype(np.float32) for i in range(5)] for j, c in ((0, 3), (1, 2), (2, 3))]
w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
serial = os.environ.get("SWF_DIAG_SERIAL") == "1"
for turn in range(world if serial else 1):
    if serial and turn != rank:
        dist.barrier()
        continue
    dn = swf.Denoiser(sc, H, W, device=0, precision=swf.PREC_FP32)
    dn.load_params(p)
    dn.train_reset()
    losses = []
    for sid in range(3, 7):
        i = sid % 5
        losses.append(dn.train_accumulate(data[0][i], data[2][i], data[1][i], w, swf.DiffusionConfig(), 31, sid))
    g = dn.train_read(1.0)
    print(f"rank {rank} serial={serial} losses={['%.12f' % v for v in losses]} gsum={float(np.abs(g).sum()):.9e}",
          flush=True)
    if serial:
        dist.barrier()
if world > 1:
    dist.destroy_process_group()
