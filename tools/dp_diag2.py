"""WP=2 training diagnostics with one process per rank: the partial losses of microbatch sid=3 (summed over
the ranks) repeated, the diffusion_loss_sample with a given z, and the plain forward, vs one process."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
d = dict(hidden_dim=64, n_heads=4, ffn_dim=128, n_layers=2, window_px=8, in_channels=8, out_channels=3, time_dim=64)
H, W = 32, 64
oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
p = o.init_params(oc, 57, random=True, scale=0.05, dtype=np.float32)
xs = [o.random_field(c, H * W, 900 + j).astype(np.float32) for j, c in ((0, 3), (1, 2), (2, 3))]
z = o.random_field(3, H * W, 77).astype(np.float32)
w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
dc = swf.DiffusionConfig()
dn = swf.Denoiser(sc, H, W, device=0, precision=swf.PREC_FP32, topology=(1, 2, 1, rank, swf.OWN_CONTIGUOUS))
dn.load_params(p)
dn.connect_peers_torch(dist)


def allsum(v):
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


res = {}
res["acc"] = [allsum(dn.train_accumulate(xs[0], xs[2], xs[1], w, dc, 31, 3)) for _ in range(3)]
res["loss_z"] = [allsum(dn.diffusion_loss_sample(xs[0], xs[2], xs[1], w, dc, 4242, z, want_grads=False)[0]) for _ in range(2)]
res["loss_zg"] = [allsum(dn.diffusion_loss_sample(xs[0], xs[2], xs[1], w, dc, 4242, z, want_grads=True)[0]) for _ in range(2)]
x = o.random_field(8, H * W, 5).astype(np.float32)
y = dn.forward(x, 0.9)
owned = np.zeros(H * W, np.int64)
swf.lib().swf_owned_pixels(dn._c, owned.ctypes.data_as(swf.C.c_void_p))
parts = [None] * world
dist.all_gather_object(parts, (owned[:dn.local_tokens()], y[owned[:dn.local_tokens()]]))
if rank == 0:
    one = swf.Denoiser(sc, H, W, device=0, precision=swf.PREC_FP32)
    one.load_params(p)
    ref = {"acc": one.train_accumulate(xs[0], xs[2], xs[1], w, dc, 31, 3),
           "loss_z": one.diffusion_loss_sample(xs[0], xs[2], xs[1], w, dc, 4242, z, want_grads=False)[0],
           "loss_zg": one.diffusion_loss_sample(xs[0], xs[2], xs[1], w, dc, 4242, z, want_grads=True)[0]}
    y1 = one.forward(x, 0.9)
    yw = np.zeros_like(y1)
    for pix, vals in parts:
        yw[pix] = vals
    for k in res:
        print(f"{k}: wp2={res[k]} single={ref[k]}", flush=True)
    print(f"forward bitwise={np.array_equal(yw, y1)} maxdiff={np.abs(yw - y1).max():.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
