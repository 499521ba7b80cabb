"""Data-parallel training step on N GPUs (launch with torchrun; NCCL): each rank runs its replica's
microbatches on its own GPU (FP32 validation mode), the device gradient accumulators are summed by
one in-place NCCL all-reduce, and the result must equal the single-rank reference_train_step
(simulator.hpp:50-86) with dp = N replicas run in order on rank 0 (fp32 summation order differs:
relative 1e-6), with identical per-microbatch losses."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
d = dict(hidden_dim=64, n_heads=4, ffn_dim=128, n_layers=2, window_px=8, in_channels=8, out_channels=3, time_dim=64)
H, W, gas = 32, 64, 2
oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
p = o.init_params(oc, 57, random=True, scale=0.05, dtype=np.float32)
data = swf.DataSet(*[[o.random_field(c, H * W, 900 + 3 * i + j).astype(np.float32) for i in range(5)]
                     for j, c in ((0, 3), (1, 2), (2, 3))])
w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
dc = swf.DiffusionConfig()
dn = swf.Denoiser(sc, H, W, device=local, precision=swf.PREC_FP32)
dn.load_params(p)
print(f"rank {rank}: replica ready", flush=True)
res = dn.train_step(data, 3, world, gas, w, dc, 31, group=dist.group.WORLD)
print(f"rank {rank}: train_step done", flush=True)
ok = True
if rank == 0:
    single = swf.Denoiser(sc, H, W, device=local, precision=swf.PREC_FP32)
    single.load_params(p)
    ref = single.train_step(data, 3, world, gas, w, dc, 31)
    rel = float(np.abs(res.grads - ref.grads).max() / np.abs(ref.grads).max())
    same_mb = res.mb_losses == ref.mb_losses
    print(f"world={world} gas={gas} loss={res.loss:.6e} ref={ref.loss:.6e} mb_losses_equal={same_mb} "
          f"grad_rel_err={rel:.3e}", flush=True)
    ok = same_mb and abs(res.loss - ref.loss) <= 1e-12 * abs(ref.loss) and rel <= 1e-6
dist.barrier()
if rank == 0:
    print("DP_CHECK", "PASS" if ok else "FAIL", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
