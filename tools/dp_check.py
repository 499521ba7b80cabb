"""Sharded training step on N GPUs (launch with torchrun; NCCL), FP32 validation mode. SWF_DP_WP=k
(default 1) ranks share each replica's windows (window parallelism: partial losses / gradients over
their own tokens, the layout changes of the backward stored into peers over NVLink); N / k replicas
are data parallel. One in-place NCCL all-reduce of the device gradient accumulators sums both. The
result must equal the single-GPU reference_train_step (simulator.hpp:50-86) with dp = N / k
replicas run in order on rank 0: per-microbatch losses bitwise without WP (1e-12 relative with WP:
partial sums), gradients within 1e-6 relative (fp32 summation order)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
if torch.cuda.device_count() >= world:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
else:  # ranks share GPUs (NCCL rejects duplicate devices): gloo all-reduce through host memory
    dist.init_process_group("gloo")
d = dict(hidden_dim=64, n_heads=4, ffn_dim=128, n_layers=2, window_px=8, in_channels=8, out_channels=3, time_dim=64)
H, W, gas = 32, 64, 2
oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
p = o.init_params(oc, 57, random=True, scale=0.05, dtype=np.float32)
data = swf.DataSet(*[[o.random_field(c, H * W, 900 + 3 * i + j).astype(np.float32) for i in range(5)]
                     for j, c in ((0, 3), (1, 2), (2, 3))])
w = swf.LossWeights.make(H, [1.0, 0.6, 1.7])
dc = swf.DiffusionConfig()
wp = int(os.environ.get("SWF_DP_WP", 1))
dp = world // wp
topo = None
if wp > 1:
    groups = [dist.new_group(list(range(r * wp, (r + 1) * wp))) for r in range(dp)]
    wa, wb = {2: (1, 2), 4: (2, 2)}[wp]
    topo = (wa, wb, 1, rank % wp, swf.OWN_CONTIGUOUS)
dn = swf.Denoiser(sc, H, W, device=local, precision=swf.PREC_FP32, topology=topo)
dn.load_params(p)
if wp > 1:
    dn.connect_peers_torch(dist, group=groups[rank // wp])
print(f"rank {rank}: replica {rank // wp} ready", flush=True)
res = dn.train_step(data, 3, dp, gas, w, dc, 31, group=dist.group.WORLD)
print(f"rank {rank}: train_step done", flush=True)
ok = True
if rank == 0:
    single = swf.Denoiser(sc, H, W, device=local, precision=swf.PREC_FP32)
    single.load_params(p)
    ref = single.train_step(data, 3, dp, gas, w, dc, 31)
    rel = float(np.abs(res.grads - ref.grads).max() / np.abs(ref.grads).max())
    mb_rel = float(np.max(np.abs(np.array(res.mb_losses) - np.array(ref.mb_losses)) / np.abs(ref.mb_losses)))
    print(f"mb_losses sharded={[round(v, 9) for v in res.mb_losses]} single={[round(v, 9) for v in ref.mb_losses]}",
          flush=True)
    print(f"world={world} wp={wp} dp={dp} gas={gas} loss={res.loss:.9e} ref={ref.loss:.9e} "
          f"mb_loss_rel_err={mb_rel:.3e} grad_rel_err={rel:.3e}", flush=True)
    ok = mb_rel <= (0.0 if wp == 1 else 1e-6) and abs(res.loss - ref.loss) <= 1e-6 * abs(ref.loss) and rel <= 1e-5
dist.barrier()
if rank == 0:
    print("DP_CHECK", "PASS" if ok else "FAIL", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
