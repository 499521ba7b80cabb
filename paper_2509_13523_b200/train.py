"""Training step over the device loss / backward.

`train_step` restates `reference_train_step` (simulator.hpp:50-86) -- microbatches sample_id =
first_sample + d * gas + g, pair index sample_id % n_pairs, per-sample noise and diffusion time from
the shared-seed protocol (rng.hpp:72-80), gradients summed then scaled by 1 / (dp * gas) -- with the
data-parallel dimension mapped onto ranks: with a `torch.distributed` group of size dp x wp, the
wp consecutive ranks of replica d run its `gas` microbatches window-parallel (each rank's loss and
gradients are partial sums over its own tokens, the engine's WP topology) into the device gradient
accumulators, and one in-place all-reduce over the group (NCCL on the device buffer; gloo through
host memory) sums the WP partials and the replicas at once -- the roles of the intra-instance
gradient sum and of `grad_allreduce` (simulator.hpp:92-120, 169-202). With group=None (or a group of size 1) one rank
runs all dp replicas in order, which is the reference's single-rank semantics.

The engine is a `Denoiser` (FP32 validation mode) or anything with the same four methods:
`train_reset()`, `train_accumulate(x_prev, x0, forcings, w, dc, run_seed, sample_id) -> loss`,
`train_grads_device() -> (ptr, n) | None` (FP32 device buffer) and `train_read(scale) -> np.ndarray`.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np


def latitude_weights(H: int) -> np.ndarray:
    """latitude_weights (grid.hpp:74-82): cos of each row centre's latitude, unit mean."""
    d = 180.0 / H
    w = np.cos((90.0 - d * (np.arange(H) + 0.5)) * np.pi / 180.0)
    return w * (H / w.sum())


@dataclass
class LossWeights:
    """LossWeights (grid.hpp:76-96): per-row latitude weights and per-variable weights."""
    alpha_row: np.ndarray
    kappa: np.ndarray

    @staticmethod
    def make(H: int, kappa) -> "LossWeights":
        k = np.asarray(kappa, np.float64)
        if not np.all(k > 0):
            raise ValueError("loss weights: kappa must be positive")
        return LossWeights(latitude_weights(H), k)

    @staticmethod
    def uniform(H: int, channels: int) -> "LossWeights":
        return LossWeights(np.ones(H), np.ones(channels))


@dataclass
class DataSet:
    """DataSet (simulator.hpp:30-38): standardized states, forcings and residual targets, [N][C] each."""
    states: list
    forcings: list
    residuals: list

    def n_pairs(self) -> int:
        return len(self.residuals)

    def pair_of_sample(self, sample_id: int) -> int:
        return int(sample_id % self.n_pairs())


@dataclass
class TrainStepResult:
    """TrainStepResult (simulator.hpp:40-45)."""
    loss: float = 0.0
    grads: np.ndarray | None = None
    mb_losses: list = field(default_factory=list)


def _log(msg):
    if os.environ.get("SWF_TRAIN_VERBOSE"):
        print(msg, flush=True)


def _world(group):
    """group=None: no data-parallel sharding (one rank runs every replica)."""
    if group is None:
        return None, 1, 0
    import torch.distributed as dist
    return dist, dist.get_world_size(group), dist.get_rank(group)


class _DeviceView:
    """__cuda_array_interface__ over the engine's FP32 gradient accumulator (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _allreduce_grads(engine, dist, group):
    """Sum the replicas' accumulators. NCCL: in place on the device buffer (returns None);
    otherwise through host memory (returns the summed host copy)."""
    import torch
    dev = engine.train_grads_device() if dist.get_backend(group) == "nccl" else None
    if dev is not None:
        ptr, n = dev
        t = torch.as_tensor(_DeviceView(ptr, n), device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t, group=group)
        torch.cuda.synchronize()
        return None
    host = torch.from_numpy(np.ascontiguousarray(engine.train_read(1.0), np.float32))
    dist.all_reduce(host, group=group)
    return host.numpy()


def train_step(engine, data: DataSet, first_sample: int, dp: int, gas: int, w: LossWeights, dc, run_seed: int,
               group=None) -> TrainStepResult:
    """reference_train_step (simulator.hpp:50-86) with replicas on ranks; see the module docstring."""
    if data.n_pairs() <= 0:
        raise ValueError("train_step: empty dataset")
    if dp < 1 or gas < 1:
        raise ValueError("train_step: dp and gas must be >= 1")
    dist, world, rank = _world(group)
    wp = int(getattr(engine, "wp_world", 1))  # ranks sharing one replica's windows
    sharded = world > 1
    if wp > 1 and not sharded:
        raise ValueError("train_step: a window-parallel engine needs the process group")
    if sharded and world != dp * wp:
        raise ValueError(f"train_step: group size {world} must equal dp={dp} x window-parallel ranks {wp}")
    if wp > 1 and getattr(engine, "wp_rank", rank % wp) != rank % wp:
        raise ValueError("train_step: window-parallel ranks of a replica must be consecutive group ranks")
    replicas = [rank // wp] if sharded else list(range(dp))
    engine.train_reset()
    mb = np.zeros(dp * gas, np.float64)
    for d in replicas:
        for g in range(gas):
            sid = first_sample + d * gas + g
            idx = data.pair_of_sample(sid)
            mb[d * gas + g] = engine.train_accumulate(data.states[idx], data.residuals[idx], data.forcings[idx], w,
                                                      dc, run_seed, sid)
    reduced = None
    if sharded:
        import torch
        _log(f"rank {rank}: microbatches done, all-reduce")
        reduced = _allreduce_grads(engine, dist, group)
        _log(f"rank {rank}: gradients reduced")
        lt = torch.from_numpy(mb)
        if dist.get_backend(group) == "nccl":
            lt = lt.cuda()
        dist.all_reduce(lt, group=group)  # slot d*gas+g: the partial losses of replica d's WP ranks
        mb = lt.cpu().numpy()
    scale = 1.0 / (dp * gas)
    res = TrainStepResult()
    res.grads = engine.train_read(scale) if reduced is None else reduced.astype(np.float64) * scale
    res.mb_losses = [float(v) for v in mb]
    res.loss = float(mb.sum()) * scale
    return res
