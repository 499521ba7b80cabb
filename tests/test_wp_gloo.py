"""world_size-2 gloo run of the multi-rank host logic (no GPU): every rank derives the same
ownership / exchange plan, the owned windows of all ranks partition the grid, and the IPC-handle
blob exchange used by Denoiser.connect_peers_torch round-trips through all_gather_object."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import paper_2509_13523_b200 as swf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    owners = swf.plan_owners(720, 1440, 60, 1, world, swf.OWN_CONTIGUOUS)
    mine = np.nonzero(owners == rank)[0]
    sent = swf.plan_exchange(720, 1440, 60, 1, world)
    blob = bytes([rank]) * 192  # stands in for the 3 cudaIpcMemHandle_t of this rank
    allh = [None] * world
    dist.all_gather_object(allh, blob)
    got = [None] * world
    dist.all_gather_object(got, (mine.tolist(), sent.tolist()))
    if rank == 0:
        q.put((b"".join(allh), got))
    dist.destroy_process_group()


def test_two_rank_plan_agreement():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    blob, got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert blob == bytes([0]) * 192 + bytes([1]) * 192
    windows = sorted(got[0][0] + got[1][0])
    assert windows == list(range(288))
    assert got[0][1] == got[1][1]
