"""Window-parallel correctness on N GPUs (launch with torchrun): the WP forward must equal the
single-GPU forward BITWISE (ownership only permutes independent rows/windows; the GEMM K-loop
order does not depend on M), and both must match the oracle at the BF16 tolerance."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from oracle import pyoracle as o  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
# more ranks than GPUs (e.g. 8 ranks on a 4-GPU box) shares devices: a functional check of the
# 8-way topology (peer stores and barriers between processes on one device), not a timing
local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
sp = int(os.environ.get("SWF_SP", 1))
wp = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}[world // sp]
own = int(os.environ.get("SWF_OWN", swf.OWN_CONTIGUOUS))
prec = swf.PREC_FP32 if os.environ.get("SWF_PREC") == "fp32" else swf.PREC_BF16
ok = True
for name, d, H, W in [
    ("C1", dict(hidden_dim=128, n_heads=4, ffn_dim=256, n_layers=2, window_px=8, in_channels=8, out_channels=3,
                time_dim=128), 32, 64),
    ("MID", dict(hidden_dim=256, n_heads=2, ffn_dim=512, n_layers=3, window_px=12, in_channels=16, out_channels=6,
                 time_dim=256), 48, 96),
    ("MID4", dict(hidden_dim=512, n_heads=4, ffn_dim=1024, n_layers=2, window_px=12, in_channels=16, out_channels=6,
                  time_dim=256), 48, 96),
]:
    if d["n_heads"] % sp or d["window_px"] % sp:
        continue
    oc, sc = o.ModelConfig(**d), swf.ModelConfig(**d)
    p = o.init_params(oc, 7, random=True, scale=0.03, dtype=np.float32)
    x = o.random_field(oc.in_channels, H * W, 8).astype(np.float32)
    if prec == swf.PREC_FP32 and sp > 1:
        continue
    dn = swf.Denoiser(sc, H, W, device=local, precision=prec, topology=(wp[0], wp[1], sp, rank, own))
    dn.load_params(p)
    dn.connect_peers_torch(dist)
    if name == "C1":  # f4: per-rank chunked input loading == host-array inputs, partial reads
        import tempfile
        tmp = os.path.join(tempfile.gettempdir(), f"swf_wp_chunked_{os.getpid() if world == 1 else 'job'}")
        if rank == 0:
            os.makedirs(tmp, exist_ok=True)
            x0 = o.random_field(3, H * W, 301).astype(np.float32)
            fo = o.random_field(2, H * W, 302).astype(np.float32)
            swf.write_chunked(os.path.join(tmp, "s.chk"), x0, H, W, 4, 16)
            swf.write_chunked(os.path.join(tmp, "f.chk"), fo, H, W, 4, 16)
        dist.barrier()
        rs, rf = swf.ChunkedReader(os.path.join(tmp, "s.chk")), swf.ChunkedReader(os.path.join(tmp, "f.chk"))
        x0, fo = rs.read_full(), rf.read_full()
        dc = swf.DiffusionConfig(solver_steps=2)
        ev = o.key_derive(41, 1, 0)
        a = dn.forecast_step(x0, fo, dc, 11, ev)
        b = dn.forecast_step_chunked(os.path.join(tmp, "s.chk"), os.path.join(tmp, "f.chk"), dc, 11, ev)
        full = 2 * rs.chunk_cover(0, 0, H, W)
        reads = dn.last_chunk_reads()
        same = bool(np.array_equal(a, b))
        # every chunk holding an owned pixel is read (state + forcing); contiguous ownership with 4 x 16
        # chunks reads exactly those, round-robin ownership may revisit a chunk from two window runs
        owned = np.zeros(H * W, np.int64)
        swf.lib().swf_owned_pixels(dn._c, owned.ctypes.data_as(swf.C.c_void_p))
        pix = owned[:dn.local_tokens()]
        need = 2 * len(np.unique((pix // W) // 4 * (W // 16) + (pix % W) // 16))
        partial = reads == need if own == swf.OWN_CONTIGUOUS else need <= reads <= full
        print(f"rank {rank}: chunked forecast bitwise={same} chunk_reads={reads}/{full} (owned chunks {need})",
              flush=True)
        ok &= same and partial
        dist.barrier()
    y = dn.forward(x, 0.9)
    for _ in range(3):  # repeated calls exercise the start-of-forward barrier
        y2 = dn.forward(x, 0.9)
        ok &= np.array_equal(y, y2)
    owned = np.zeros(H * W, np.int64)
    swf.lib().swf_owned_pixels(dn._c, owned.ctypes.data_as(swf.C.c_void_p))
    n_loc = dn.local_tokens()
    parts = [None] * world
    dist.all_gather_object(parts, (owned[:n_loc], y[owned[:n_loc]]))
    if rank == 0:
        y_wp = np.zeros_like(y)
        cover = np.zeros(H * W, np.int64)
        for pix, vals in parts:
            y_wp[pix] = vals
            cover[pix] += 1
        single = swf.Denoiser(sc, H, W, device=local, precision=prec)
        single.load_params(p)
        y1 = single.forward(x, 0.9)
        ref = o.forward(oc, p, x, np.float32(0.9), H, W)
        scale = np.maximum(np.abs(ref).max(axis=0), 1e-30)
        err = float((np.abs(y_wp - ref).max(axis=0) / scale).max())
        bitwise = np.array_equal(y_wp, y1)
        print(f"{name}: world={world} wp={wp} sp={sp} own={own} cover_ok={bool((cover == 1).all())} "
              f"bitwise_vs_1gpu={bitwise} err_vs_oracle={err:.3e}", flush=True)
        ok &= bool((cover == 1).all()) and bitwise and err <= 2e-2
    dn.close()
dist.barrier()
if rank == 0:
    print("WP_CHECK", "PASS" if ok else "FAIL", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
