#!/usr/bin/env python
"""bench.py -- AERIS-1.3B-shaped denoiser step at 0.25 deg on B200 (BASELINE.json configs[1]).

One "step" = one full denoiser forward (swinflow::forward, swin.hpp:327-368) over the 720 x 1440
grid: encode, 20 shifted-window blocks (h=1536, 12 heads, ffn 9216, 60 x 60 windows), decode.
Synthetic fields and random-init weights of that architecture (no checkpoints offline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0). `value` = whole-job pixels/s with inputs resident in HBM;
`e2e` = the same metric through the C-ABI host-buffer call (H2D input + D2H output inside the
timed region); `roofline` = the dominant kernel vs the measured bf16 peak; `cpu_baseline` = the
CPU oracle (test infrastructure, not the product) on a bounded sample, extrapolated per FLOP.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---------------------------------------------------------------------- workload (BASELINE.json)
H, W = 720, 1440
CFG = dict(hidden_dim=1536, n_heads=12, ffn_dim=9216, n_layers=10, blocks_per_layer=2, window_px=60,
           in_channels=144, out_channels=70, time_dim=1536)  # perf_model.cpp:49-61 row "1.3B", w=60
# BASELINE.json configs[3]: wide-layer slice of the 40B shape (perf_model.cpp:38 row "40B": dim 6144,
# 48 heads, ffn 40960, w=60), 2 blocks (shift 0, 30), on the same 720x1440 grid; needs >= 2 GPUs
CFG_C4 = dict(hidden_dim=6144, n_heads=48, ffn_dim=40960, n_layers=1, blocks_per_layer=2, window_px=60,
              in_channels=144, out_channels=70, time_dim=6144)
T_STEP = math.pi / 4
SEED = 2024
WEIGHT_SCALE = 0.01
METRIC = "denoiser-step pixels/sec"


def flops_per_step(c: dict, npix: int, nblocks: int | None = None) -> float:
    """perf::flops_forward_per_sample (perf_model.cpp:63-74)."""
    h, f, s, w = c["hidden_dim"], c["ffn_dim"], float(npix), c["window_px"]
    nb = nblocks if nblocks is not None else c["n_layers"] * c["blocks_per_layer"]
    per_block = 6 * s * h * h + 4 * s * w * w * h + 2 * s * h * h + 6 * s * h * f
    return nb * per_block + 2 * s * c["in_channels"] * h + 2 * s * h * c["out_channels"]


def class_flops(c: dict, M: int) -> dict:
    """Algorithmic FLOPs (or bytes, for the norm) per launch of each kernel class."""
    h, f, w = c["hidden_dim"], c["ffn_dim"], c["window_px"]
    return {
        "qkv_gemm": 2.0 * M * h * 3 * h,
        "attention": 4.0 * M * w * w * h,
        "out_gemm": 2.0 * M * h * h,
        "gateup_gemm": 2.0 * M * h * 2 * f,
        "down_gemm": 2.0 * M * f * h,
        "encode_gemm": 2.0 * M * c["in_channels"] * h,
        "decode_gemm": 2.0 * M * h * c["out_channels"],
    }


def attention_executed(c: dict, H_: int, W_: int, nloc_frac: float = 1.0) -> dict:
    """Executed vs algorithmic attention FLOPs per step for the BF16 kernel (k_attn_pp, k_attn.cu): a work
    item is a pair of 128-query tiles (M = 256) of one (window, head) over 64-key tiles; the last pair and
    the last key tile are partly padding, and on the shifted blocks the seam-masked bottom window row
    skips the key tiles outside each query range (pp::range_of). Counts 2 x 2 x 256 x 64 x d per (item,
    key tile) (QK^T and PV), against perf_model's 4 s w^2 h."""
    KT = 64
    w, h, d = c["window_px"], c["hidden_dim"], c["hidden_dim"] // c["n_heads"]
    s = w * w
    ny, nx = H_ // w, W_ // w
    nb = c["n_layers"] * c["blocks_per_layer"]
    npairs = -(-s // 256)
    ex = 0.0
    for b in range(nb):
        shift = 0 if b % 2 == 0 else w // 2
        for masked in (False, True):
            nwin = nx if masked else (ny - 1) * nx + (0 if shift else nx)
            if masked and not shift:
                continue
            tiles = 0
            for qp in range(npairs):
                qp0 = qp * 256
                split = (w - shift) * w if masked else s
                qlast = min(qp0 + 256, s) - 1
                lo = split if (masked and qp0 >= split) else 0
                hi = split if (masked and qlast < split) else s
                tiles += -(-hi // KT) - lo // KT
            ex += nwin * c["n_heads"] * tiles * 2 * 2 * 256 * KT * d
    alg = nb * 4.0 * H_ * W_ * s * h
    return {"algorithmic_per_step": alg * nloc_frac, "executed_per_step": ex * nloc_frac, "executed_over_algorithmic": ex / alg}


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sus": p["bf16_tflops_sustained"],
                "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self._stop = device, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------- synthetic input
def synthetic_input(dn, cfg: dict) -> np.ndarray:
    """[x_t ; x_prev ; forcings (3 + 1 zero pad)] + posenc, fp32 [N][144].
    x_t is the window-keyed noise field (diffusion.hpp:91-108, sigma_d = 1)."""
    cp, cin = cfg["out_channels"], cfg["in_channels"]
    n = H * W
    rng = np.random.default_rng(SEED)
    x = np.empty((n, cin), np.float32)
    x[:, :cp] = dn.noise_field(SEED, 1, cp, 1.0)
    x[:, cp:2 * cp] = rng.standard_normal((n, cp), dtype=np.float32)
    x[:, 2 * cp:cin] = 0.0
    x[:, 2 * cp:2 * cp + 3] = rng.standard_normal((n, 3), dtype=np.float32)
    # sinusoidal_pos_encode (posenc.hpp:16-37)
    per_axis = cin // 2
    nf = (per_axis + 1) // 2
    yy, xx = np.divmod(np.arange(n), W)
    for axis, pos in ((0, yy), (1, xx)):
        for i in range(per_axis):
            om = 10000.0 ** (-(i // 2) / max(1, nf))
            v = np.sin(pos * om) if i % 2 == 0 else np.cos(pos * om)
            x[:, axis * per_axis + i] += v.astype(np.float32)
    return x


# ---------------------------------------------------------------------- CPU baselines (oracle)
def cpu_sample(windows: int, blocks: int) -> dict:
    """Oracle (fp32, all host threads) on `windows` 60x60 windows x `blocks` blocks at the C2
    widths; returns pixels/s extrapolated per FLOP to the full 20-block 720x1440 step."""
    from oracle import pyoracle as o
    o.use_all_cores()
    c = dict(CFG, n_layers=1, blocks_per_layer=blocks)
    oc = o.ModelConfig(**c)
    p = o.init_params(oc, SEED, random=False, dtype=np.float32)
    hh, ww = 60, 60 * windows
    x = o.random_field(oc.in_channels, hh * ww, SEED + 1).astype(np.float32)
    t0 = time.perf_counter()
    o.forward(oc, p, x, np.float32(T_STEP), hh, ww)
    dt = time.perf_counter() - t0
    fl = flops_per_step(c, hh * ww)
    pix_per_s = fl / dt / (flops_per_step(CFG, H * W) / (H * W))
    return {"value": pix_per_s, "seconds": dt, "flops": fl, "cores": o.num_threads(),
            "sample": f"C2 widths (h=1536, 12 heads, ffn 9216, w=60), {windows} window(s) of 60x60 x {blocks} "
                      f"block(s) + encode/decode, fp32 oracle; pixels/s extrapolated per FLOP to the "
                      f"20-block 720x1440 step"}


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference's CPU algorithm (oracle port; the reference itself cannot be
    built here: Eigen3 / doctest / CLI11 absent) on the host cores, rank 0 only."""
    if rank != 0:
        return
    from oracle import pyoracle as o
    o.use_all_cores()  # all host threads, also under torchrun (which exports OMP_NUM_THREADS=1)
    c = dict(CFG, n_layers=1, blocks_per_layer=1)
    oc = o.ModelConfig(**c)
    p = o.init_params(oc, SEED, random=False, dtype=np.float32)
    x = o.random_field(oc.in_channels, 3600, SEED + 1).astype(np.float32)
    for _ in range(args.warmup):
        o.forward(oc, p, x, np.float32(T_STEP), 60, 60)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.forward(oc, p, x, np.float32(T_STEP), 60, 60)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    fl = flops_per_step(c, 3600)
    v = fl / dt / (flops_per_step(CFG, H * W) / (H * W))
    sample = ("one 60x60 window x 1 block (+ encode/decode) at the C2 widths per step, fp32 oracle port of "
              "swin.hpp forward; pixels/s extrapolated per FLOP to the 20-block 720x1440 step")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "pixels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "AERIS-1.3B denoiser step, 720x1440, w=60 (sampled on CPU)",
                       "grid": [H, W], "model": "swin-dit-1.3B", "window": 60},
            "cpu_baseline": {"value": v, "unit": "pixels/s", "cores": o.num_threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "pixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- ours
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import paper_2509_13523_b200 as swf

    global CFG
    if args.workload == "c4":
        CFG = CFG_C4

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    cfg = swf.ModelConfig(**CFG)
    sp = args.sp
    wp = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}[world // sp]
    topo = (wp[0], wp[1], sp, rank, swf.OWN_CONTIGUOUS) if world > 1 else None
    dn = swf.Denoiser(cfg, H, W, device=local_rank, precision=swf.PREC_BF16, topology=topo)
    if world > 1:
        dn.connect_peers_torch(dist)
    # init_parameters_random(seed, 0.01): every branch live (attention logits with real spread, so the
    # kernel's online-softmax rescale path runs in the timed region; tests/test_gpu_c2_spot.py)
    dn.init_params(SEED, mode=1, scale=WEIGHT_SCALE)

    x_host = synthetic_input(dn, CFG)
    n_in, n_out = x_host.size, H * W * CFG["out_channels"]
    stream = torch.cuda.ExternalStream(dn.stream, device=torch.device("cuda", local_rank))
    d_in = torch.from_numpy(x_host).to(f"cuda:{local_rank}")
    d_out = torch.empty(n_out, dtype=torch.float32, device=f"cuda:{local_rank}")
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        dn.forward_device(d_in.data_ptr(), T_STEP, d_out.data_ptr())
    dn.sync()
    out0 = d_out.cpu().numpy()
    finite = bool(np.isfinite(out0).all())
    out_rms = float(np.sqrt(np.mean(out0.astype(np.float64) ** 2)))

    # ---- timed region: device-resident inputs (value) + per-kernel events (roofline)
    dn.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            dn.forward_device(d_in.data_ptr(), T_STEP, d_out.data_ptr())
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    dn.sync()
    prof = dn.profile_read()
    dn.profile(False)
    launches = dn.kernel_launches() * args.steps
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pixels = H * W  # strong scaling: the whole grid is one step at every N (WP shards it)
    value = pixels / (ms / 1e3)
    step_flops = flops_per_step(CFG, H * W)
    peaks = measured_peaks()
    tflops_gpu = step_flops / (ms / 1e3) / world / 1e12

    # ---- roofline of the dominant kernel class
    M = dn.local_tokens()
    cf = class_flops(CFG, M)
    dom = max((k for k in prof if k in cf), key=lambda k: prof[k][0])
    dom_ms = prof[dom][0] / max(prof[dom][1], 1)
    achieved = cf[dom] / (dom_ms / 1e3) / 1e12
    total_ms = sum(v[0] for v in prof.values())
    shares = {k: round(v[0] / total_ms, 4) for k, v in prof.items() if v[1]}
    per_class = {k: {"ms_per_launch": v[0] / v[1], "launches": v[1],
                     "tflops": (cf[k] / (v[0] / v[1] / 1e3) / 1e12) if k in cf else None}
                 for k, v in prof.items() if v[1]}

    # ---- e2e through the C-ABI host-buffer call (pinned host memory, copies inside)
    e2e = None
    if not args.no_e2e:
        h_in = torch.from_numpy(x_host).pin_memory()
        h_out = torch.empty((H * W, CFG["out_channels"]), dtype=torch.float32).pin_memory()
        import ctypes
        for _ in range(1):
            swf._check(swf.lib().swf_forward(dn._c, ctypes.c_void_p(h_in.data_ptr()), T_STEP,
                                             ctypes.c_void_p(h_out.data_ptr()), swf.F32))
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            swf._check(swf.lib().swf_forward(dn._c, ctypes.c_void_p(h_in.data_ptr()), T_STEP,
                                             ctypes.c_void_p(h_out.data_ptr()), swf.F32))
        barrier()
        e2e_s = (time.perf_counter() - t0) / args.steps
        if dist is not None:
            t = torch.tensor([e2e_s], device=f"cuda:{local_rank}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": pixels / e2e_s, "unit": "pixels/s", "h2d_bytes_per_step": n_in * 4 * world,
               "d2h_bytes_per_step": n_out * 4 * world, "ms_per_step": e2e_s * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        s = cpu_sample(windows=1, blocks=2)
        cpu = {"value": s["value"], "unit": "pixels/s", "cores": s["cores"], "kind": "port", "sample": s["sample"],
               "seconds": round(s["seconds"], 2)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pixels/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": ("AERIS-1.3B-shaped denoiser step (BASELINE.json configs[1])" if args.workload == "c2"
                                    else "AERIS-40B-shaped wide-layer slice, 2 blocks (BASELINE.json configs[3])"),
                       "grid": [H, W],
                       "model": ("swin-dit-1.3B (h=1536, 12 heads, ffn 9216, 20 blocks, w=60, C_in=144, C_out=70)"
                                 if args.workload == "c2" else
                                 "swin-dit-40B slice (h=6144, 48 heads, ffn 40960, 2 blocks, w=60, C_in=144, C_out=70)"),
                       "parallelism": f"wp{wp[0]}x{wp[1]}" + (f"_sp{sp}" if sp > 1 else ""),
                       "params": swf.param_count(cfg),
                       "weights": f"init_parameters_random(seed=2024, scale={WEIGHT_SCALE}) (every branch live)",
                       "t": T_STEP, "l2": "inputs + per-step traffic (~50 GB) far larger than the 126 MB L2"},
            "tflops_per_gpu": tflops_gpu,
            "frac_of_peak": {"bf16_measured_burst": tflops_gpu / peaks["bf16"],
                             "bf16_measured_sustained": tflops_gpu / peaks["bf16_sus"],
                             "bf16_datasheet_2250": tflops_gpu / 2250.0},
            "flops_per_step": step_flops,
            "roofline": {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peaks["bf16_sus"],
                         "peak_kind": f"{peaks['src']} sustained bf16 (kernel timed inside a long step)",
                         "unit": "TFLOP/s", "frac": achieved / peaks["bf16_sus"], "traffic": ncu_traffic(dom),
                         "traffic_unit": "DRAM bytes per launch (ncu --set full capture, profiles/)",
                         "flops_per_launch": cf[dom], "ms_per_launch": dom_ms},
            "kernel_shares": shares, "kernels": per_class,
            "attention_flops": attention_executed(CFG, H, W, 1.0 / world),
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary(),
            "output_check": {"finite": finite, "rms": out_rms},
        }
        print(json.dumps(line), flush=True)
    dn.close()
    if dist is not None:
        dist.destroy_process_group()


def ncu_traffic(kernel_class: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class from the committed
    ncu --set full capture (profiles/ncu_traffic_bytes.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic_bytes.json")) as f:
            return json.load(f)["dram_bytes_per_launch"].get(kernel_class)
    except Exception:
        return None


def run_c5(args, rank: int, world: int, local_rank: int):
    """BASELINE.json configs[4]: ensemble generation, members x (2 x solver_steps) TrigFlow sampler
    evaluations x 1 autoregressive step on the C2 model, replicas only (members split across ranks;
    each rank holds the whole grid). "20 TrigFlow sampler steps" is read as 10 DPM-Solver++ 2S
    steps = 20 network evaluations (test_trigflow.cpp:239-245). One rollout_ensemble call per
    rank (device-resident solver, window-keyed noise) with host buffers in and out; value = member
    evaluations x pixels / max-over-ranks wall time."""
    import torch
    import paper_2509_13523_b200 as swf

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    if args.members % world:
        raise SystemExit(f"--members {args.members} must divide over {world} ranks")
    per = args.members // world
    cfg = swf.ModelConfig(**CFG)
    dn = swf.Denoiser(cfg, H, W, device=local_rank, precision=swf.PREC_BF16)
    dn.init_params(SEED, mode=1, scale=WEIGHT_SCALE)
    cp, cf = CFG["out_channels"], CFG["in_channels"] - 2 * CFG["out_channels"]
    rng = np.random.default_rng(SEED + 7)
    x0 = rng.standard_normal((H * W, cp), dtype=np.float32)
    forc = [rng.standard_normal((H * W, cf), dtype=np.float32)]
    dc = swf.DiffusionConfig(solver_steps=args.solver_steps)
    evals = 2 * args.solver_steps

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    x_in = synthetic_input(dn, CFG)
    d_in = torch.from_numpy(x_in).to(f"cuda:{local_rank}")
    d_out = torch.empty(H * W * cp, dtype=torch.float32, device=f"cuda:{local_rank}")
    for _ in range(max(args.warmup, 1)):  # warm the forward path (kernels, clocks)
        dn.forward_device(d_in.data_ptr(), T_STEP, d_out.data_ptr())
    dn.sync()
    with ClockSampler(local_rank) as clk:
        barrier()
        t0 = time.perf_counter()
        out = dn.rollout_ensemble(x0, forc, per, 1, dc, SEED, 1000 + rank)
        barrier()
        sec = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([sec], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    finite = bool(np.isfinite(out).all())
    total_evals = args.members * evals
    value = total_evals * H * W / sec
    if rank == 0:
        step_flops = flops_per_step(CFG, H * W)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "pixels/s", "n_gpus": world, "steps": 1, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "ensemble generation (BASELINE.json configs[4]), replicas",
                       "grid": [H, W], "members": args.members, "members_per_gpu": per,
                       "sampler": f"{args.solver_steps} DPM-Solver++ 2S steps = {evals} denoiser evaluations per member",
                       "autoregressive_steps": 1, "model": "swin-dit-1.3B (C2)", "parallelism": f"replicas x{world}",
                       "step": "one rollout_ensemble call per rank (host buffers in/out, device-resident solver)"},
            "tflops_per_gpu": total_evals * step_flops / sec / world / 1e12,
            "evals_per_s": total_evals / sec,
            "e2e": {"value": value, "unit": "pixels/s", "h2d_bytes_per_step": int(x0.nbytes + forc[0].nbytes) * world,
                    "d2h_bytes_per_step": int(out.nbytes) * world, "ms_per_step": sec * 1e3},
            "clocks": clk.summary(), "output_check": {"finite": finite},
        }), flush=True)
    dn.close()
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------------------- f3: training step
def run_train(args, rank: int, world: int, local_rank: int):
    """One data-parallel training step of the AERIS-1.3B-shaped model (C2 widths, 20 blocks) on a
    TH x TW grid slice in the FP32 validation mode: per rank `gas` microbatches (swf_train_accumulate:
    H2D of the sample's fields, device noise / t, forward with saved block inputs, loss, backward,
    accumulate) and one in-place NCCL all-reduce of the device gradients. The optimizer update is not
    part of the reference step (reference_train_step returns the gradients) and the gradients stay
    on the device. FLOPs counted as 3x the forward (forward + input and weight gradients), the
    backward's recompute of the block internals excluded."""
    import torch
    import paper_2509_13523_b200 as swf
    from paper_2509_13523_b200.train import _DeviceView

    TH, TW = args.train_grid
    dist = None
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    cfg = swf.ModelConfig(**CFG)
    dn = swf.Denoiser(cfg, TH, TW, device=local_rank, precision=swf.PREC_FP32)
    dn.init_params(SEED, mode=2, scale=0.02 / math.sqrt(CFG["time_dim"]))
    bf16 = args.train_precision == "bf16"
    if bf16:  # BF16 training mode: linears and attention (fwd + bwd) on the tensor cores
        dn.set_backward_precision(swf.PREC_BF16)
    rng = np.random.default_rng(SEED + rank)
    cp, cf = CFG["out_channels"], CFG["in_channels"] - 2 * CFG["out_channels"]
    fields = [(rng.standard_normal((TH * TW, cp), dtype=np.float32),
               rng.standard_normal((TH * TW, cp), dtype=np.float32),
               rng.standard_normal((TH * TW, cf), dtype=np.float32)) for _ in range(2)]
    w = swf.LossWeights.make(TH, np.ones(cp))
    dc = swf.DiffusionConfig()
    ptr, n = dn.train_grads_device()
    grads = torch.as_tensor(_DeviceView(ptr, n), device=torch.device("cuda", local_rank))
    stream = torch.cuda.ExternalStream(dn.stream, device=torch.device("cuda", local_rank))
    gas = args.gas
    losses = []

    def step(k):
        dn.train_reset()
        for g in range(gas):
            sid = (k * world + rank) * gas + g
            xp, x0, fo = fields[sid % 2]
            losses.append(dn.train_accumulate(xp, x0, fo, w, dc, SEED, sid))
        if dist is not None:
            dist.all_reduce(grads)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            step(args.warmup + k)
        e1.record(torch.cuda.current_stream())  # after the all-reduce (NCCL orders after the current stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    samples = world * gas
    model_flops = 3.0 * flops_per_step(CFG, TH * TW) * samples
    fp32_peak = 148 * 128 * 2 * 1965e6 / 1e12  # FFMA lanes x 2 x max SM clock (no measured FP32 peak)
    if rank == 0:
        tf = model_flops / (ms * 1e-3) / world / 1e12
        if bf16:
            mp = measured_peaks()
            peak, peak_kind, bound = mp["bf16_sus"], f"bf16 sustained ({mp['src']})", "tensor"
        else:
            peak, bound = fp32_peak, "fp32"
            peak_kind = "computed: 148 SMs x 128 FFMA lanes x 2 x 1965 MHz (no measured FP32 peak)"
        print(json.dumps({
            "metric": "training samples/sec", "value": samples / (ms * 1e-3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if bf16 else "f32", "data": "synthetic",
            "config": {"workload": "f3 training step (reference_train_step, "
                                   + ("BF16 training mode" if bf16 else "FP32 validation mode")
                                   + "), AERIS-1.3B widths / 20 blocks on a grid slice",
                       "grid": [TH, TW], "gas": gas, "parallelism": f"dp{world}", "model": "swin-dit-1.3B (C2)",
                       "l2": "inputs far larger than L2 (weights 5.3 GB fp32 + activations)"},
            "roofline": {"bound": bound, "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "peak_kind": peak_kind,
                         "traffic": None, "flops": "3 x forward per sample (perf_model.cpp:63-74), recompute excluded"},
            "e2e": {"value": samples / (ms * 1e-3), "unit": "samples/s",
                    "h2d_bytes_per_step": int(sum(a.nbytes for a in fields[0])) * samples, "d2h_bytes_per_step": 8 * samples},
            "loss_finite": bool(np.isfinite(losses).all()),
            "clocks": clk.summary(),
        }), flush=True)
    dn.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sp", type=int, default=1, help="sequence-parallel degree (window rows split into SP bands)")
    ap.add_argument("--workload", choices=["c2", "c4", "c5", "train"], default="c2",
                    help="c2: AERIS-1.3B 20-block step (headline); c4: 40B-shaped 2-block wide-layer slice; "
                         "c5: ensemble generation (members x sampler evaluations, replicas); "
                         "train: FP32 data-parallel training step (f3)")
    ap.add_argument("--members", type=int, default=16, help="c5: ensemble members over all ranks")
    ap.add_argument("--solver-steps", type=int, default=10, help="c5: DPM-Solver++ 2S steps (2 evaluations each)")
    ap.add_argument("--gas", type=int, default=1, help="train: microbatches per rank")
    ap.add_argument("--train-grid", type=int, nargs=2, default=[120, 240], help="train: grid slice (H W)")
    ap.add_argument("--train-precision", choices=["fp32", "bf16"], default="fp32",
                    help="train: FP32 validation mode or the BF16 training mode (tensor cores)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "c5":
        run_c5(args, rank, world, local_rank)
    elif args.workload == "train":
        run_train(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
