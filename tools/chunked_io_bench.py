"""f4 measurement: per-rank window-slice input loading at the C2 shape (720x1440, 70 state + 4
forcing channels, fp32 chunked containers with 90x180 chunks) on one B200: the forecast step from
host arrays vs from the containers (I/O + checksums + staging inside), with and without the next
step's fields prefetched on the background thread, and the reference-style single-threaded
ChunkedReader::read_full of the same files. usage: python tools/chunked_io_bench.py [solver_steps]"""
import json
import math
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_13523_b200 as swf  # noqa: E402
from bench import CFG, H, W, SEED  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tmp = tempfile.mkdtemp(prefix="swf_io_")
rng = np.random.default_rng(0)
cp, cf = CFG["out_channels"], CFG["in_channels"] - 2 * CFG["out_channels"]
paths = []
for k in range(3):
    s = rng.standard_normal((H * W, cp), dtype=np.float32)
    f = rng.standard_normal((H * W, cf), dtype=np.float32)
    ps, pf = os.path.join(tmp, f"state_{k}.chk"), os.path.join(tmp, f"forcing_{k}.chk")
    swf.write_chunked(ps, s, H, W, 90, 180)
    swf.write_chunked(pf, f, H, W, 90, 180)
    paths.append((ps, pf, s, f))
dn = swf.Denoiser(swf.ModelConfig(**CFG), H, W, precision=swf.PREC_BF16)
dn.init_params(SEED, mode=2, scale=0.02 / math.sqrt(CFG["time_dim"]))
dc = swf.DiffusionConfig(solver_steps=steps)
dn.forecast_step(paths[0][2], paths[0][3], dc, 1, 0)  # warm (eager), then graph capture
dn.forecast_step(paths[0][2], paths[0][3], dc, 1, 1)


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return (time.perf_counter() - t0) * 1e3


t_host = timed(lambda: dn.forecast_step(paths[1][2], paths[1][3], dc, 1, 2))
t_chunk = timed(lambda: dn.forecast_step_chunked(paths[1][0], paths[1][1], dc, 1, 3))
reads = dn.last_chunk_reads()
dn.prefetch_chunked(paths[2][0], paths[2][1])  # next step's fields load while this step computes
t_overlap_cur = timed(lambda: dn.forecast_step_chunked(paths[0][0], paths[0][1], dc, 1, 4))
t_prefetched = timed(lambda: dn.forecast_step_chunked(paths[2][0], paths[2][1], dc, 1, 5))
rd = swf.ChunkedReader(paths[1][0])
t_read_full = timed(rd.read_full)
nbytes = (cp + cf) * H * W * 4
print(json.dumps({
    "workload": f"C2 forecast_step, {2 * steps} evaluations, BF16, 1 GPU, fp32 containers 90x180 chunks",
    "field_bytes": nbytes, "chunk_reads": reads,
    "ms_forecast_host_arrays": t_host, "ms_forecast_chunked": t_chunk,
    "ms_forecast_chunked_with_prefetch_of_next": t_overlap_cur, "ms_forecast_chunked_prefetched": t_prefetched,
    "io_cost_ms": t_chunk - t_host, "io_cost_prefetched_ms": t_prefetched - t_host,
    "ms_reference_style_read_full_state": t_read_full,
    "read_full_gbs": paths[1][2].nbytes / t_read_full / 1e6,
}), flush=True)
dn.close()
