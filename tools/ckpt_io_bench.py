"""f2 measurement: load a reference-format checkpoint (save_named_arrays: .manifest + .bin, fnv1a64
per array) of the AERIS-1.3B-shaped model (C2) into the BF16 K-major device layout, with the
read-ahead reader at 1 thread (serial, the reference loader's order) and at the default depth; also
the host-only verify. usage: python tools/ckpt_io_bench.py [f32|f64]"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_13523_b200 as swf  # noqa: E402
from bench import CFG, H, W  # noqa: E402

dt = np.float64 if (len(sys.argv) > 1 and sys.argv[1] == "f64") else np.float32
cfg = swf.ModelConfig(**CFG)
base = os.path.join(tempfile.mkdtemp(prefix="swf_ckpt_"), "aeris13b")
rng = np.random.default_rng(0)
t0 = time.perf_counter()
swf.save_checkpoint(base, cfg, ((rng.standard_normal(r * c, dtype=np.float32) * 0.02).astype(dt)
                                for _, r, c in swf.param_arrays(cfg)))
t_write = time.perf_counter() - t0
nbytes = os.path.getsize(base + ".bin")
res = {"workload": f"AERIS-1.3B checkpoint ({dt.__name__}), {nbytes / 1e9:.2f} GB, C2 BF16 context",
       "write_s": t_write}
dn = swf.Denoiser(cfg, H, W, precision=swf.PREC_BF16)
for threads in ("1", None, None):
    if threads:
        os.environ["SWF_CKPT_THREADS"] = threads
    else:
        os.environ.pop("SWF_CKPT_THREADS", None)
    t0 = time.perf_counter()
    dn.load_checkpoint(base)
    dn.sync()
    s = time.perf_counter() - t0
    key = "load_serial_s" if threads else "load_readahead_s"
    res[key] = min(res.get(key, 1e9), s)
t0 = time.perf_counter()
swf.verify_checkpoint(cfg, base)
res["verify_readahead_s"] = time.perf_counter() - t0
res["load_readahead_gbs"] = nbytes / res["load_readahead_s"] / 1e9
res["load_serial_gbs"] = nbytes / res["load_serial_s"] / 1e9
print(json.dumps(res), flush=True)
dn.close()
os.remove(base + ".bin")
