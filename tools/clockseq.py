"""Alternate kernel classes on the C2 buffers with nvidia-smi clocks sampled every 10 ms, to see
how the power cap moves the SM clock between kernels."""
import math
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_13523_b200 as swf  # noqa: E402

cfg = swf.ModelConfig(**bench.CFG)
dn = swf.Denoiser(cfg, bench.H, bench.W, precision=swf.PREC_BF16)
dn.init_params(bench.SEED, mode=2, scale=0.02 / math.sqrt(bench.CFG["time_dim"]))
x = bench.synthetic_input(dn, bench.CFG)
d_in = torch.from_numpy(x).cuda()
d_out = torch.empty(bench.H * bench.W * bench.CFG["out_channels"], device="cuda")
dn.forward_device(d_in.data_ptr(), bench.T_STEP, d_out.data_ptr())
dn.sync()
smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=timestamp,clocks.sm,power.draw", "--format=csv,noheader",
                        "-lms", "10"], stdout=open("gpurun_out/clockseq_smi.csv", "w"))
time.sleep(1.0)
seq = sys.argv[1].split(",")
t0 = time.time()
for k in seq:
    ts = time.time() - t0
    ms = dn.bench_kernel(k, block=1, reps=int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    print(f"{ts:8.3f}s {k:12s} {ms:8.2f} ms/launch", flush=True)
time.sleep(0.5)
smi.terminate()
