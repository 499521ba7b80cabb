"""Per-block kernel times of one C2 forward (CUDA events per launch)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2509_13523_b200 as swf
cfg = swf.ModelConfig(**bench.CFG)
dn = swf.Denoiser(cfg, bench.H, bench.W, precision=swf.PREC_BF16)
dn.init_params(bench.SEED, mode=2, scale=0.02 / math.sqrt(bench.CFG["time_dim"]))
x = bench.synthetic_input(dn, bench.CFG)
d_in = torch.from_numpy(x).cuda(); d_out = torch.empty(bench.H * bench.W * 70, device="cuda")
for _ in range(2): dn.forward_device(d_in.data_ptr(), bench.T_STEP, d_out.data_ptr())
dn.sync(); dn.profile(True)
dn.forward_device(d_in.data_ptr(), bench.T_STEP, d_out.data_ptr()); dn.sync()
L = dn.profile_launches()
att = [ms for k, ms in L if k == "attention"]
gu = [ms for k, ms in L if k == "gateup_gemm"]
print("attention per block:", " ".join(f"{v:.1f}" for v in att))
print("gateup per block:   ", " ".join(f"{v:.1f}" for v in gu))
print("kbench attention (block 1 replay):", dn.bench_kernel("attention", 1, 5))
