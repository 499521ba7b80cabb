import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time
import bench
import paper_2509_13523_b200 as swf
cfg = swf.ModelConfig(**bench.CFG)
dn = swf.Denoiser(cfg, bench.H, bench.W, precision=swf.PREC_BF16)
dn.init_params(bench.SEED, mode=2, scale=0.02 / math.sqrt(bench.CFG["time_dim"]))
x = bench.synthetic_input(dn, bench.CFG)
d_in = torch.from_numpy(x).cuda(); d_out = torch.empty(bench.H * bench.W * 70, device="cuda")
dn.forward_device(d_in.data_ptr(), bench.T_STEP, d_out.data_ptr()); dn.sync()
time.sleep(2.0)
print("attention cold after idle:", dn.bench_kernel("attention", 1, -1))
for _ in range(3):
    g = dn.bench_kernel("gateup_gemm", 1, 4)
    a1 = dn.bench_kernel("attention", 1, -1)
    a2 = dn.bench_kernel("attention", 1, -1)
    a3 = dn.bench_kernel("attention", 1, -1)
    print(f"after 4x gateup ({g:.1f} ms): attention #1 {a1:.1f}  #2 {a2:.1f}  #3 {a3:.1f} ms")
