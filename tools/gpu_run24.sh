for sp in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$sp bench.py --gpus 2 --steps 3 --warmup 2 --workload c4 --sp $sp --no-e2e > gpurun_out/r24_c4_sp$sp.log 2>&1; echo "c4 sp$sp rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/r24_c4_sp$sp.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['tflops_per_gpu'], d['config']['parallelism'], d['clocks']['sm_mhz'])
print(d['kernel_shares'])" 2>&1 | tail -3
done
