# WP scaling lines (contiguous ownership) on 2 and 4 GPUs of one box; usage: bash tools/gpurun/gpu_scale.sh TAG
T=${1:-scale}
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n \
      bench.py --gpus $n > gpurun_out/${T}_${n}gpu.log 2>&1; echo "$n gpu rc=$?"; grep '^{' gpurun_out/${T}_${n}gpu.log | tail -1 | cut -c1-220
done
