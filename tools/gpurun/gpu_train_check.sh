# Sharded training-step checks on a 4-GPU box: DP only, WP 1x2 x DP 2, WP 2x2 (tools/dp_check.py).
T=${1:-train}
for wp in 1 2 4; do
  SWF_DP_WP=$wp timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
      --master-port $((29720 + wp)) tools/dp_check.py > gpurun_out/${T}_wp$wp.log 2>&1; echo "dp_check wp=$wp rc=$?"
done
SWF_DP_WP=2 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
    --master-port 29730 tools/dp_check.py > gpurun_out/${T}_2gpu_wp2.log 2>&1; echo "dp_check 2 GPUs wp=2 rc=$?"
