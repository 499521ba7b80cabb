# 8-rank functional checks on a 4-GPU box (2 ranks per GPU, gloo plumbing): WP/SP bitwise checks;
# the NCCL data-parallel training check at 4 ranks (NCCL needs one rank per GPU).
T=${1:-wp8}
for cfg in "0 1" "1 1" "0 2"; do
  set -- $cfg
  SWF_OWN=$1 SWF_SP=$2 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 \
      --master-port 29700 tools/wp_check.py > gpurun_out/${T}_own$1_sp$2.log 2>&1; echo "wp own=$1 sp=$2 rc=$?"
done
timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29710 \
    tools/dp_check.py > gpurun_out/${T}_dp4.log 2>&1; echo "dp4 rc=$?"
