# BF16 training step on 2 GPUs (data parallel, one rank per GPU, NCCL all-reduce of the gradients)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload train --train-precision bf16 > gpurun_out/g99_train_1gpu.log 2>&1; echo "1gpu rc=$?"; tail -1 gpurun_out/g99_train_1gpu.log | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 \
    bench.py --gpus 2 --workload train --train-precision bf16 > gpurun_out/g99_train_2gpu.log 2>&1; echo "2gpu rc=$?"; grep '^{' gpurun_out/g99_train_2gpu.log | tail -1 | cut -c1-300
