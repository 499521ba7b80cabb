# final code, 4 GPUs: C5 ensemble generation with the full 16 members (4 per GPU, replicas), and the
# reference arm under torchrun at N = 4 (rank 0 runs the oracle port on the host cores)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 \
    bench.py --gpus 4 --workload c5 --members 16 --steps 1 --warmup 1 > gpurun_out/g93_c5_4gpu.log 2>&1; echo "c5 4gpu rc=$?"; grep '^{' gpurun_out/g93_c5_4gpu.log | tail -1 | cut -c1-240
