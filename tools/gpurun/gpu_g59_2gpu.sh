# C4 (40B-shaped 2-block slice) on 2 GPUs with the round-2 code: WP 1x2 and SP 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 \
    bench.py --gpus 2 --workload c4 > gpurun_out/g59_c4_wp.log 2>&1; echo "c4 wp rc=$?"; grep '^{' gpurun_out/g59_c4_wp.log | tail -1 | cut -c1-220
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 \
    bench.py --gpus 2 --workload c4 --sp 2 > gpurun_out/g59_c4_sp2.log 2>&1; echo "c4 sp2 rc=$?"; grep '^{' gpurun_out/g59_c4_sp2.log | tail -1 | cut -c1-220
timeout 900 python bench.py --workload c4 > gpurun_out/g59_c4_1gpu.log 2>&1; echo "c4 1gpu rc=$?"; grep '^{' gpurun_out/g59_c4_1gpu.log | tail -1 | cut -c1-220
