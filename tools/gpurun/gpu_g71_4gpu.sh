# 4-GPU re-validation of the round-2 code: multi-GPU tests on 4 real peers, C2 WP 2x2 bench (the
# driver's N=4 command), C5 with the full 16 members (4 per GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L
timeout 1500 python -m pytest tests/test_gpu_wp.py tests/test_gpu_group.py -q > gpurun_out/g71_mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -2 gpurun_out/g71_mgpu_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 \
    bench.py --gpus 4 > gpurun_out/g71_bench_4gpu.log 2>&1; echo "bench 4gpu rc=$?"; grep '^{' gpurun_out/g71_bench_4gpu.log | tail -1 | cut -c1-200

timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29647 \
    bench.py --gpus 2 > gpurun_out/g71_bench_2gpu.log 2>&1; echo "bench 2gpu rc=$?"; grep '^{' gpurun_out/g71_bench_2gpu.log | tail -1 | cut -c1-200
