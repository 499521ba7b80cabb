# 4-GPU validation of the final code: multi-GPU tests on 4 real peers, then the driver's scaling commands
# on one box: C2 at N = 1, 2 (WP 1x2) and 4 (WP 2x2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L
timeout 1500 python -m pytest tests/test_gpu_wp.py tests/test_gpu_group.py -q > gpurun_out/g90_mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -1 gpurun_out/g90_mgpu_tests.log
timeout 900 python bench.py > gpurun_out/g90_bench_1gpu.log 2>&1; echo "bench 1gpu rc=$?"; grep '^{' gpurun_out/g90_bench_1gpu.log | tail -1 | cut -c1-160
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29647 \
    bench.py --gpus 2 > gpurun_out/g90_bench_2gpu.log 2>&1; echo "bench 2gpu rc=$?"; grep '^{' gpurun_out/g90_bench_2gpu.log | tail -1 | cut -c1-160
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 \
    bench.py --gpus 4 > gpurun_out/g90_bench_4gpu.log 2>&1; echo "bench 4gpu rc=$?"; grep '^{' gpurun_out/g90_bench_4gpu.log | tail -1 | cut -c1-160
