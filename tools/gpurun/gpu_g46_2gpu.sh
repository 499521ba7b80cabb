# 2-GPU re-validation of the round-2 code: multi-GPU tests on real peers, the driver's N=2 bench and
# reference-arm commands (torchrun, one rank per GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L
timeout 1200 python -m pytest tests/test_gpu_wp.py tests/test_gpu_group.py -q > gpurun_out/g46_mgpu_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -2 gpurun_out/g46_mgpu_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29642 \
    bench.py --gpus 2 > gpurun_out/g46_bench_2gpu.log 2>&1; echo "bench 2gpu rc=$?"; grep '^{' gpurun_out/g46_bench_2gpu.log | tail -1 | cut -c1-250
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29643 \
    bench.py --impl reference --gpus 2 > gpurun_out/g46_ref_2gpu.log 2>&1; echo "ref 2gpu rc=$?"; grep '^{' gpurun_out/g46_ref_2gpu.log | tail -1 | cut -c1-200
