# final-code 2-GPU line (the driver's N=2 command) and the reference arm under torchrun
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 \
    bench.py --gpus 2 > gpurun_out/g77_bench_2gpu.log 2>&1; echo "bench 2gpu rc=$?"; grep '^{' gpurun_out/g77_bench_2gpu.log | tail -1 | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29663 \
    bench.py --impl reference --gpus 2 > gpurun_out/g77_ref_2gpu.log 2>&1; echo "ref 2gpu rc=$?"; grep '^{' gpurun_out/g77_ref_2gpu.log | tail -1 | cut -c1-300
