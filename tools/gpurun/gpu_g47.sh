cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bwd_tc.py tests/test_gpu_parity.py -q -k "bwd or backward or train or loss or gemm" > gpurun_out/g47_t.log 2>&1; echo "bwd tests rc=$?"; tail -2 gpurun_out/g47_t.log
timeout 300 python tools/bwd_err_probe.py 0.03 2>&1 | tail -3
timeout 900 python tools/bwd_bench.py 240 480 2 > gpurun_out/g47_bwd_mid.log 2>&1; echo "rc=$?"; cat gpurun_out/g47_bwd_mid.log
timeout 900 python bench.py --workload train --train-precision bf16 --steps 2 --warmup 1 > gpurun_out/g47_train_bf16.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/g47_train_bf16.log | cut -c1-200
