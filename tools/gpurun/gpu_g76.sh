cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_depth.py tests/test_gpu_group.py tests/test_gpu_ops.py -x -q > gpurun_out/g76_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g76_t.log
bash tools/gpurun/gpu_var_cycles.sh g76 down_gemm,gateup_gemm k_gemm_tc
