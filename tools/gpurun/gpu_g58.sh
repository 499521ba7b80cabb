cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_group.py tests/test_gpu_attention.py -x -q > gpurun_out/g58_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g58_t.log
bash tools/gpurun/gpu_var_cycles.sh g58 qkv_gemm,gateup_gemm k_gemm_tc
