cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py -x -q > gpurun_out/g72_t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g72_t.log
bash tools/gpurun/gpu_var_cycles.sh g72 out_gemm,qkv_gemm,gateup_gemm k_gemm_tc
