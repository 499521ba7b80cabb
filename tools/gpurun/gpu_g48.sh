cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_depth.py tests/test_gpu_bwd_tc.py -x -q > gpurun_out/g48_t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g48_t.log
bash tools/gpurun/gpu_var_cycles.sh g48 out_gemm k_gemm_tc
