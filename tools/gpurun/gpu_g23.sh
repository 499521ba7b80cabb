cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_depth.py -x -q > gpurun_out/g23_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g23_tests.log
bash tools/gpurun/gpu_var_cycles.sh g23 out_gemm,down_gemm k_gemm_tc
