# out GEMM epilogue: full chunks through shared memory in 16-byte pieces (r_v4) vs HEAD (r_base)
# parity tests on the working-tree build, then base-clock cycles and free-clock ms of the QKV GEMM.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_depth.py tests/test_gpu_group.py tests/test_gpu_wp.py -m gpu -x -q > gpurun_out/g84_t.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/g84_t.log)"
bash tools/gpurun/gpu_var_cycles.sh g84 out_gemm 'k_gemm_tc' > /dev/null 2>&1
cat gpurun_out/g84_cyc.log
