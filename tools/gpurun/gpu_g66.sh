cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_spot.py tests/test_gpu_group.py tests/test_gpu_ops.py tests/test_gpu_bwd_tc.py -x -q > gpurun_out/g66_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g66_t.log
rm -f gpurun_out/g66_gtrace.bin
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/gtrace.so SWF_GEMM_TRACE_OUT=gpurun_out/g66_gtrace.bin timeout 600 python tools/kbench.py 1 qkv_gemm,out_gemm,gateup_gemm,down_gemm > gpurun_out/g66_k.log 2>&1; echo "trace rc=$?"
python tools/gemm_trace.py gpurun_out/g66_gtrace.bin | grep -v decode | head -5
rm -f paper_2509_13523_b200/_build_variants/gtrace.so
bash tools/gpurun/gpu_var_cycles.sh g66 qkv_gemm,out_gemm,gateup_gemm,down_gemm k_gemm_tc
