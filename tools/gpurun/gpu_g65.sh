cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/g65_gtrace.bin
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/gtrace.so SWF_GEMM_TRACE_OUT=gpurun_out/g65_gtrace.bin timeout 600 python tools/kbench.py 1 qkv_gemm,out_gemm,gateup_gemm,down_gemm > gpurun_out/g65_k.log 2>&1; echo "rc=$?"
python tools/gemm_trace.py gpurun_out/g65_gtrace.bin
