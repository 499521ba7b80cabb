cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/pr1.so timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_c2_spot.py tests/test_gpu_parity.py -x -q > gpurun_out/g61_t.log 2>&1; echo "pairs tests rc=$?"; tail -3 gpurun_out/g61_t.log
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/trace.so SWF_ATTN_TRACE_OUT=gpurun_out/g61_trace.bin timeout 300 python tools/kbench.py 2 attention > gpurun_out/g61_k.log 2>&1; echo "trace rc=$?"
python tools/attn_pp_trace.py gpurun_out/g61_trace.bin | head -14
rm -f paper_2509_13523_b200/_build_variants/trace.so
bash tools/gpurun/gpu_var_cycles.sh g61 attention k_attn_pp
