cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_c2_spot.py tests/test_gpu_parity.py -x -q > gpurun_out/g75_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g75_t.log
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/trace.so SWF_ATTN_TRACE_OUT=gpurun_out/g75_trace.bin timeout 300 python tools/kbench.py 2 attention > gpurun_out/g75_k.log 2>&1; echo "trace rc=$?"
python tools/attn_pp_trace.py gpurun_out/g75_trace.bin 2>&1 | grep "epilogue item" | head -4
rm -f paper_2509_13523_b200/_build_variants/trace.so
bash tools/gpurun/gpu_var_cycles.sh g75 attention k_attn_pp
