cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/g28_t.log 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/g28_t.log
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/trace.so SWF_ATTN_TRACE_OUT=gpurun_out/g28_trace.bin timeout 300 python tools/kbench.py 2 attention > gpurun_out/g28_k.log 2>&1; echo "trace rc=$?"
python tools/attn_pp_trace.py gpurun_out/g28_trace.bin
rm -f paper_2509_13523_b200/_build_variants/trace.so
bash tools/gpurun/gpu_var_cycles.sh g28 attention k_attn_pp
