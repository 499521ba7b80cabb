cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/trace.so SWF_ATTN_TRACE_OUT=gpurun_out/g74_trace.bin timeout 300 python tools/kbench.py 2 attention > gpurun_out/g74_k.log 2>&1; echo "trace rc=$?"
python tools/attn_pp_trace.py gpurun_out/g74_trace.bin 2>&1 | tail -14
