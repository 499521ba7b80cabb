cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/g62_t.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/g62_t.log
bash tools/gpurun/gpu_var_cycles.sh g62 attention k_attn_pp
