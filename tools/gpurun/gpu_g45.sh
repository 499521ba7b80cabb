cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpurun/gpu_var_cycles.sh g45 attention k_attn_pp
