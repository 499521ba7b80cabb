# GEMM weight-operand L2 policy: evict_last (b_last, current) vs evict_normal (b_normal), base-clock cycles and
# DRAM bytes of the forward GEMMs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpurun/gpu_var_cycles.sh g103 qkv_gemm,out_gemm,gateup_gemm,down_gemm 'k_gemm_tc' > /dev/null 2>&1
cat gpurun_out/g103_cyc.log
