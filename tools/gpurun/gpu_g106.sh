# out-projection residual L2 prefetch on (x_on, current) vs off (x_off) with the 16-byte epilogue
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpurun/gpu_var_cycles.sh g106 out_gemm 'k_gemm_tc' > /dev/null 2>&1
cat gpurun_out/g106_cyc.log
