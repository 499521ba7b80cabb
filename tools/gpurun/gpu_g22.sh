cd $GRAFT_REPO_ROOT
bash tools/gpurun/gpu_hbm.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc" -s 22 -c 4 \
    -o gpurun_out/g22_gemm -f python tools/kbench.py 2 qkv_gemm > gpurun_out/g22_ncu.log 2>&1; echo "ncu gemm rc=$?"
for id in 0 1 2 3; do
  ncu -i gpurun_out/g22_gemm.ncu-rep --page details --launch-skip $id --launch-count 1 2>/dev/null | grep -E "k_gemm_tc|Duration|Tensor|Issue Slots|Eligible|DRAM Throughput|Memory Throughput" | head -8
done
