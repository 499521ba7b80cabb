cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc" -s 2 -c 1 \
    -o gpurun_out/g50_out -f python tools/kbench.py 2 out_gemm > gpurun_out/g50_ncu.log 2>&1; echo "ncu rc=$?"
