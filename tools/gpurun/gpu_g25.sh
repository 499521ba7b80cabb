cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn_pp" -s 2 -c 1 \
    -o gpurun_out/g25_attn -f python tools/kbench.py 2 attention > gpurun_out/g25_ncu.log 2>&1; echo "ncu attn rc=$?"
