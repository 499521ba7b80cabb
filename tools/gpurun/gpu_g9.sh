cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g9_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/g9_bench.log | tail -1 | head -c 3000; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attn_pp" -s 1 -c 1 \
    -o gpurun_out/g9_attn -f python tools/kbench.py 2 attention > gpurun_out/g9_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/g9_attn.ncu-rep --page details > gpurun_out/g9_attn_details.txt 2>&1
ncu -i gpurun_out/g9_attn.ncu-rep --page raw --csv > gpurun_out/g9_attn_raw.csv 2>&1
grep -E "Duration|SM Frequency|Tensor|Issue Slots|Stall|Throughput|Eligible|Active Warps" gpurun_out/g9_attn_details.txt | head -60
