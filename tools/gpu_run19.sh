timeout 300 python tools/kbench.py 10 gateup_gemm,down_gemm,qkv_gemm,out_gemm > gpurun_out/r19_kbench.log 2>&1; cat gpurun_out/r19_kbench.log | tail -4
timeout 300 python tools/kbench.py 1 gateup_gemm,down_gemm > gpurun_out/r19_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemm_tc -s 82 -c 4 --csv python tools/kbench.py 1 gateup_gemm,down_gemm > gpurun_out/r19_ncu.csv 2>&1; echo "ncu rc=$?"
grep -E "k_gemm_tc" gpurun_out/r19_ncu.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -30
