# A/B of library build variants (paper_2509_13523_b200/_build/var/lib_*.so via SWF_LIB): kernel
# isolation of the GEMM classes and ncu tensor-pipe activity. usage: bash tools/gpurun/gpu_libvar_ab.sh TAG
T=${1:-var}
for lib in paper_2509_13523_b200/_build/var/lib_*.so; do
  v=$(basename $lib .so)
  SWF_LIB=$PWD/$lib timeout 300 python tools/kbench.py 20 gateup_gemm,down_gemm,qkv_gemm,out_gemm > gpurun_out/${T}_${v}_k.log 2>&1
  echo "== $v rc=$?"; grep -o '^[a-z_]* {"ms": [0-9.]*\|J_per_launch": [0-9.]*' gpurun_out/${T}_${v}_k.log | paste - -
  SWF_LIB=$PWD/$lib timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum \
    --clock-control none -k "regex:k_gemm_tc" -s 6 -c 4 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_${v}_ncu.csv 2>&1
done
