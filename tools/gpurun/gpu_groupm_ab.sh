# GEMM rasterisation band height (SWF_GEMM_GROUPM) under the dynamic schedule: kernel isolation
# (time, J/launch) per value, then the full bench for the best candidates.
T=${1:-gm}
for g in 1 2 4 8; do
  SWF_GEMM_GROUPM=$g timeout 300 python tools/kbench.py 20 gateup_gemm,down_gemm,qkv_gemm,out_gemm > gpurun_out/${T}_k$g.log 2>&1
  echo "== groupm $g rc=$?"; grep -o '^[a-z_]* {"ms": [0-9.]*\|J_per_launch": [0-9.]*' gpurun_out/${T}_k$g.log | paste - - 
done
for g in ${2:-1 4}; do
  SWF_GEMM_GROUPM=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench$g.log 2>&1
  echo "bench groupm $g rc=$?"; tail -1 gpurun_out/${T}_bench$g.log | cut -c1-200
done
