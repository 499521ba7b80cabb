# one ncu --set full capture of the kernels matching $1 (after the same command ran clean)
K=${1:-k_gemm_tc}; T=${2:-ncuk}
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_plain.log 2>&1; rc=$?; echo "plain rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${3:-9} -c ${4:-6} \
    -o gpurun_out/${T} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
