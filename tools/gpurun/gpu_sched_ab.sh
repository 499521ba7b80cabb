# Dynamic vs static GEMM tile schedule: GEMM self-test + parity, kernel isolation A/B (time, energy),
# full bench A/B, and an ncu DRAM-traffic check of the down GEMM under both schedules.
T=${1:-sched}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
bash tools/gpurun/gpu_ab.sh ${T}_k SWF_GEMM_STATIC
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_dyn.log 2>&1; echo "bench dyn rc=$?"; tail -1 gpurun_out/${T}_bench_dyn.log | cut -c1-400
SWF_GEMM_STATIC=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_static.log 2>&1; echo "bench static rc=$?"; tail -1 gpurun_out/${T}_bench_static.log | cut -c1-400
for v in dyn static; do
  if [ $v = static ]; then export SWF_GEMM_STATIC=1; else unset SWF_GEMM_STATIC; fi
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k "regex:k_gemm_tc" -s 6 -c 6 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_$v.csv 2>&1; echo "ncu $v rc=$?"
done
