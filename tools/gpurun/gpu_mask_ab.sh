# Full-bench A/B of per-mode static GEMM schedules (SWF_GEMM_STATIC_MASK), alternating, twice.
T=${1:-mask}; M=${2:-8}
for rep in 1 2; do
  for m in 0 $M; do
    SWF_GEMM_STATIC_MASK=$m timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${T}_m${m}_$rep.log 2>&1
    echo "mask $m rep $rep rc=$? $(tail -1 gpurun_out/${T}_m${m}_$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), "ms", d["clocks"]["sm_mhz"], "MHz", {k: round(v["ms_per_launch"],2) for k,v in d["kernels"].items() if "gemm" in k or k=="attention"})')"
  done
done
