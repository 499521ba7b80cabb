# in-step (power-capped) A/B of the attention's polynomial-exp share: full C2 bench per library variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in p1 p2; do
    SWF_LIB=$PWD/paper_2509_13523_b200/_build_variants/$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/g51_${v}_$rep.log 2>&1
    tail -1 gpurun_out/g51_${v}_$rep.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$v rep$rep', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], 'attn', round(k['attention']['ms_per_launch'],2), 'gateup', round(k['gateup_gemm']['ms_per_launch'],2))"
  done
done
