# attention A/B: split (round-1) vs ping-pong kernel, isolated and in-step (C2, live weights)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in split default; do
  echo "== $k" >> gpurun_out/g6_ab.log
  SWF_ATTN=$k timeout 300 python tools/kbench.py 10 attention >> gpurun_out/g6_ab.log 2>&1
  SWF_ATTN=$k timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g6_bench_$k.log 2>&1
  grep '^{' gpurun_out/g6_bench_$k.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('bench', d['value'], d['ms_per_step'], json.dumps({k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}), d['clocks'])" >> gpurun_out/g6_ab.log
done
cat gpurun_out/g6_ab.log
