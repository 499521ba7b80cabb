cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "1 2 60 0 0" "2 2 60 30 1" "2 4 8 4 1" "1 2 12 6 1"; do
  timeout 120 python tools/attn_diag.py $args >> gpurun_out/g20_diag.log 2>&1 || echo "rc=$? ($args)" >> gpurun_out/g20_diag.log
done
grep -E "kernel|max rel" gpurun_out/g20_diag.log | awk '{print}' | head -30
for v in nopf pf pfp3 pfp1; do
  SWF_LIB=paper_2509_13523_b200/_build_variants/$v.so timeout 300 ncu --clock-control base -k regex:"k_attn_pp" -s 2 -c 8 \
    --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --csv python tools/kbench.py 3 attention > gpurun_out/g20_$v.csv 2>/dev/null
  echo "== $v" >> gpurun_out/g20_cyc.log
  python - gpurun_out/g20_$v.csv >> gpurun_out/g20_cyc.log <<'PY'
import csv, io, sys, collections
t = open(sys.argv[1]).read(); i = t.find('"ID"')
agg = collections.defaultdict(list)
for r in csv.DictReader(io.StringIO(t[i:])):
    agg[r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
for m, v in sorted(agg.items()):
    print(f"  {m:70s} n={len(v):3d} median={sorted(v)[len(v)//2]:.4g}")
PY
done
cat gpurun_out/g20_cyc.log
