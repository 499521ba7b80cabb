# attention variants: correctness (diag) + cycle counts at locked base clocks (ncu --clock-control base)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "1 2 60 0 0" "2 2 60 30 1" "2 4 8 4 1"; do
  timeout 120 python tools/attn_diag.py $args >> gpurun_out/g11_diag.log 2>&1 || echo "rc=$? ($args)" >> gpurun_out/g11_diag.log
done
cat gpurun_out/g11_diag.log
for v in spec0 spec1 spec1p1 spec1p3 pb40 oldqkv; do
  SWF_LIB=paper_2509_13523_b200/_build_variants/$v.so timeout 300 ncu --clock-control base -k regex:"k_attn_pp|k_gemm_tc" -s 2 -c 40 \
    --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --csv python tools/kbench.py 3 attention,qkv_gemm > gpurun_out/g11_$v.csv 2>/dev/null
  echo "== $v" >> gpurun_out/g11_cyc.log
  python - gpurun_out/g11_$v.csv >> gpurun_out/g11_cyc.log <<'PY'
import csv, io, sys, collections
t = open(sys.argv[1]).read(); i = t.find('"ID"')
agg = collections.defaultdict(list)
for r in csv.DictReader(io.StringIO(t[i:])):
    k = r["Kernel Name"].split("(")[0].split("::")[-1][:40]
    agg[(k, r["Metric Name"])].append(float(r["Metric Value"].replace(",", "")))
for (k, m), v in sorted(agg.items()):
    print(f"  {k:40s} {m:70s} n={len(v):3d} median={sorted(v)[len(v)//2]:.4g}")
PY
done
cat gpurun_out/g11_cyc.log
