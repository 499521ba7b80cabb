# Variant A/B at locked base clocks: for every paper_2509_13523_b200/_build_variants/*.so, ncu
# --clock-control base over kbench's kernel classes (median of the launches), then kernel isolation
# at free clocks (ms, J/launch). usage: bash tools/gpurun/gpu_var_cycles.sh TAG CLASSES KERNEL_REGEX
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-var}; CL=${2:-out_gemm,down_gemm}; KR=${3:-k_gemm_tc}
for lib in paper_2509_13523_b200/_build_variants/*.so; do
  v=$(basename $lib .so)
  SWF_LIB=$PWD/$lib timeout 400 ncu --clock-control base -k regex:"$KR" -s 2 -c 40 \
    --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv python tools/kbench.py 3 $CL > gpurun_out/${T}_$v.csv 2>/dev/null
  echo "== $v (ncu rc=$?)" >> gpurun_out/${T}_cyc.log
  python - gpurun_out/${T}_$v.csv >> gpurun_out/${T}_cyc.log <<'PY'
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
for rep in 1 2; do
  for lib in paper_2509_13523_b200/_build_variants/*.so; do
    v=$(basename $lib .so)
    SWF_LIB=$PWD/$lib timeout 300 python tools/kbench.py 20 $CL > gpurun_out/${T}_${v}_k$rep.log 2>&1
    echo "$v rep$rep rc=$? $(grep -o '^[a-z_]* {"ms": [0-9.]*\|J_per_launch": [0-9.]*\|"sm_mhz": [0-9.]*' gpurun_out/${T}_${v}_k$rep.log | tr '\n' ' ')" >> gpurun_out/${T}_cyc.log
  done
done
cat gpurun_out/${T}_cyc.log
