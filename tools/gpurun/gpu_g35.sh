cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/bwd_once.py 120 240 > gpurun_out/g35_bwd_launches.csv 2> gpurun_out/g35.err; echo "rc=$?"
python - <<'PY'
import csv, io, collections
t = open('gpurun_out/g35_bwd_launches.csv').read(); i = t.find('"ID"')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in csv.DictReader(io.StringIO(t[i:])):
    if r["Metric Name"] != "gpu__time_duration.sum": continue
    k = r["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1][:50]
    v = float(r["Metric Value"].replace(",", "")); u = r["Metric Unit"]
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1e-6)
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} ms")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{ms:9.2f} ms {100*ms/tot:5.1f}%  n={n:4d}  {k}")
PY
