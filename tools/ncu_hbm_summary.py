"""Summarise an ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum) of the
HBM-bound kernels: per kernel name, launches, median duration, DRAM bytes per launch and achieved
DRAM GB/s against the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs).
usage: python tools/ncu_hbm_summary.py <csv> [peak_gbs]"""
import collections
import csv
import io
import re
import sys

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.4
t = open(path, errors="replace").read()
rows = list(csv.DictReader(io.StringIO(t[t.find('"ID"'):])))
per = collections.defaultdict(lambda: collections.defaultdict(dict))
for r in rows:
    name = re.sub(r"\(.*$", "", r["Kernel Name"]).replace("swf::(anonymous namespace)::", "").replace("swf::", "")
    unit, v = r.get("Metric Unit", ""), float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        v = v * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)
    elif "bytes" in r["Metric Name"]:
        v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per[name][r["ID"]][r["Metric Name"]] = v
print(f"# {'kernel':32s} {'launches':>8s} {'median_us':>10s} {'DRAM MB/launch':>15s} {'GB/s':>8s} {'frac':>6s}")
for name, launches in sorted(per.items()):
    ds, bs = [], []
    for m in launches.values():
        d = m.get("gpu__time_duration.sum")
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if d:
            ds.append(d)
            bs.append(b)
    if not ds:
        continue
    i = sorted(range(len(ds)), key=lambda k: ds[k])[len(ds) // 2]
    gbs = bs[i] / ds[i] / 1e9
    print(f"  {name:32s} {len(ds):8d} {ds[i] * 1e6:10.1f} {bs[i] / 1e6:15.1f} {gbs:8.0f} {gbs / peak:6.2f}")
