timeout 300 python tools/clockseq.py attention,gateup_gemm,attention,down_gemm,attention,qkv_gemm,attention,attention 3 > gpurun_out/r18_seq.log 2>&1; cat gpurun_out/r18_seq.log | tail -9
python - <<'PY'
rows=[l.strip().split(", ") for l in open("gpurun_out/clockseq_smi.csv") if "MHz" in l]
import statistics
c=[int(r[1].split()[0]) for r in rows]; p=[float(r[2].split()[0]) for r in rows]
print("samples", len(c), "clock min/med/max", min(c), statistics.median(c), max(c), "power med/max", statistics.median(p), max(p))
# print a compressed trace: every 10th sample
print(" ".join(f"{c[i]}" for i in range(0, len(c), 5)))
PY
