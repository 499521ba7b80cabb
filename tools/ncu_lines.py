"""Per-CUDA-source-line stall breakdown of one kernel in an ncu report (--import-source on):
warp-stall samples, executed instructions and the top stall reasons per line.
usage: python tools/ncu_lines.py REPORT.ncu-rep [N_LINES] [LAUNCH_INDEX]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sel = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"] + sel,
                     capture_output=True, text=True).stdout


def num(x):
    try:
        return int(x)
    except ValueError:
        return None


agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
hdr, fname = None, None
for r in csv.reader(io.StringIO(out)):
    if not r or r[0] == "Function Name":
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or num(r[0]) is None or len(r) != len(hdr):
        continue
    key = (fname, int(r[0]), r[1].strip()[:70])
    agg[key][0] += num(r[4]) or 0
    agg[key][1] += num(r[7]) or 0
    for i, c in enumerate(hdr):
        if c.startswith("stall_") and "(Not" not in c and num(r[i]):
            agg[key][2][c] += int(r[i])
tot = sum(v[0] for v in agg.values()) or 1
tote = sum(v[1] for v in agg.values()) or 1
print(f"# {rep}: {tot} stall samples, {tote} warp instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = ", ".join(f"{a[6:]}:{b * 100 // max(v[0], 1)}" for a, b in v[2].most_common(3))
    print(f"{v[0] / tot * 100:5.1f}% st {v[1] / tote * 100:5.1f}% ex  {k[0]}:{k[1]} {k[2]!r}  [{top}]")
