"""Summarise the attention pipeline trace of CTA 0 (development build: make EXTRA=-DSWF_ATTN_TRACE,
SWF_ATTN_TRACE_OUT=path). Per key tile g: 0 S ready, 1 row max exchanged, 2 P stores issued,
3 P stored, 4 P seen by the MMA issuer, 5 P V issued; per item n: 6 MMA saw Q, 7 MMA saw O free,
8 epilogue start, 9 epilogue end."""
import sys

import numpy as np

T = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(2, 2, -1, 1024).astype(np.int64)
cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
t = T[0][cta]
W = T[1][cta]  # per softmax warp: rows 0-7 S ready, 8-15 P done
gg = np.arange(8, 200)
print("per-warp S ready rel. warp4:", [float(np.median(W[w][gg] - W[0][gg])) for w in range(8)])
print("per-warp P done rel. warp4 S ready:", [float(np.median(W[8 + w][gg] - W[0][gg])) for w in range(8)])
ntile = int(sys.argv[2]) if len(sys.argv) > 2 else 29
lo, hi = 8, 200
med = lambda a: float(np.median(a))  # noqa: E731
sl = slice(lo, hi)
period = np.diff(t[0][lo:hi + 1])
print(f"period {med(period):.0f} (p90 {np.percentile(period, 90):.0f}, max {period.max()})  "
      f"ld+max+xchg {med((t[1] - t[0])[sl]):.0f}  exp {med((t[2] - t[1])[sl]):.0f}  st-wait {med((t[3] - t[2])[sl]):.0f}  "
      f"P->MMA {med((t[4] - t[3])[sl]):.0f}  PV issue {med((t[5] - t[4])[sl]):.0f}  "
      f"P(g) done -> S(g+1) ready {med(t[0][lo + 1:hi + 1] - t[3][sl]):.0f}")
big = np.nonzero(period > 2 * med(period))[0]
print("long periods at tiles", (big + lo).tolist()[:12], "values", period[big].tolist()[:12])
for n in range(1, 6):
    last = ntile * n - 1
    base = t[0][last]
    print(f"item {n}: MMA saw Q {t[6][n] - base}, MMA saw O free {t[7][n] - base}, "
          f"epi [{t[8][n - 1] - base}, {t[9][n - 1] - base}], next S ready {t[0][last + 1] - base}")
if t.shape[0] >= 16:
    g = np.arange(lo, hi)
    print(f"MMA warp (rel. to S(g) ready): S(g+1) entry {med(t[10][g + 1] - t[0][g]):.0f}, K(g+1) landed "
          f"{med(t[11][g + 1] - t[0][g]):.0f}, S(g+1) issued {med(t[12][g + 1] - t[0][g]):.0f}, "
          f"PV(g) entry {med(t[13][g] - t[0][g]):.0f}, P(g) seen {med(t[14][g] - t[0][g]):.0f}, "
          f"P(g) done {med(t[3][g] - t[0][g]):.0f}, PV(g) issued {med(t[5][g] - t[0][g]):.0f}, "
          f"S(g+1) ready {med(t[0][g + 1] - t[0][g]):.0f}")
