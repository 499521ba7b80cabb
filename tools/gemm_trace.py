"""Summarise the GEMM MMA-thread trace (development build -DSWF_GEMM_TRACE, SWF_GEMM_TRACE_OUT=path):
per launch (epilogue mode), per tile of cluster 0: tile-queue wait, accumulator-free wait, operand
(full-barrier) waits, and the remaining issue / pipe time. usage: python tools/gemm_trace.py TRACE"""
import sys

import numpy as np

N = 2048
raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
rec = 1 + 5 * N
names = {1: "QKV", 2: "out", 3: "gate/up", 4: "down", 0: "encode", 5: "decode"}
for k in range(len(raw) // rec):
    r = raw[k * rec:(k + 1) * rec]
    tag, t = int(r[0]), r[1:].reshape(5, N)
    n = int(np.argmin(t[3] > 0)) if (t[3] == 0).any() else N  # tiles recorded (contiguous from 0)
    if n < 4:
        continue
    i = np.arange(1, n)
    tile = t[3][i] - t[0][i]
    q = t[1][i] - t[0][i]
    te = t[2][i] - t[1][i]
    fw = t[4][i]
    rest = tile - q - te - fw
    gap = t[0][i] - t[3][i - 1]
    med = lambda a: float(np.median(a))  # noqa: E731
    print(f"{names.get(tag // 1000, tag)} (BN {tag % 1000}): {n} tiles; per tile median cycles: total {med(tile + gap):.0f} = "
          f"queue {med(q):.0f} + acc-free wait {med(te):.0f} + operand waits {med(fw):.0f} + MMA issue {med(rest):.0f} "
          f"+ gap {med(gap):.0f}; mean operand wait {np.mean(fw):.0f}, p90 {np.percentile(fw, 90):.0f}")
