"""Pipeline trace of the ping-pong attention kernel (k_attn_pp), CTA 0 of cluster 0 (development build:
tools/build_variant.sh NAME "" -DSWF_ATTN_TRACE, run with SWF_ATTN_TRACE_OUT=path). clock64 stamps per
global key tile g: S issuer 10 entry / 11 K landed / 12 ring slot free (= S issued); P V issuer 13 entry /
14 P seen / 15 V landed (= P V issued); softmax warp w: S ready (w), S in registers (8 + w), P handed
over (16 + w); per item n: 6 S issuer saw Q, 7 P V issuer saw O free, 8 epilogue start, 9 epilogue end.
usage: python tools/attn_pp_trace.py TRACE NTILES_PER_ITEM"""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
N = 1024
t = raw[:2 * 16 * N].reshape(2, 16, N)[0]
w = raw[2 * 16 * N:].reshape(2, 32, N)[0]
starts = t[1]  # global tile index at each item's start (S issuer)
z = np.nonzero(starts[1:] == 0)[0]
nitems = int(z[0]) + 1 if len(z) else N
item_of_g = np.searchsorted(starts[:nitems], np.arange(N), side="right") - 1
lo, hi = int(starts[1]), int(min(starts[min(8, nitems)], N - 8))  # skip the first item (cold)
g = np.arange(lo, hi)
nt = int(starts[2] - starts[1])
med = lambda a: float(np.median(a))  # noqa: E731
p90 = lambda a: float(np.percentile(a, 90))  # noqa: E731
grp = g % 2  # within an item tile j's group is j % 2; items have nt tiles (odd nt flips parity per item)
# softmax warp of tile g: group = (g - item_start) % 2, quadrant 0 -> warp 4 + 4 * group
item_start = starts[item_of_g[g]]
wg = 4 * ((g - item_start) % 2)  # row index (warp - 4) of quadrant-0 warp of that group
s_ready = w[wg, g]
s_regs = w[8 + wg, g]
p_done = w[16 + wg, g]
s_issue = t[12, g]
pv_issue = t[15, g]
print(f"tiles {lo}..{hi}, period (S issue) med {med(np.diff(s_issue)):.0f}  mean {np.mean(np.diff(s_issue)):.0f}")
print(f"S issue -> S ready (softmax)      med {med(s_ready - s_issue):6.0f}  p90 {p90(s_ready - s_issue):6.0f}")
print(f"S ready -> S in registers         med {med(s_regs - s_ready):6.0f}  p90 {p90(s_regs - s_ready):6.0f}")
print(f"S in regs -> P handed over        med {med(p_done - s_regs):6.0f}  p90 {p90(p_done - s_regs):6.0f}")
print(f"P handed over -> PV issuer sees P med {med(t[14, g] - p_done):6.0f}  p90 {p90(t[14, g] - p_done):6.0f}")
print(f"PV issuer entry -> P seen (wait)  med {med(t[14, g] - t[13, g]):6.0f}  p90 {p90(t[14, g] - t[13, g]):6.0f}")
print(f"P seen -> V landed (PV issued)    med {med(pv_issue - t[14, g]):6.0f}  p90 {p90(pv_issue - t[14, g]):6.0f}")
gg = g[g + 4 < hi]
print(f"PV(g) issued -> S(g+4) issued     med {med(t[12, gg + 4] - t[15, gg]):6.0f}  p90 {p90(t[12, gg + 4] - t[15, gg]):6.0f}")
print(f"S issuer entry -> K landed        med {med(t[11, g] - t[10, g]):6.0f}  p90 {p90(t[11, g] - t[10, g]):6.0f}")
print(f"K landed -> slot free (S issued)  med {med(t[12, g] - t[11, g]):6.0f}  p90 {p90(t[12, g] - t[11, g]):6.0f}")
# softmax warp idle: from its P handed over (tile g) to S ready of its next tile (g + 2, same item)
same = (g + 2 < hi) & (item_of_g[np.minimum(g + 2, N - 1)] == item_of_g[g])
g2 = g[same]
wg2 = wg[same]
print(f"softmax: P(g) done -> S(g+2) ready med {med(w[wg2, g2 + 2] - w[16 + wg2, g2]):6.0f}  "
      f"p90 {p90(w[wg2, g2 + 2] - w[16 + wg2, g2]):6.0f}  (negative = S was already there)")
busy = np.maximum(0, w[wg2, g2 + 2] - w[16 + wg2, g2])
print(f"softmax per own tile: work {med(p_done - s_regs) + med(s_regs - s_ready):.0f}, wait for S {np.mean(busy):.0f} (mean)")
for n in range(1, 7):
    if t[5, n]:
        print(f"  epilogue item {n}: stats exchange {t[2, n] - t[8, n]}, last P V wait {t[3, n] - t[2, n]}, "
              f"O read / merge / stage {t[4, n] - t[3, n]}, sync {t[5, n] - t[4, n]}, store issue + rest {t[9, n] - t[5, n]}")
    print(f"item {n}: epilogue {t[9, n] - t[8, n]} cyc; PV issuer saw O free {t[7, n] - t[9, n - 1] if n else 0} after "
          f"prev epilogue end; first S ready of item {w[0, starts[n]] - t[8, n - 1]} after prev epilogue start; tiles {starts[n + 1] - starts[n]}")
# per-quadrant skew of S ready / P done for one tile
g0t = g[(g - item_start) % 2 == 0]
print("P done skew over the 4 warps of group 0 (max - min):", med(np.max(w[16:20, g0t], 0) - np.min(w[16:20, g0t], 0)))
