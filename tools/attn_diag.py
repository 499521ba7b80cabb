"""Attention self-test diagnostics: per (window, head, 16-row block) max |err| of the kernel vs float64,
to localise wrong rows (tails, seam boundaries). Usage: python tools/attn_diag.py [nwin heads w shift sharp]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_13523_b200 as swf  # noqa: E402
from tests.test_gpu_attention import make_qkv, reference  # noqa: E402

n_wy, heads, w, shift, sharp = (int(a) for a in (sys.argv[1:] + ["1", "2", "60", "0", "0"][len(sys.argv) - 1:]))
q, k, v = make_qkv(n_wy, heads, w * w, 128, 11, sharp=bool(sharp))
ref = reference(q, k, v, n_wy, 1, w, shift)
got = swf.selftest_attention(q, k, v, n_wy, 1, w, shift)
s, d = w * w, 128
print(f"kernel={os.environ.get('SWF_ATTN', 'default')} n_wy={n_wy} heads={heads} w={w} shift={shift} sharp={sharp}")
for win in range(n_wy):
    for hh in range(heads):
        e = np.abs(got[win, :, hh * d:(hh + 1) * d] - ref[win, :, hh * d:(hh + 1) * d]).max(axis=1)
        sc = np.abs(ref[win, :, hh * d:(hh + 1) * d]).max()
        blocks = e.reshape(-1, 16).max(axis=1) / sc if s % 16 == 0 else e / sc
        bad = np.nonzero(blocks > 2e-2)[0]
        print(f"  win {win} head {hh}: max rel {blocks.max():.3e}; bad 16-row blocks: {bad.tolist()[:40]}")
