"""Repro helper: one fused query at a given lambda on the Long config's first N documents (or the
Tweet documents against the Long query with "short", or N documents of LO-HI words), reporting
the last error.

    python tools/small_lambda_repro.py LAMBDA [N] [short | LO-HI]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

lam = float(sys.argv[1])
N = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
wl = synth.make_workload("long", N=N)
q, w = wl.queries[0]
cp, ri, va = wl.col_ptr, wl.row_idx, wl.val
if "short" in sys.argv[3:]:
    s = synth.make_workload("tweet", N=2000)
    cp, ri, va = s.col_ptr, s.row_idx, s.val
for a in sys.argv[3:]:
    if "-" in a:  # LO-HI: N documents of LO..HI words
        lo, hi = (int(x) for x in a.split("-"))
        rng = np.random.Generator(np.random.PCG64(5))
        cp, ri, va = synth.make_corpus(rng, wl.cfg.V, N, lo, hi, 1.07, 0.3)
h = wmd.wmd_create(wl.E)
wmd.wmd_set_targets(h, cp, ri, va)
d = np.empty(cp.shape[0] - 1, np.float32)
try:
    wmd.wmd_query(h, q, w, lam, 10, d)
    wmd.wmd_sync(h)
    print(lam, N, d[:4], wmd.wmd_get_stats(h)["last_ld"], flush=True)
except Exception as e:
    print(lam, N, "ERROR", e, flush=True)
