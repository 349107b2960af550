"""Experiment helper: one fused query with long documents (v_r, lengths from argv) for
compute-sanitizer runs.  python tools/cta_repro.py V_R LEN [LEN ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

v_r = int(sys.argv[1])
lengths = []
for x in sys.argv[2:] or ["100", "200", "300"]:
    L, _, cnt = x.partition("*")
    lengths += [int(L)] * int(cnt or 1)
rng = np.random.default_rng(0)
V, d = 5000, 64
E = rng.standard_normal((V, d)).astype(np.float32)
docs = []
for L in lengths:
    ids = rng.choice(V, L, replace=False)
    cnt = rng.geometric(0.3, L).astype(np.float64)
    docs.append({int(k): float(x) for k, x in zip(ids, (cnt / cnt.sum()).astype(np.float32))})
cp, ri, va = synth.csc_from_lists(docs, V)
q = np.sort(rng.choice(V, v_r, replace=False)).astype(np.int32)
w = np.full(v_r, 1.0 / v_r, np.float32)
h = wmd.wmd_create(E)
wmd.wmd_set_targets(h, cp, ri, va)
if os.environ.get("NOFB"):
    wmd.wmd_set_option(h, wmd.WMD_OPT_FALLBACK, 0)
out = np.empty(len(lengths), np.float32)
wmd.wmd_query(h, q, w, 10.0, 30, out)
wmd.wmd_sync(h)
print(out[:4], np.isfinite(out).all(), "flagged", int(np.count_nonzero(wmd.wmd_read_flags(h, len(lengths)))), wmd.wmd_get_stats(h)["last_path"], wmd.wmd_get_stats(h)["last_ld"])
