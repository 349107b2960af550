"""Experiment helper: the Long workload restricted to its first NDOCS documents, one fused query;
prints the checksum, flagged count and max relative difference to the per-iteration path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
wl = synth.make_workload("long", n_queries=1)
docs = np.arange(nd)
cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
q, w = wl.queries[0]
res = {}
for path in (wmd.WMD_PATH_FUSED, wmd.WMD_PATH_PER_ITER):
    h = wmd.wmd_create(wl.E)
    wmd.wmd_set_option(h, wmd.WMD_OPT_PATH, path)
    wmd.wmd_set_targets(h, cp, ri, va)
    if os.environ.get("NOFB"):
        wmd.wmd_set_option(h, wmd.WMD_OPT_FALLBACK, 0)
    out = np.empty(nd, np.float32)
    wmd.wmd_query(h, q, w, wl.cfg.lam, wl.cfg.iters, out)
    wmd.wmd_sync(h)
    st = wmd.wmd_get_stats(h)
    res[path] = out.astype(np.float64)
    bad = np.nonzero(~np.isfinite(out))[0]
    fl = wmd.wmd_read_flags(h, nd)
    print(path, "flagged", int(np.count_nonzero(fl)), np.nonzero(fl)[0][:10], "lengths", np.diff(cp)[np.nonzero(fl)[0][:10]])
    print(path, "non-finite", bad.size, bad[:10], "lengths", np.diff(cp)[bad[:10]])
    print(path, "checksum", out.astype(np.float64).sum(), "fallback docs", st["fallback_docs"], flush=True)
    wmd.wmd_destroy(h)
a, b = res[wmd.WMD_PATH_FUSED], res[wmd.WMD_PATH_PER_ITER]
print("max rel diff fused vs per-iter", np.max(np.abs(a - b) / np.abs(b)))
