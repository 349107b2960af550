"""Time one workload's query phases through the C ABI (experiment helper; not the bench).

    python tools/pass_timing.py [config] [path: iter|fused|auto] [queries] [iters,iters,...]
Prints one JSON line per iteration count with per-phase ms per query (CUDA events inside the
library); several iteration counts separate a fused kernel's per-document fixed cost (setup,
staging, final step) from its per-iteration cost.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "scaling"
path = {"iter": wmd.WMD_PATH_PER_ITER, "fused": wmd.WMD_PATH_FUSED, "auto": wmd.WMD_PATH_AUTO}[
    sys.argv[2] if len(sys.argv) > 2 else "iter"]
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 5
wl = synth.make_workload(cfgname, n_queries=1)
iters_list = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [wl.cfg.iters]
q, w = wl.queries[0]
h = wmd.wmd_create(wl.E)
wmd.wmd_set_option(h, wmd.WMD_OPT_PATH, path)
wmd.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
out = np.empty(wl.N, np.float32)
for iters in iters_list:
    for _ in range(2):
        wmd.wmd_query(h, q, w, wl.cfg.lam, iters, out)
    wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 1)
    wmd.wmd_reset_stats(h)
    for _ in range(nq):
        wmd.wmd_query(h, q, w, wl.cfg.lam, iters, out)
    wmd.wmd_sync(h)
    st = wmd.wmd_get_stats(h)
    res = {k: st[k] / nq for k in ("build_ms", "iter_ms", "final_ms", "fallback_ms", "query_ms")}
    res["iter_launch_ms"] = st["iter_ms"] / max(1, st["iter_launches"])
    res["lib"] = os.path.basename(wmd.LIB_PATH)
    res["config"] = cfgname
    res["iters"] = iters
    res["fallback_docs_per_query"] = st["fallback_docs"] / nq
    res["checksum"] = float(np.sum(out.astype(np.float64)))
    print(json.dumps(res), flush=True)
    wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 0)
wmd.wmd_destroy(h)
