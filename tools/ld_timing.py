"""Fused-phase time per query of the Many config by table width, half-warp vs one-warp kernel
(experiment helper).   python tools/ld_timing.py [reps]
One JSON line per (query width class, kernel): fused ms per query from the library's events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = synth.make_workload("many")
by_ld = {}
for q, w in wl.queries:
    by_ld.setdefault(-(-q.shape[0] // 8) * 8, (q, w))
h = wmd.wmd_create(wl.E)
wmd.wmd_set_option(h, wmd.WMD_OPT_PATH, wmd.WMD_PATH_FUSED)
wmd.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
out = np.empty(wl.N, np.float32)
for ld in sorted(by_ld):
    q, w = by_ld[ld]
    for half in ("0", "1"):
        os.environ["WMD_FUSED_HALF"] = half
        wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 0)
        wmd.wmd_query(h, q, w, 10.0, 15, out)
        wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 1)
        wmd.wmd_reset_stats(h)
        for _ in range(reps):
            wmd.wmd_query(h, q, w, 10.0, 15, out)
        wmd.wmd_sync(h)
        st = wmd.wmd_get_stats(h)
        print(json.dumps({"v_r": int(q.shape[0]), "ld": int(st["last_ld"]), "half": half == "1",
                          "fused_ms": st["iter_ms"] / reps, "query_ms": st["query_ms"] / reps}), flush=True)
wmd.wmd_destroy(h)
