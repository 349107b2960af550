"""Time the distance build (a2) of each build kernel on the configs (experiment helper).

    python tools/build_timing.py [config,config,...] [queries]
One JSON line per (config, build kernel): build_ms per query from the library's CUDA events
(fused path, 1 iteration: the build is the phase of interest), the table checksum of the first
query's distances, and the max |difference| of the WMDs against the direct-difference build.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tweet", "many", "long", "scaling"]
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10
names = {wmd.WMD_BUILD_DIRECT: "direct", wmd.WMD_BUILD_TENSOR_CORE: "tf32x3", wmd.WMD_BUILD_EXACT: "exact"}
for cfgname in cfgs:
    wl = synth.make_workload(cfgname, n_queries=1)
    q, w = wl.queries[0]
    h = wmd.wmd_create(wl.E)
    wmd.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
    out = np.empty(wl.N, np.float32)
    ref = None
    for b in (wmd.WMD_BUILD_DIRECT, wmd.WMD_BUILD_TENSOR_CORE, wmd.WMD_BUILD_EXACT):
        wmd.wmd_set_option(h, wmd.WMD_OPT_BUILD, b)
        wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 0)
        for _ in range(2):
            wmd.wmd_query(h, q, w, wl.cfg.lam, wl.cfg.iters, out)
        wmd.wmd_sync(h)
        d = out.astype(np.float64).copy()
        if ref is None:
            ref = d
        wmd.wmd_set_option(h, wmd.WMD_OPT_TIMING, 1)
        wmd.wmd_reset_stats(h)
        for _ in range(nq):
            wmd.wmd_query(h, q, w, wl.cfg.lam, 1, out)
        wmd.wmd_sync(h)
        st = wmd.wmd_get_stats(h)
        print(json.dumps({"config": cfgname, "build": names[b], "build_ms": st["build_ms"] / nq,
                          "v_r": int(np.unique(q).shape[0]), "V": wl.cfg.V, "d": wl.cfg.d,
                          "max_rel_vs_direct": float(np.max(np.abs(d - ref) / np.abs(ref)))}), flush=True)
    wmd.wmd_destroy(h)
