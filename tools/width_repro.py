"""Repro helper: test_query_width_boundaries' inputs (Tiny config, the first NDOCS documents,
v_r query words) on one path and build kernel.
    python tools/width_repro.py V_R PATH BUILD [REPEAT [LAMBDA [ITERS [NDOCS]]]]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

v_r, path, build = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rep = int(sys.argv[4]) if len(sys.argv) > 4 else 1
lam = float(sys.argv[5]) if len(sys.argv) > 5 else 10.0
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 15
ndocs = int(sys.argv[7]) if len(sys.argv) > 7 else 37
wl = synth.make_workload("tiny")
rng = np.random.default_rng(v_r)
q = np.sort(rng.choice(wl.cfg.V, v_r, replace=False)).astype(np.int32)
cnt = rng.geometric(0.5, v_r).astype(np.float64)
w = (cnt / cnt.sum()).astype(np.float32)
cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, np.arange(ndocs))
try:
    for _ in range(rep):
        h = wmd.wmd_create(wl.E)
        wmd.wmd_set_option(h, wmd.WMD_OPT_PATH, path)
        wmd.wmd_set_option(h, wmd.WMD_OPT_BUILD, build)
        wmd.wmd_set_targets(h, cp, ri, va)
        d = np.empty(ndocs, np.float32)
        wmd.wmd_query(h, q, w, lam, iters, d)
        wmd.wmd_sync(h)
        fl = wmd.wmd_read_flags(h, ndocs)
        wmd.wmd_destroy(h)
    print(v_r, path, build, lam, iters, ndocs, "ok", d[:3], "flags", np.bincount(fl, minlength=32)[[1, 2, 4, 8, 16]], flush=True)
except Exception as e:
    print(v_r, path, build, lam, iters, ndocs, "ERROR", e, flush=True)
