"""FP32 numpy emulation behind DESIGN.md R39 (no per-iteration gauge in the half-warp kernel):
runs the doc-local rescaled iteration (Kh = 2^(-alpha (D - mu)), flushed below FLT_MIN, uh0 =
v_r 2^(-alpha mu)) WITHOUT any gauge on a sample of Scaling documents and reports the range the
iterates reach and the spread max uh / min uh over all iterations that the ratio-form certificate
compares with 2^110 / v_r. Experiment helper (FP32 restatement of the kernel's arithmetic, not the
oracle).

    python tools/emulate_ungauged.py [config] [n_docs] [iters]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "scaling"
ndocs = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
wl = synth.make_workload(cfg, n_queries=1)
q, r = wl.queries[0]
r = r.astype(np.float32)
alpha = np.float32(wl.cfg.lam * np.log2(np.e))
docs = np.random.default_rng(0).choice(wl.N, min(ndocs, wl.N), replace=False)
Eq = wl.E[q].astype(np.float64)
tiny = np.finfo(np.float32).tiny
rows = []
for j in docs:
    ids = wl.row_idx[wl.col_ptr[j]:wl.col_ptr[j + 1]]
    c = wl.val[wl.col_ptr[j]:wl.col_ptr[j + 1]].astype(np.float32)
    M = np.sqrt(((Eq[:, None, :] - wl.E[ids][None, :, :].astype(np.float64)) ** 2).sum(-1)).astype(np.float32)
    D = (M - M.min(0)[None, :]).T
    mu = D.min(0)
    Kh = np.exp2(-alpha * (D - mu[None, :])).astype(np.float32)
    Kh[Kh < tiny] = 0
    u = (len(q) * np.exp2(-alpha * mu)).astype(np.float32)
    umax, umin, vmax, vmin = 0.0, np.inf, 0.0, np.inf
    for _ in range(iters):
        v = (c / (Kh @ u)).astype(np.float32)
        u = (r / (Kh.T @ v)).astype(np.float32)
        umax, umin = max(umax, u.max()), min(umin, u.min())
        vmax, vmin = max(vmax, v.max()), min(vmin, v.min())
    rows.append((np.log2(umax), np.log2(umin), np.log2(vmax), np.log2(umax / umin), np.log2(vmax / vmin)))
st = np.array(rows)
lim = 110 - np.log2(len(q))
print(f"{cfg}: {len(docs)} documents, {iters} iterations, no gauge")
print(f"  log2 max uh over all t: {st[:, 0].min():.1f} .. {st[:, 0].max():.1f}; log2 min uh >= {st[:, 1].min():.1f}; log2 max vh <= {st[:, 2].max():.1f}")
print(f"  log2 spread uh (max / min over all t): p50 {np.percentile(st[:, 3], 50):.1f}  p99 {np.percentile(st[:, 3], 99):.1f}  max {st[:, 3].max():.1f}"
      f"  (ratio-form limit {lim:.1f}: {(st[:, 3] > lim).sum()} documents above)")
