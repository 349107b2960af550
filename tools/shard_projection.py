"""Per-rank device time of the sharded Scaling step, emulated on one GPU (experiment helper).

For P ranks, every shard of the nnz-balanced document partition (wmd_partition) is solved on
its own handle after a build of that rank's vocabulary rows only (the two-phase API, as
ShardedEngine(shard_build=True) does); the NCCL all-gathers of the tables and of the distances
cannot run on one GPU and are reported as byte counts. Prints, per P, the slowest shard's
device time (build of R rows + solve of its documents) and T1 / (P * that).

    python tools/shard_projection.py [config] [P ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402
from paper_2005_06727_b200.sharded import build_rows, local_shard, shard_bounds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "scaling"
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
wl = synth.make_workload(cfg, n_queries=1)
q, w = wl.queries[0]
V = wl.cfg.V
out = {}
for P in Ps:
    bounds = shard_bounds(wl.col_ptr, P)
    worst = 0.0
    per = []
    for g in range(P):
        cp, ri, va = local_shard(wl.col_ptr, wl.row_idx, wl.val, bounds, g)
        h = wmd.wmd_create(wl.E)
        wmd.wmd_set_targets(h, cp, ri, va)
        n = cp.shape[0] - 1
        d = torch.empty(max(n, 1), dtype=torch.float32, device="cuda:0")
        wmd.wmd_set_stream(h, torch.cuda.current_stream())
        b, e, R = build_rows(V, P, g) if P > 1 else (0, V, V)
        times = []
        for it in range(5):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            wmd.wmd_query_begin(h, q, w, wl.cfg.lam, wl.cfg.iters, b, e, table_rows=P * R)
            wmd.wmd_query_finish(h, d[:n])
            a1.record()
            torch.cuda.synchronize()
            if it >= 2:
                times.append(a0.elapsed_time(a1))
        wmd.wmd_destroy(h)
        t = float(np.median(times))
        per.append(t)
        worst = max(worst, t)
    ld = 32 if wl.cfg.v_r <= 32 else 64
    out[P] = {"worst_rank_ms": worst, "ranks_ms": per,
              "table_allgather_bytes": P * (-(-V // P)) * (ld + 4) * 4 if P > 1 else 0,
              "dist_allgather_bytes": int(np.diff(bounds).max()) * 4 * P if P > 1 else 0}
T1 = out[Ps[0]]["worst_rank_ms"] if Ps[0] == 1 else None
for P in Ps:
    o = out[P]
    if T1:
        o["projected_efficiency_without_collectives"] = T1 / (P * o["worst_rank_ms"])
    print(json.dumps({"config": cfg, "P": P, **o}))
