"""Queries/s of wmd_query_batch on the Many config for several WMD_OPT_BATCH values (experiment
helper; not the bench).   python tools/batch_timing.py [batch,batch,...] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2005_06727_b200 import wmd  # noqa: E402

batches = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,0,2,4,8,16").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = synth.make_workload("many")
eng = wmd.Engine(torch.from_numpy(wl.E).cuda(), timing=True)
eng.set_targets(wl.col_ptr, wl.row_idx, wl.val)
out = torch.empty((len(wl.queries), wl.N), dtype=torch.float32, device="cuda")
ref = None
for bsz in batches:
    eng.set_option(wmd.WMD_OPT_BATCH, bsz)
    eng.query_batch(wl.queries, 10.0, 15, out=out)
    torch.cuda.synchronize()
    wmd.wmd_reset_stats(eng.h)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.query_batch(wl.queries, 10.0, 15, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    st = eng.stats()
    if ref is None:
        ref = out.clone()
    print(json.dumps({"batch": bsz, "ms_per_256": ms, "queries_per_s": 256e3 / ms,
                      "build_ms": st["build_ms"] / reps, "fused_ms": st["iter_ms"] / reps,
                      "rerun_ms": st["fallback_ms"] / reps, "launches": st["kernel_launches"] / reps,
                      "bitwise_equal_to_first": bool(torch.equal(out, ref))}), flush=True)
eng.close()
