#!/usr/bin/env python
"""Benchmark of the sparse Sinkhorn-WMD hot path (BASELINE.json metric:
"Sinkhorn nnz-updates/sec (nnz(c) x v_r x iters)").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config scaling] [--path auto|iter|fused]
    python bench.py --impl reference ...   # the FP64 CPU oracle (this tier's reference arm)

One step = one wmd_query: K~ build + all Sinkhorn iterations + final step + FP64 fallback
(+ the NCCL all-gather of the distances when N > 1), on synthetic inputs already resident in
HBM. Multi-GPU: launched by torch.distributed.run, one process per GPU, nnz-balanced document
shards (strong scaling: the total workload is fixed). Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Sinkhorn nnz-updates/sec (nnz(c) x v_r x iters)"
UNIT = "nnz-updates/s"
L2_BYTES = 126 * 2 ** 20
# Measured on this pool's B200 (profiles/r01_gather_bw.jsonl): random 128-B row gathers from an
# L2-resident table, all SMs. MEASURED_PEAKS.json has no L2 figure.
L2_GATHER_GBS = 20112.2


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def _traffic(cfg_name):
    """DRAM bytes (read + write) of the fused phase per step (one query) from the committed ncu
    --set full capture (profiles/r01_traffic.json, written by tools/ncu_traffic.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            t = json.load(f)[cfg_name]
        return t["dram_bytes_per_query"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_oracle_rate(wl, q, w, target_s: float, seed: int = 0):
    """Time the FP64 oracle (as it stands) on a bounded document sample; returns dict."""
    import oracle
    cfg = wl.cfg
    rng = np.random.default_rng(seed)
    # calibrate the sample: ~0.2 s probe, then scale to target_s
    n = min(wl.N, 200)
    docs = np.sort(rng.choice(wl.N, n, replace=False))
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
    t0 = time.perf_counter()
    oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
    dt = time.perf_counter() - t0
    n2 = n
    for _ in range(4):  # grow the sample until it takes ~target_s (M build is sublinear in n)
        if dt >= 0.5 * target_s or n2 >= wl.N:
            break
        n2 = int(min(wl.N, max(n2 + 1, n2 * target_s / max(dt, 1e-3))))
        docs = np.sort(rng.choice(wl.N, n2, replace=False))
        cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
        t0 = time.perf_counter()
        oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
        dt = time.perf_counter() - t0
    units = int(cp[-1]) * len(q) * cfg.iters
    return {"value": units / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n2} of {wl.N} docs ({int(cp[-1])} nnz), query 0, full build of M for the "
                      f"sample's words + {cfg.iters} iterations + final, FP64 single thread, {dt:.2f} s"}


def run_reference(args, wl):
    """--impl reference: the FP64 CPU oracle, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cfg = wl.cfg
    q, w = wl.queries[0]
    rng = np.random.default_rng(1)
    per_step = float(os.environ.get("WMD_REF_STEP_S", "4.0"))
    # size one step's doc sample so a step takes ~per_step seconds
    probe = cpu_oracle_rate(wl, q, w, target_s=0.5)
    nnz_per_s = probe["value"] / (len(q) * cfg.iters)
    n_docs = int(min(wl.N, max(10, per_step * nnz_per_s / (wl.nnz / wl.N))))
    times, units_tot = [], 0
    for s in range(args.warmup + args.steps):
        docs = np.sort(rng.choice(wl.N, n_docs, replace=False))
        cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
        t0 = time.perf_counter()
        oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            units_tot += int(cp[-1]) * len(q) * cfg.iters
    T = sum(times)
    value = units_tot / T
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Zipf bag-of-words, N(0,1) embeddings; BASELINE.json config)",
        "config": config_dict(cfg, wl, args, sample_docs=n_docs),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"each step: {n_docs} random docs of {wl.N}, query 0, FP64 single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, wl, args, **extra):
    d = {"workload": cfg.name, "V": cfg.V, "d": cfg.d, "N": cfg.N, "nnz": wl.nnz,
         "v_r": int(len(wl.queries[0][0])), "lambda": cfg.lam, "iters": cfg.iters,
         "words_per_doc": f"{cfg.doc_lo}-{cfg.doc_hi}", "zipf_s": cfg.zipf_s,
         "parallelism": f"doc-shard x{args.gpus}" if args.gpus > 1 else "1 GPU",
         "l2": ("inputs larger than L2 (E %.0f MB + c %.0f MB > 126 MB)" % (cfg.V * cfg.d * 4 / 1e6, wl.nnz * 8 / 1e6))
         if (cfg.V * cfg.d * 4 + wl.nnz * 8) > 2 * L2_BYTES else "L2 flushed (256 MB write) before every timed step"}
    d.update(extra)
    return d


def run_many(args, wl):
    """BASELINE config "Many queries": 256 queries (v_r 15..40) against 200k tweet-like documents,
    K rebuilt per query; one step = the whole batch. Query-parallel across ranks (NEXT-2 (i):
    every rank holds all documents, queries g, g+P, ...; one all-gather of the distance rows)."""
    import torch
    import torch.distributed as dist
    from paper_2005_06727_b200 import wmd
    from paper_2005_06727_b200.sharded import QueryParallelEngine

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    cfg = wl.cfg
    queries = wl.queries
    nq = len(queries)
    path = {"auto": wmd.WMD_PATH_AUTO, "iter": wmd.WMD_PATH_PER_ITER, "fused": wmd.WMD_PATH_FUSED}[args.path]
    E = torch.from_numpy(wl.E).cuda()
    eng = QueryParallelEngine(E, wl.col_ptr, wl.row_idx, wl.val, rank, world, local_rank, path=path)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        out = eng.query_batch(queries, cfg.lam, cfg.iters)
    torch.cuda.synchronize()
    eng.engine.sync()
    wmd.wmd_reset_stats(eng.engine.h)
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    t_ms = 0.0
    with ClockSampler(local_rank) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = eng.query_batch(queries, cfg.lam, cfg.iters)
            b.record(stream)
            torch.cuda.synchronize()
            t_ms += a.elapsed_time(b)
    barrier()
    eng.engine.sync()
    launches = int(wmd.wmd_get_stats(eng.engine.h)["kernel_launches"])
    t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    T = float(t.item()) / 1e3
    units = sum(wl.nnz * len(q) * cfg.iters for q, _ in queries) * args.steps
    assert bool(torch.isfinite(out).all()), "non-finite distances"
    # e2e: the same batch through the C ABI from host query arrays into pinned host rows
    # (rank-local rows; the all-gather is device-side and already in `value`)
    pin = torch.empty((len(range(rank, nq, world)), wl.N), dtype=torch.float32, pin_memory=True)
    mine = [queries[q] for q in range(rank, nq, world)]
    e2e_ms = 0.0
    for s in range(args.warmup + args.steps):
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if mine:
            wmd.wmd_query_batch(eng.engine.h, mine, cfg.lam, cfg.iters, pin)
        b.record(stream)
        torch.cuda.synchronize()
        if s >= args.warmup:
            e2e_ms += a.elapsed_time(b)
    e = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": METRIC, "value": units / T, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf bag-of-words, N(0,1) embeddings; BASELINE.json config)",
            "config": dict(config_dict(cfg, wl, args, path=args.path), queries=nq,
                           v_r=f"{min(len(q) for q, _ in queries)}-{max(len(q) for q, _ in queries)}",
                           parallelism=f"query-parallel x{world}" if world > 1 else "1 GPU"),
            "queries_per_s": nq * args.steps / T,
            "e2e": {"value": units / (float(e.item()) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(sum(8 * len(q) for q, _ in mine)),
                    "d2h_bytes_per_step": int(4 * len(mine) * wl.N)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("WMD_BENCH_CONFIG", "scaling"),
                    choices=sorted(synth.CONFIGS))
    ap.add_argument("--path", default="auto", choices=["auto", "iter", "fused"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true", help="replay each query as a CUDA graph (WMD_OPT_GRAPH)")
    ap.add_argument("--no-shard-build", action="store_true",
                    help="N > 1: every rank builds the whole distance table (default: vocabulary rows "
                         "split over the ranks + NCCL all-gather of the table)")
    args = ap.parse_args()

    wl = synth.make_workload(args.config)
    if args.impl == "reference":
        return run_reference(args, wl)
    if args.config == "many":
        return run_many(args, wl)

    import torch
    import torch.distributed as dist
    from paper_2005_06727_b200 import wmd
    from paper_2005_06727_b200.sharded import ShardedEngine, gather_distances

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = wl.cfg
    q, w = wl.queries[0]
    v_r = len(q)
    path = {"auto": wmd.WMD_PATH_AUTO, "iter": wmd.WMD_PATH_PER_ITER, "fused": wmd.WMD_PATH_FUSED}[args.path]
    E = torch.from_numpy(wl.E).cuda()
    eng = ShardedEngine(E, wl.col_ptr, wl.row_idx, wl.val, rank, world, local_rank, path=path,
                        timing=not args.graph, shard_build=not args.no_shard_build)
    h = eng.engine.h
    if args.graph:
        wmd.wmd_set_option(h, wmd.WMD_OPT_GRAPH, 1)
    stream = torch.cuda.current_stream()
    small = (cfg.V * cfg.d * 4 + wl.nnz * 8) <= 2 * L2_BYTES
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda") if small else None

    # ---------------------------------------------------------------- device-resident timing
    for _ in range(args.warmup):
        eng.query(q, w, cfg.lam, cfg.iters)
    torch.cuda.synchronize()
    eng.engine.sync()
    wmd.wmd_reset_stats(h)
    # Inputs larger than L2: K steps back to back between one barrier + synchronize on each side
    # (consecutive queries may overlap: the library builds query k+1's table while query k is
    # solved). Configs that fit in L2: a 256 MB L2-flushing write, then one synchronised,
    # separately timed step at a time (no overlap across steps).
    with ClockSampler(local_rank) as clk:
        if flush is None:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            torch.cuda.synchronize()
            t0.record(stream)
            for s in range(args.steps):
                out = eng.query(q, w, cfg.lam, cfg.iters)
            t1.record(stream)
            torch.cuda.synchronize()
            t_ms = t0.elapsed_time(t1)
        else:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for s in range(args.steps):
                flush.fill_(float(s))
                barrier()
                torch.cuda.synchronize()
                ev[s][0].record(stream)
                out = eng.query(q, w, cfg.lam, cfg.iters)
                ev[s][1].record(stream)
                torch.cuda.synchronize()
            t_ms = sum(a.elapsed_time(b) for a, b in ev)
    barrier()
    st = wmd.wmd_get_stats(h) if eng.n_local > 0 else None
    eng.engine.sync()
    st_sync = wmd.wmd_get_stats(h) if eng.n_local > 0 else None
    t_max = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    T = float(t_max.item()) / 1e3
    units = wl.nnz * v_r * cfg.iters * args.steps
    value = units / T
    check = out.float().cpu().numpy()
    assert np.all(np.isfinite(check)), "non-finite distances"

    # ---------------------------------------------------------------- end-to-end through the C ABI
    # host query arrays -> wmd_query (H2D inside) -> [all-gather] -> D2H into pinned host memory
    pin_out = torch.empty(wl.N, dtype=torch.float32, pin_memory=True)
    q_pin = torch.from_numpy(q.copy()).pin_memory()
    w_pin = torch.from_numpy(w.copy()).pin_memory()
    e2e_ms = 0.0
    for s in range(args.warmup + args.steps):
        if flush is not None:
            flush.fill_(float(s))
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if world == 1:
            wmd.wmd_query(h, q_pin.numpy(), w_pin.numpy(), cfg.lam, cfg.iters, pin_out)  # host out
        else:
            res = eng.query(q_pin.numpy(), w_pin.numpy(), cfg.lam, cfg.iters)
            pin_out.copy_(res, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        if s >= args.warmup:
            e2e_ms += a.elapsed_time(b)
    e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = units / (float(e2e_t.item()) / 1e3)
    assert np.array_equal(pin_out.numpy(), check), "e2e result differs from the device-resident run"

    if rank == 0:
        peaks, peak_src = _peaks()
        launches_per_query = st["kernel_launches"] / max(1, st["queries"]) if st else 0
        nl, nnz_l = eng.n_local, eng.nnz_local
        path_used = st["last_path"] if st else 0
        if not (st and st["timing_valid"]):
            roofline = {"kernel": None, "note": "per-phase timing is off in --graph mode (one graph per query)"}
        elif path_used == wmd.WMD_PATH_PER_ITER:
            n_iter_launch = st["iter_launches"]
            t_launch = st["iter_ms"] / 1e3 / max(1, n_iter_launch)
            B_it = 8 * nnz_l + 4 * (nl + 1) + 8 * v_r * nl      # streamed (HBM) bytes per launch
            G_it = 4 * v_r * nnz_l                              # K~ row gathers (L2) per launch
            roofline = {
                "kernel": "sddmm_spmm_iter", "bound": "l2",
                "achieved": (B_it + G_it) / t_launch / 1e9, "peak": L2_GATHER_GBS, "unit": "GB/s",
                "frac": (B_it + G_it) / t_launch / 1e9 / L2_GATHER_GBS,
                "peak_source": "measured L2 row-gather bandwidth, profiles/r01_gather_bw.jsonl",
                "algorithmic_bytes_per_launch": {"streamed": B_it, "gathered": G_it},
                "launch_ms": t_launch * 1e3,
                "hbm": {"achieved": B_it / t_launch / 1e9, "peak": peaks["hbm_gbs"],
                        "frac": B_it / t_launch / 1e9 / peaks["hbm_gbs"], "peak_source": peak_src},
                "roof_time_frac": max(B_it / (peaks["hbm_gbs"] * 1e9), (B_it + G_it) / (L2_GATHER_GBS * 1e9)) / t_launch,
                "traffic": None,
                "share_of_step": st["iter_ms"] / max(st["query_ms"], 1e-9),
            }
        else:
            # fused path: all iterations + final in one pass (one launch per length bucket);
            # the roofline is over the whole fused phase of the step
            t_phase = st["iter_ms"] / 1e3 / args.steps
            flops = 4.0 * v_r * nnz_l * (cfg.iters + 1)           # 2 FMAs per (nnz, row) per pass
            mhz = peaks.get("sm_max_mhz", 1965.0)
            peak_tf = 148 * 128 * 2 * mhz * 1e6 / 1e12
            ld = st["last_ld"]
            warp_max = 0 if ld > 64 else (48 if ld == 64 else 64)   # one-warp kernel's longest document
            kname = ("sinkhorn_cta" if cfg.doc_lo > warp_max else
                     ("sinkhorn_fused + sinkhorn_cta" if cfg.doc_hi > warp_max else "sinkhorn_fused"))
            roofline = {
                "kernel": kname, "bound": "alu",
                "achieved": flops / t_phase / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": flops / t_phase / 1e12 / peak_tf,
                "peak_source": f"derived: 148 SMs x 128 FP32 FMA/clk x 2 flops x {mhz:.0f} MHz "
                               "(sm_max_mhz of MEASURED_PEAKS.json; DESIGN.md §5)",
                "algorithmic_flops_per_step": flops,
                "phase_ms": t_phase * 1e3,
                "launches_per_step": st["iter_launches"] / args.steps,
                "l2_gather_bytes_per_step": 4 * (st["last_ld"] + 4) * nnz_l,  # one M row (+ m_k) per nonzero, once
                "traffic": _traffic(cfg.name) if world == 1 else None,
                "share_of_step": st["iter_ms"] / max(st["query_ms"], 1e-9),
            }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf bag-of-words, N(0,1) embeddings; BASELINE.json config)",
            "config": config_dict(cfg, wl, args, path=args.path, graph=bool(args.graph),
                                  build=("tensor-core 3xTF32, vocabulary rows sharded + NCCL table all-gather"
                                         if world > 1 and not args.no_shard_build else "tensor-core 3xTF32")),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(v_r * 8),
                    "d2h_bytes_per_step": int(wl.N * 4)},
            "gpu_launches": int(st["kernel_launches"]) if st else 0,
            "roofline": roofline,
            "phases_ms_per_step": ({k: st[k] / args.steps for k in ("build_ms", "iter_ms", "final_ms", "fallback_ms", "query_ms")}
                                   if st and st["timing_valid"] else None),
            "fallback_docs": int(st_sync["fallback_docs"]) if st_sync else 0,
            "launches_per_query": launches_per_query,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_oracle_rate(wl, q, w, target_s=float(os.environ.get("WMD_CPU_S", "15")))
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
