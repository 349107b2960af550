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
TRAFFIC_JSON = os.path.join(ROOT, "profiles", "r02_traffic.json")


BUILD_NAMES = {0: "tensor-core 3xTF32 (tcgen05 kind::tf32)",
               1: "direct difference (FP32 SIMT)",
               2: "exact fixed point (tcgen05 kind::i8, TMA)"}

def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def _traffic(cfg_name):
    """DRAM bytes (read + write) of the Sinkhorn phase per step (one query) from the committed ncu
    --set full capture of this round (profiles/r02_traffic.json, written by tools/ncu_traffic.py),
    else None; with the capture's L2 hit rate when recorded."""
    for path in (TRAFFIC_JSON, os.path.join(ROOT, "profiles", "r01_traffic.json")):
        try:
            with open(path) as f:
                t = json.load(f)[cfg_name]
            return t["dram_bytes_per_query"], os.path.relpath(path, ROOT), t.get("l2_hit_rate_pct")
        except Exception:
            continue
    return None, None, None


def _cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class RoofBench:
    """In-run roofline denominators (tools/microbench/libroofbench.so, built by build()): L2 row
    gathers with the config's own word-id stream from a table of the config's M-table shape,
    a plain HBM stream read, and FP32 FMA issue. CUDA events on the current stream, best of 5."""

    def __init__(self):
        import ctypes
        from paper_2005_06727_b200 import build as b
        self.lib = ctypes.CDLL(b.build_roofbench())
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        self.lib.rb_gather_ms.argtypes = [P, I32, P, I64, P, P, I32, ctypes.POINTER(ctypes.c_float)]
        self.lib.rb_stream_ms.argtypes = [P, I64, P, P, I32, ctypes.POINTER(ctypes.c_float)]
        self.lib.rb_ffma_ms.argtypes = [I32, I32, P, P, I32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(I64)]
        self.ct = ctypes

    def measure(self, rows, row_floats, ids):
        import torch
        ct = self.ct
        st = torch.cuda.current_stream().cuda_stream
        sink = torch.zeros(4, dtype=torch.float32, device="cuda")
        out = {}
        rf = int(min(128, (row_floats + 3) // 4 * 4))
        tab = torch.zeros(rows * rf, dtype=torch.float32, device="cuda")
        n = int(min(ids.shape[0], 64 << 20))
        idx = torch.from_numpy(np.ascontiguousarray(ids[:n], dtype=np.int32)).cuda()
        ms = ct.c_float()
        rc = self.lib.rb_gather_ms(tab.data_ptr(), rf, idx.data_ptr(), n, sink.data_ptr(), st, 5, ct.byref(ms))
        if rc == 0:
            out["l2_gather_gbs"] = (n * rf * 4 + n * 4) / (ms.value * 1e-3) / 1e9
            out["l2_gather_how"] = (f"{n} gathers of {rf * 4}-B rows from a {rows} x {rf * 4}-B table "
                                    f"({rows * rf * 4 / 1e6:.1f} MB), row ids = the config's word-id stream; "
                                    "bytes = rows + ids")
        del tab, idx
        buf = torch.empty((2 << 30) // 4, dtype=torch.float32, device="cuda")
        buf.zero_()
        rc = self.lib.rb_stream_ms(buf.data_ptr(), buf.numel() // 4, sink.data_ptr(), st, 5, ct.byref(ms))
        if rc == 0:
            out["hbm_read_gbs"] = buf.numel() * 4 / (ms.value * 1e-3) / 1e9
        del buf
        fm = ct.c_int64()
        rc = self.lib.rb_ffma_ms(8, 4096, sink.data_ptr(), st, 5, ct.byref(ms), ct.byref(fm))
        if rc == 0:
            out["ffma_tflops"] = 2 * fm.value / (ms.value * 1e-3) / 1e12
        torch.cuda.synchronize()
        return out


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
    """Time the FP64 oracle (as it stands) on a bounded document sample. Returns (baseline dict,
    sampled document ids, the oracle's distances for them) — the distances double as the bench
    line's in-run parity sample."""
    import oracle
    cfg = wl.cfg
    rng = np.random.default_rng(seed)
    n = min(wl.N, 200)   # calibrate: a ~0.2 s probe, then grow the sample to ~target_s
    dt, o, docs, cp = 0.0, None, None, None
    for _ in range(5):
        docs = np.sort(rng.choice(wl.N, n, replace=False))
        cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
        t0 = time.perf_counter()
        o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
        dt = time.perf_counter() - t0
        if dt >= 0.5 * target_s or n >= wl.N:
            break
        n = int(min(wl.N, max(n + 1, n * target_s / max(dt, 1e-3))))
    units = int(cp[-1]) * len(q) * cfg.iters
    res = {"value": units / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{n} of {wl.N} docs ({int(cp[-1])} nnz), query 0, full build of M for the "
                     f"sample's words + {cfg.iters} iterations + final, FP64 single thread, {dt:.2f} s",
           **_cpu_info()}
    return res, docs, o


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
    probe, _, _ = cpu_oracle_rate(wl, q, w, target_s=0.5)
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
                         "sample": f"each step: {n_docs} random docs of {wl.N}, query 0, FP64 single thread",
                         **_cpu_info()},
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


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_distributed(n):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, one
    process per GPU (rendezvous on 127.0.0.1), as the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


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
    ap.add_argument("--no-roofbench", action="store_true", help="skip the in-run roofline microbenchmarks")
    ap.add_argument("--graph", action="store_true", help="replay each query as a CUDA graph (WMD_OPT_GRAPH)")
    ap.add_argument("--build", default="default", choices=["default", "exact", "direct", "tf32x3"],
                    help="distance build kernel (WMD_OPT_BUILD); default: the library's (exact where available)")
    ap.add_argument("--no-shard-build", action="store_true",
                    help="N > 1: every rank builds the whole distance table (default: vocabulary rows "
                         "split over the ranks + NCCL all-gather of the table)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch_distributed(args.gpus))
    wl = synth.make_workload(args.config)
    synth.check_manifest(wl)
    if args.impl == "reference":
        return run_reference(args, wl)
    if args.config == "many":
        return run_many(args, wl)

    import torch
    import torch.distributed as dist
    from paper_2005_06727_b200 import wmd
    from paper_2005_06727_b200.sharded import ShardedEngine

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world == 1:
            return [x]
        out = torch.empty(world, dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(out, t)
        return out.cpu().tolist()

    cfg = wl.cfg
    q, w = wl.queries[0]
    v_r = len(q)
    path = {"auto": wmd.WMD_PATH_AUTO, "iter": wmd.WMD_PATH_PER_ITER, "fused": wmd.WMD_PATH_FUSED}[args.path]
    E = torch.from_numpy(wl.E).cuda()
    eng = ShardedEngine(E, wl.col_ptr, wl.row_idx, wl.val, rank, world, local_rank, path=path,
                        timing=not args.graph, shard_build=not args.no_shard_build)
    h = eng.engine.h
    if args.build != "default":
        wmd.wmd_set_option(h, wmd.WMD_OPT_BUILD, {"exact": wmd.WMD_BUILD_EXACT, "direct": wmd.WMD_BUILD_DIRECT,
                                                  "tf32x3": wmd.WMD_BUILD_TENSOR_CORE}[args.build])
    if args.graph:
        wmd.wmd_set_option(h, wmd.WMD_OPT_GRAPH, 1)
    stream = torch.cuda.current_stream()
    small = (cfg.V * cfg.d * 4 + wl.nnz * 8) <= 2 * L2_BYTES
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda") if small else None

    def timed_steps(k):
        """k steps, device time in ms. Inputs larger than L2: k back-to-back queries between one
        barrier + synchronize on each side (each query's work is stream-ordered after the
        previous one's). Configs that fit in L2: a 256 MB L2-flushing write, then one
        synchronised, separately timed step at a time."""
        if flush is None:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            torch.cuda.synchronize()
            t0.record(stream)
            for _ in range(k):
                o = eng.query(q, w, cfg.lam, cfg.iters)
            t1.record(stream)
            torch.cuda.synchronize()
            return t0.elapsed_time(t1), o
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for s_ in range(k):
            flush.fill_(float(s_))
            barrier()
            torch.cuda.synchronize()
            ev[s_][0].record(stream)
            o = eng.query(q, w, cfg.lam, cfg.iters)
            ev[s_][1].record(stream)
            torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev), o

    # ---------------------------------------------------------------- device-resident timing
    for _ in range(args.warmup):
        eng.query(q, w, cfg.lam, cfg.iters)
    torch.cuda.synchronize()
    eng.engine.sync()
    wmd.wmd_reset_stats(h)
    with ClockSampler(local_rank) as clk:
        t_ms, out = timed_steps(args.steps)
    barrier()
    st = wmd.wmd_get_stats(h) if eng.n_local > 0 else None
    eng.engine.sync()
    st_sync = wmd.wmd_get_stats(h) if eng.n_local > 0 else None
    rank_ms = all_ranks(t_ms)
    T = max(rank_ms) / 1e3
    units = wl.nnz * v_r * cfg.iters * args.steps
    value = units / T
    check = out.float().cpu().numpy()
    assert np.all(np.isfinite(check)), "non-finite distances"

    # the other build mode at N > 1 (replicated build vs vocabulary-sharded build + table gather)
    alt = None
    if world > 1 and not args.graph:
        eng.shard_build = not eng.shard_build
        timed_steps(1)
        a_ms = max(all_ranks(timed_steps(args.steps)[0]))
        alt = {"build": "vocabulary rows sharded + NCCL table all-gather" if eng.shard_build else "replicated",
               "value": units / (a_ms / 1e3), "ms_per_step": a_ms / args.steps}
        eng.shard_build = not eng.shard_build

    # ---------------------------------------------------------------- end-to-end through the C ABI
    # host query arrays -> wmd_query (H2D inside) -> [all-gather] -> D2H into pinned host memory
    pin_out = torch.empty(wl.N, dtype=torch.float32, pin_memory=True)
    q_pin = torch.from_numpy(q.copy()).pin_memory()
    w_pin = torch.from_numpy(w.copy()).pin_memory()
    e2e_ms = 0.0
    for s_ in range(args.warmup + args.steps):
        if flush is not None:
            flush.fill_(float(s_))
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
        if s_ >= args.warmup:
            e2e_ms += a.elapsed_time(b)
    e2e_value = units / (max_over_ranks(e2e_ms) / 1e3)
    assert np.array_equal(pin_out.numpy(), check), "e2e result differs from the device-resident run"

    peaks_in_run = {}
    if rank == 0 and not args.no_roofbench and st:
        ld = int(st["last_ld"])
        fused = st["last_path"] == wmd.WMD_PATH_FUSED
        peaks_in_run = RoofBench().measure(cfg.V, (ld + 4) if fused else ld, wl.row_idx)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf bag-of-words, N(0,1) embeddings; BASELINE.json config; "
                    "inputs pinned by synth/manifest.json)",
            "config": config_dict(cfg, wl, args, path=args.path, graph=bool(args.graph),
                                  build=BUILD_NAMES.get(int(st["last_build"]) if st else -1, "?") +
                                  (", vocabulary rows sharded + NCCL table all-gather"
                                   if world > 1 and not args.no_shard_build else "")),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(v_r * 8),
                    "d2h_bytes_per_step": int(wl.N * 4)},
            "gpu_launches": int(st["kernel_launches"]) if st else 0,
        }
        line.update(roofline_fields(st, cfg, wl, eng, args, world, v_r, peaks_in_run))
        line.update({
            "phases_ms_per_step": ({k: st[k] / args.steps for k in ("build_ms", "iter_ms", "final_ms", "fallback_ms", "query_ms")}
                                   if st and st["timing_valid"] else None),
            "fallback_docs": int(st_sync["fallback_docs"]) if st_sync else 0,
            "launches_per_query": st["kernel_launches"] / max(1, st["queries"]) if st else 0,
            "clocks": clk.summary(),
        })
        if world > 1:
            line["rank_ms_per_step"] = [x / args.steps for x in rank_ms]
            if alt:
                line["alt_build"] = alt
        if world == 1 and not args.no_cpu_baseline:
            base, docs, o = cpu_oracle_rate(wl, q, w, target_s=float(os.environ.get("WMD_CPU_S", "15")))
            line["cpu_baseline"] = base
            g = check[docs].astype(np.float64)
            err = np.abs(g - o)
            line["parity_sample"] = {
                "docs": int(docs.shape[0]), "max_rel_err": float((err / np.abs(o)).max()),
                "within_tol": bool(np.all(err <= 1e-4 * np.abs(o) + 1e-5)),
                "what": "the timed run's distances on the cpu_baseline sample vs the FP64 oracle "
                        "(full-N parity: tests/test_full_parity_gpu.py, profiles/r02_parity.json)"}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def roofline_fields(st, cfg, wl, eng, args, world, v_r, pk):
    """The `roofline` object (dominant kernel) and the memory-roofline view BASELINE.json's metric
    asks for ("achieved GB/s vs B200 HBM/L2 peak"), from the library's per-phase CUDA events."""
    from paper_2005_06727_b200 import wmd
    peaks, peak_src = _peaks()
    if not (st and st["timing_valid"]):
        return {"roofline": {"kernel": None, "note": "per-phase timing is off in --graph mode (one graph per query)"}}
    nl, nnz_l = eng.n_local, eng.nnz_local
    t = cfg.iters
    hbm = peaks["hbm_gbs"]
    l2g = pk.get("l2_gather_gbs")
    traffic, traffic_src, l2hit = _traffic(cfg.name) if world == 1 else (None, None, None)
    # SURVEY.md §8(d) algorithmic bytes of the per-iteration formulation
    B_it = 8 * nnz_l + 4 * (nl + 1) + 8 * v_r * nl    # streamed: c, doc pointers, u read + write
    G_it = 4 * v_r * nnz_l                              # gathered: one K~ row slice per nonzero
    # the distance build (a2): HBM-bound streaming of the embedding rows (the exact build's limb
    # planes are 4 B per padded coordinate, like FP32 E) + the table writes
    rows = -(-cfg.V // world) if (world > 1 and eng.shard_build) else cfg.V
    dp = -(-cfg.d // 32) * 32
    per_iter = st["last_path"] == wmd.WMD_PATH_PER_ITER
    ldb = st["last_ld"]
    b_bytes = rows * (4 * dp + 4 * (ldb + 4) + (4 * ldb if per_iter else 0))
    t_b = st["build_ms"] / 1e3 / max(1, st["queries"])
    build_roof = {"kernel": BUILD_NAMES.get(int(st["last_build"]), "?"), "bound": "hbm",
                  "algorithmic_bytes": b_bytes, "ms": t_b * 1e3, "achieved": b_bytes / t_b / 1e9,
                  "peak": hbm, "unit": "GB/s", "frac": b_bytes / t_b / 1e9 / hbm, "peak_source": peak_src,
                  "share_of_step": st["build_ms"] / max(st["query_ms"], 1e-9)}
    if st["last_path"] == wmd.WMD_PATH_PER_ITER:
        n_launch = st["iter_launches"]
        t_launch = st["iter_ms"] / 1e3 / max(1, n_launch)
        ach = (B_it + G_it) / t_launch / 1e9
        roof = {
            "kernel": "sinkhorn_pass (one SDDMM_SpMM iteration)", "bound": "l2",
            "achieved": ach, "peak": l2g, "unit": "GB/s", "frac": ach / l2g if l2g else None,
            "peak_source": "measured in this run: " + pk.get("l2_gather_how", "n/a"),
            "algorithmic_bytes_per_launch": {"streamed": B_it, "gathered": G_it},
            "launch_ms": t_launch * 1e3,
            "hbm": {"achieved": B_it / t_launch / 1e9, "peak": hbm, "frac": B_it / t_launch / 1e9 / hbm,
                    "peak_source": peak_src},
            "traffic": traffic, "traffic_source": traffic_src,
            "share_of_step": st["iter_ms"] / max(st["query_ms"], 1e-9),
        }
        return {"roofline": roof, "build_roofline": build_roof}
    # fused path: all t iterations + the final step per document in one pass (one launch per
    # length bucket): FP32 issue-bound; the roofline is over the step's whole fused phase
    t_phase = st["iter_ms"] / 1e3 / args.steps
    flops = 4.0 * v_r * nnz_l * (t + 1)              # 2 FMAs per (nonzero, query row) per pass
    mhz = peaks.get("sm_max_mhz", 1965.0)
    sms = 148
    peak_tf = sms * 128 * 2 * mhz * 1e6 / 1e12
    ld = st["last_ld"]
    warp_max = 0 if ld > 64 else (48 if ld == 64 else 64)   # one-warp kernel's longest document
    # documents <= 40 words run two per warp (sinkhorn_half) at widths 16-40 on corpora of
    # >= 32768 documents (WMD_OPT_LAYOUT_DOCS: the global count at N > 1); DESIGN.md §5
    half = (ld in (16, 24, 32, 40) and wl.N >= 32768 and os.environ.get("WMD_FUSED_HALF") != "0") or \
        (os.environ.get("WMD_FUSED_HALF") == "1" and ld in (16, 24, 32, 40))
    parts = []
    if half and cfg.doc_lo <= 40:
        parts.append("sinkhorn_half")
    if cfg.doc_lo <= warp_max and (cfg.doc_hi > 40 or not half):
        parts.append("sinkhorn_fused")
    if cfg.doc_hi > warp_max:
        parts.append("sinkhorn_cta")
    kname = " + ".join(parts)
    roof = {
        "kernel": kname, "bound": "alu",
        "achieved": flops / t_phase / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
        "frac": flops / t_phase / 1e12 / peak_tf,
        "peak_source": f"derived: {sms} SMs x 128 FP32 FMA/clk x 2 flops x {mhz:.0f} MHz "
                       "(sm_max_mhz of MEASURED_PEAKS.json; DESIGN.md §5)",
        "ffma_measured_tflops": pk.get("ffma_tflops"),
        "algorithmic_flops_per_step": flops,
        "phase_ms": t_phase * 1e3,
        "launches_per_step": st["iter_launches"] / args.steps,
        "traffic": traffic, "traffic_source": traffic_src,
        "share_of_step": st["iter_ms"] / max(st["query_ms"], 1e-9),
    }
    # memory view: what the fused pass must move (c once, the M rows once, headers, output) and
    # the per-iteration formulation's bytes it replaces (t x (B_it + G_it) + the final step)
    streamed = 8 * nnz_l + 16 * nl + 4 * nl            # entries, headers, distances
    gathered = 4 * (ld + 4) * nnz_l                    # one M row (+ m_k) per nonzero, once
    equiv = t * (B_it + G_it) + (B_it - 4 * v_r * nl) + 2 * G_it
    mem = {
        "hbm": {"algorithmic_bytes_per_step": streamed, "achieved_gbs": streamed / t_phase / 1e9,
                "peak_gbs": hbm, "frac": streamed / t_phase / 1e9 / hbm, "peak_source": peak_src},
        "l2_gather": {"algorithmic_bytes_per_step": gathered, "achieved_gbs": gathered / t_phase / 1e9,
                      "peak_gbs": l2g, "frac": gathered / t_phase / 1e9 / l2g if l2g else None,
                      "peak_source": "measured in this run: " + pk.get("l2_gather_how", "n/a")},
        "per_iteration_equivalent": {
            "bytes_per_step": equiv, "achieved_gbs": equiv / t_phase / 1e9,
            "frac_of_l2_gather_peak": equiv / t_phase / 1e9 / l2g if l2g else None,
            "frac_of_hbm_peak": equiv / t_phase / 1e9 / hbm,
            "what": "SURVEY.md §8(d) bytes of t per-iteration SDDMM_SpMM passes + the final pass "
                    "(streamed B_it + gathered G_it each) over the fused phase's time: the bandwidth the "
                    "paper's per-iteration formulation would need to match it"},
        "dram_measured": {"bytes_per_step": traffic, "achieved_gbs": traffic / t_phase / 1e9 if traffic else None,
                          "l2_hit_rate_pct": l2hit, "source": traffic_src},
        "hbm_read_measured_gbs": pk.get("hbm_read_gbs"),
    }
    return {"roofline": roof, "memory_roofline": mem, "build_roofline": build_roof}


if __name__ == "__main__":
    main()
