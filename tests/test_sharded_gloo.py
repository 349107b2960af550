"""Multi-process (world_size 2, gloo, CPU) test of the N>1 host path: nnz-balanced shard bounds,
rebased shard CSC, padded all_gather_into_tensor and the bit-exact compaction
(paper_2005_06727_b200/sharded.py). Per-shard distances come from the FP64 oracle here (test
infrastructure); on the GPU box the same gather/compaction code runs over NCCL after the CUDA
kernels. Documents are independent, so the gathered vector must equal the
single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    # sharded.py's host-side helpers (no CUDA needed); partition via the oracle's linear scan,
    # which tests/test_abi_host.py proves equal to wmd_partition
    from paper_2005_06727_b200 import sharded
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    bounds = oracle.partition(wl.col_ptr, world)
    cp, ri, va = sharded.local_shard(wl.col_ptr, wl.row_idx, wl.val, bounds, rank)
    local = np.zeros(0)
    if cp.shape[0] > 1:
        local = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, wl.cfg.lam, wl.cfg.iters)
    out = sharded.gather_distances(torch.from_numpy(local.astype(np.float32)), bounds)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_gather_matches_single_process(tmp_path, world):
    import oracle
    import synth
    try:
        from paper_2005_06727_b200 import sharded  # noqa: F401  (needs the built library)
    except ImportError as e:
        pytest.fail(f"library not built: {e}")
    res = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(world, _free_port(), res), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(res)
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    ref = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, wl.cfg.lam,
                              wl.cfg.iters).astype(np.float32)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_local_shard_and_compaction_index():
    from paper_2005_06727_b200 import sharded
    import synth
    wl = synth.make_workload("tiny")
    for P in (1, 2, 3, 7, 150):  # 150 > N: trailing empty shards
        b = sharded.shard_bounds(wl.col_ptr, P)
        assert b[0] == 0 and b[-1] == wl.N and np.all(np.diff(b) >= 0)
        parts = [sharded.local_shard(wl.col_ptr, wl.row_idx, wl.val, b, g) for g in range(P)]
        assert sum(p[0].shape[0] - 1 for p in parts) == wl.N
        assert np.array_equal(np.concatenate([p[1] for p in parts]), wl.row_idx)
        assert np.array_equal(np.concatenate([p[2] for p in parts]), wl.val)
        for p in parts:
            assert p[0][0] == 0
        lens = np.diff(b)
        n_max = max(1, int(lens.max()))
        idx = sharded._compaction_index(tuple(int(x) for x in b), n_max, "cpu").numpy()
        buf = np.full(P * n_max, -1.0)
        for g in range(P):
            buf[g * n_max: g * n_max + lens[g]] = np.arange(b[g], b[g + 1])
        assert np.array_equal(buf[idx], np.arange(wl.N))


def _qp_worker(rank, world, port, result_path, nq):
    """Query-parallel decomposition (NEXT-2 (i)): rank g runs queries g, g+P, ...; the padded
    row all-gather + interleave must give every query's row in query order."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2005_06727_b200 import sharded
    wl = synth.make_workload("tiny", n_queries=nq)
    mine = sharded.query_assignment(nq, world, rank)
    rows = [oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, *wl.queries[q], wl.cfg.lam,
                                wl.cfg.iters).astype(np.float32) for q in mine]
    local = torch.from_numpy(np.stack(rows) if rows else np.zeros((0, wl.N), np.float32))
    out = sharded.gather_query_rows(local, nq, world)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nq", [(2, 5), (3, 2)])
def test_query_parallel_gather_matches_single_process(tmp_path, world, nq):
    import oracle
    import synth
    res = str(tmp_path / "qp.npy")
    mp.start_processes(_qp_worker, args=(world, _free_port(), res, nq), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(res)
    wl = synth.make_workload("tiny", n_queries=nq)
    ref = np.stack([oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, *wl.queries[q], wl.cfg.lam,
                                        wl.cfg.iters).astype(np.float32) for q in range(nq)])
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_query_assignment_partitions_queries():
    from paper_2005_06727_b200 import sharded
    for nq in (0, 1, 5, 256):
        for P in (1, 2, 3, 8):
            parts = [sharded.query_assignment(nq, P, g) for g in range(P)]
            assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(nq))


def _table_worker(rank, world, port, result_path, V, width):
    """Sharded build bookkeeping: each rank fills its build_rows slice, gather_table (in-place
    all_gather_into_tensor of equal R-row slices) must give every rank the full table."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_06727_b200 import sharded
    b, e, R = sharded.build_rows(V, world, rank)
    table = torch.full((world * R * width,), -1.0)
    rows = torch.arange(b, e, dtype=torch.float32).repeat_interleave(width)
    table[b * width:e * width] = rows
    sharded.gather_table(table, R, width, world, rank)
    if rank == 0:
        np.save(result_path, table.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,V", [(2, 11), (3, 10), (3, 2)])
def test_sharded_build_table_gather(tmp_path, world, V):
    width = 5
    res = str(tmp_path / "table.npy")
    mp.start_processes(_table_worker, args=(world, _free_port(), res, V, width), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(res)
    assert np.array_equal(got[: V * width], np.arange(V, dtype=np.float32).repeat(width))
