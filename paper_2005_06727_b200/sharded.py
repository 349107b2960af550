"""Multi-GPU driver: target documents (columns of c) sharded across ranks, one process per GPU.

Documents are independent for the whole solve (Algorithm 1 touches column j only through
c[:,j], x[:,j], u[:,j]), so each rank runs the full hot path on its own
nnz-balanced contiguous document range (the paper's binary-search nnz split, PAPER.md:158,
snapped to document boundaries: wmd_partition) with no inter-GPU traffic inside the loop.
The one exchange step is the output: a padded all_gather_into_tensor of the FP32 distances
(NCCL over NVLink/NVSwitch), then a bit-exact compaction by the shard bounds.

The embeddings and the per-query K~ table are replicated (each rank builds its own K~: no
traffic). Per-document arithmetic does not depend on shard membership, so the distances are
bitwise identical for every world size.

QueryParallelEngine is the other decomposition, for many queries
against the same corpus: every rank holds all documents and runs whole queries (q = rank,
rank + P, ...), so there is neither a replicated distance build nor a per-query exchange; one
all-gather of the finished distance rows at the end of a batch.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

from . import wmd


def shard_bounds(col_ptr, world: int) -> np.ndarray:
    return wmd.wmd_partition(col_ptr, world)


def local_shard(col_ptr, row_idx, val, bounds, rank: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Rebased CSC of documents [bounds[rank], bounds[rank+1]) (integer bookkeeping only)."""
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    e0, e1 = int(col_ptr[b0]), int(col_ptr[b1])
    cp = np.asarray(col_ptr[b0:b1 + 1], dtype=np.int64) - e0
    return cp, np.ascontiguousarray(row_idx[e0:e1]), np.ascontiguousarray(val[e0:e1])


def global_max_doc_nnz(col_ptr) -> int:
    """Longest document of the whole corpus (integer bookkeeping; the layout every rank of a
    sharded run assumes, WMD_OPT_LAYOUT_DOC_NNZ)."""
    cp = np.asarray(col_ptr, np.int64)
    return int(np.diff(cp).max()) if cp.shape[0] > 1 else 0


def gather_distances(local, bounds, group=None, out=None):
    """All-gather the ranks' local distance vectors (lengths bounds[g+1]-bounds[g]) into the
    global order. `local` is a 1-D float32 tensor on this rank's device (CUDA for NCCL, CPU for
    gloo). Pads every shard to N_max = max shard length, one all_gather_into_tensor, then
    compacts: out[bounds[g] + i] = buf[g * N_max + i]."""
    import torch
    import torch.distributed as dist

    world = len(bounds) - 1
    lens = np.diff(np.asarray(bounds, np.int64))
    n_max = int(max(1, lens.max()))
    send = torch.zeros(n_max, dtype=local.dtype, device=local.device)
    send[: local.shape[0]] = local
    buf = torch.empty(world * n_max, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, send, group=group)
    N = int(bounds[-1])
    if out is None:
        out = torch.empty(N, dtype=local.dtype, device=local.device)
    if world > 0:
        idx = _compaction_index(tuple(int(b) for b in bounds), n_max, str(local.device))
        torch.index_select(buf, 0, idx, out=out)
    return out


_IDX_CACHE = {}


def _compaction_index(bounds, n_max, device):
    key = (bounds, n_max, device)
    if key not in _IDX_CACHE:
        import torch
        b = np.asarray(bounds, np.int64)
        idx = np.concatenate([g * n_max + np.arange(b[g + 1] - b[g]) for g in range(len(b) - 1)])
        _IDX_CACHE[key] = torch.from_numpy(idx.astype(np.int64)).to(device)
    return _IDX_CACHE[key]


def build_rows(V: int, world: int, rank: int) -> Tuple[int, int, int]:
    """Sharded distance build: rank g builds vocabulary rows [g R, min(V, (g+1) R)), R = ceil(V/P);
    returns (row_begin, row_end, R)."""
    R = -(-V // world)
    b = min(V, rank * R)
    return b, min(V, b + R), R


def gather_table(table, R: int, width: int, world: int, rank: int, group=None):
    """In-place all-gather of equal R-row slices of a flat (P R width) table view (NCCL)."""
    import torch.distributed as dist
    full = table[: world * R * width]
    dist.all_gather_into_tensor(full, full[rank * R * width:(rank + 1) * R * width], group=group)


class ShardedEngine:
    """One rank's view: owns a wmd handle over its document shard. With shard_build the per-query
    distance build is split over the ranks by vocabulary rows and the tables are all-gathered
    (NEXT-4; removes the replicated build from the per-rank critical path)."""

    def __init__(self, vocab_emb, col_ptr, row_idx, val, rank: int, world: int, device: int,
                 group=None, path: int = wmd.WMD_PATH_AUTO, timing: bool = False,
                 shard_build: bool = False):
        self.rank, self.world, self.group = rank, world, group
        self.device = device
        self.shard_build = shard_build and world > 1
        self.V = int(vocab_emb.shape[0])
        self.bounds = shard_bounds(col_ptr, world)
        self.N = int(np.shape(col_ptr)[0]) - 1
        cp, ri, va = local_shard(col_ptr, row_idx, val, self.bounds, rank)
        self.n_local = cp.shape[0] - 1
        self.nnz_local = int(cp[-1])
        self.engine: Optional[wmd.Engine] = None
        self.engine = wmd.Engine(vocab_emb, device=device, path=path, timing=timing)
        # every rank decides path and table width from the GLOBAL longest document (all ranks
        # hold the global col_ptr), so the ranks agree on the layout whatever their shard holds
        self.global_max_doc_nnz = global_max_doc_nnz(col_ptr)
        self.engine.set_option(wmd.WMD_OPT_LAYOUT_DOC_NNZ, self.global_max_doc_nnz)
        self.engine.set_option(wmd.WMD_OPT_LAYOUT_DOCS, self.N)   # same fused kernels on every rank
        if self.n_local > 0:
            self.engine.set_targets(cp, ri, va)
        elif self.shard_build:  # no documents, but this rank still builds and gathers its rows
            self.engine.set_targets(np.array([0, 1], np.int64), np.array([0], np.int32),
                                    np.array([1.0], np.float32))
        import torch
        self._local = torch.zeros(max(self.n_local, 1), dtype=torch.float32, device=f"cuda:{device}")
        self._out = torch.empty(self.N, dtype=torch.float32, device=f"cuda:{device}")

    def query(self, ids, weights, lam: float, iters: int):
        """Distances of all N documents (global order) on every rank."""
        if self.shard_build:
            # every rank builds its vocabulary rows, the tables are all-gathered, then each rank
            # solves its documents (ranks without documents still build and gather)
            h = self.engine.h
            b, e, R = build_rows(self.V, self.world, self.rank)
            wmd.wmd_query_begin(h, ids, weights, lam, iters, b, e, table_rows=self.world * R)
            mx, wm, kt, wk = wmd.wmd_query_tables(h, self.world * R, self.device)
            gather_table(mx, R, wm, self.world, self.rank, self.group)
            if kt is not None:
                gather_table(kt, R, wk, self.world, self.rank, self.group)
            wmd.wmd_query_finish(h, self._local[: max(self.n_local, 1)])
        elif self.n_local > 0:
            self.engine.query(ids, weights, lam, iters, out=self._local[: self.n_local])
        if self.world == 1:
            return self._local[: self.n_local]
        return gather_distances(self._local[: self.n_local], self.bounds, self.group, out=self._out)

    def close(self):
        if self.engine is not None:
            self.engine.close()


def query_assignment(nq: int, world: int, rank: int) -> np.ndarray:
    """Queries of one rank in the query-parallel decomposition: q = rank, rank + P, ..."""
    return np.arange(rank, nq, world, dtype=np.int64)


def gather_query_rows(local, nq: int, world: int, group=None):
    """All-gather the ranks' query rows (local: (len(query_assignment(nq, P, rank)), N) tensor)
    into the (nq, N) result in query order: one padded all_gather_into_tensor, then the
    row interleave out[q] = buf[q % P][q // P]."""
    import torch
    import torch.distributed as dist

    per = (nq + world - 1) // world
    N = local.shape[1]
    send = torch.zeros((per, N), dtype=local.dtype, device=local.device)
    send[: local.shape[0]] = local
    buf = torch.empty((world * per, N), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, send, group=group)
    q = np.arange(nq)
    idx = torch.from_numpy(((q % world) * per + q // world).astype(np.int64)).to(local.device)
    return torch.index_select(buf, 0, idx)


class QueryParallelEngine:
    """One rank's view of the query-parallel decomposition: all documents, a share of queries."""

    def __init__(self, vocab_emb, col_ptr, row_idx, val, rank: int, world: int, device: int,
                 group=None, path: int = wmd.WMD_PATH_AUTO, timing: bool = False):
        self.rank, self.world, self.group = rank, world, group
        self.N = int(np.shape(col_ptr)[0]) - 1
        self.engine = wmd.Engine(vocab_emb, device=device, path=path, timing=timing)
        self.engine.set_targets(col_ptr, row_idx, val)

    def query_batch(self, queries, lam: float, iters: int, gather: bool = True):
        """Distances (len(queries), N) in query order on every rank (gather=True), else this
        rank's rows (queries rank, rank + P, ...)."""
        import torch
        mine = query_assignment(len(queries), self.world, self.rank)
        if mine.shape[0]:
            local = self.engine.query_batch([queries[q] for q in mine], lam, iters)
        else:
            local = torch.empty((0, self.N), dtype=torch.float32, device=f"cuda:{self.engine.device}")
        if not gather or self.world == 1:
            return local
        return gather_query_rows(local, len(queries), self.world, self.group)

    def close(self):
        self.engine.close()
