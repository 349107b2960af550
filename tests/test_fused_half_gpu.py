"""NEXT-1 for short documents: the half-warp fused kernel (csrc/wmd_fused_half.cu, two documents
per warp, M recovered from the block in the final step, R37) against the FP64 oracle
(Algorithm 1) and against the one-warp kernel it replaces (WMD_FUSED_HALF=0)."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5


@pytest.fixture(scope="module")
def W():
    from paper_2005_06727_b200 import build
    build.build()
    from paper_2005_06727_b200 import wmd
    return wmd


def _run(W, E, cp, ri, va, q, w, lam, iters, half=True, batch=None):
    old = os.environ.get("WMD_FUSED_HALF")
    os.environ["WMD_FUSED_HALF"] = "1" if half else "0"
    h = W.wmd_create(E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_FUSED)
        W.wmd_set_targets(h, cp, ri, va)
        N = cp.shape[0] - 1
        if batch is not None:
            W.wmd_set_option(h, W.WMD_OPT_BATCH, len(batch))
            out = np.empty((len(batch), N), np.float32)
            W.wmd_query_batch(h, batch, lam, iters, out)
            W.wmd_sync(h)
            return out, None, W.wmd_get_stats(h)
        d = np.empty(N, np.float32)
        W.wmd_query(h, q, w, lam, iters, d)
        W.wmd_sync(h)
        return d, W.wmd_read_flags(h, N), W.wmd_get_stats(h)
    finally:
        W.wmd_destroy(h)
        if old is None:
            del os.environ["WMD_FUSED_HALF"]
        else:
            os.environ["WMD_FUSED_HALF"] = old


def _parity(g, o, what):
    g = np.asarray(g, np.float64)
    bad = np.nonzero(~(np.abs(g - o) <= RTOL * np.abs(o) + ATOL))[0]
    assert bad.size == 0, f"{what}: {bad.size} docs off; first {bad[:5]} gpu={g[bad[:5]]} oracle={o[bad[:5]]}"


@pytest.mark.parametrize("name", ["tiny", "tweet"])
def test_half_kernel_full_config(W, name):
    wl = synth.make_workload(name)
    q, w = wl.queries[0]
    cfg = wl.cfg
    o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
    g, flags, st = _run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
    assert st["last_path"] == W.WMD_PATH_FUSED and st["last_ld"] in (16, 32)
    _parity(g, o, name)
    g0, _, _ = _run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, half=False)
    np.testing.assert_allclose(g, g0, rtol=2e-5)


def _docs(V, lens, seed):
    rng = np.random.default_rng(seed)
    docs = []
    for n in lens:
        ids = np.sort(rng.choice(V, n, replace=False))
        wt = rng.random(n) + 0.05
        docs.append({int(k): float(x) for k, x in zip(ids, wt / wt.sum())})
    return synth.csc_from_lists(docs, V)


@pytest.mark.parametrize("v_r", [3, 9, 16, 17, 22, 30, 32, 33, 40])
@pytest.mark.parametrize("lam,iters", [(10.0, 15), (1e-3, 5), (0.05, 2), (25.0, 1), (10.0, 0)])
def test_half_kernel_shapes(W, v_r, lam, iters):
    """Every half-warp bucket (8/16/20/24/32/36/40 rows, lengths 1-40 incl. bucket edges), an odd number
    of documents per bucket (an empty half-warp item), table widths 16, 24, 32, 40, lambda down to the
    fused path's minimum, 0-15 iterations."""
    wl = synth.make_workload("tiny")
    V = wl.cfg.V
    lens = list(range(1, 41)) + [8, 9, 16, 17, 20, 21, 24, 25, 32, 33, 36, 37, 40, 1, 2]
    cp, ri, va = _docs(V, lens, 7 * v_r + iters)
    rng = np.random.default_rng(v_r)
    q = np.sort(rng.choice(V, v_r, replace=False)).astype(np.int32)
    w = (rng.random(v_r) + 0.1).astype(np.float32)
    w /= w.sum(dtype=np.float32)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, lam, iters, dense=True)
    g, flags, st = _run(W, wl.E, cp, ri, va, q, w, lam, iters)
    assert st["last_ld"] == -(-v_r // 8) * 8   # widths 8 and 24: the one-warp kernel
    _parity(g, o, f"v_r={v_r} lam={lam} iters={iters}")


def test_half_kernel_batched_queries(W):
    """wmd_query_batch (document-major (document, query) items) through the half-warp kernel equals
    the one-warp kernel and the oracle."""
    wl = synth.make_workload("tweet", N=1200, n_queries=6)
    cfg = wl.cfg
    batch = [(q, w) for q, w in wl.queries]
    g, _, _ = _run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, None, None, cfg.lam, cfg.iters, batch=batch)
    g0, _, _ = _run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, None, None, cfg.lam, cfg.iters, half=False, batch=batch)
    np.testing.assert_allclose(g, g0, rtol=2e-5)
    for i, (q, w) in enumerate(batch[:2]):
        o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
        _parity(g[i], o, f"batch query {i}")


def test_half_kernel_range_machinery_on_clustered_embeddings(W):
    """Clustered embeddings (the FP32 range certificate, flags, FP32 re-runs / FP64 fallback of
    flagged documents decide the result) through the half-warp kernel."""
    wl = synth.make_workload("tweet", N=2000)
    cfg = wl.cfg
    E = synth.make_clustered_embeddings(22, cfg.V, cfg.d, n_clusters=32, spread=0.2, norm_lo=0.5, norm_hi=1.25)
    q, w = wl.queries[0]
    o = oracle.sinkhorn_wmd(E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
    assert np.all(np.isfinite(o))
    g, flags, st = _run(W, E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
    _parity(g, o, "clustered")
    assert np.any(flags & 16), "no block had flushed entries: the UND path was not exercised"


def test_half_kernel_choice_is_shard_invariant(W):
    """The half-warp kernel runs on corpora of >= 32768 documents; WMD_OPT_LAYOUT_DOCS (the global
    document count, set by ShardedEngine on every rank) makes small shards take the same kernels,
    so the sharded distances stay bitwise those of one handle."""
    from paper_2005_06727_b200 import sharded
    wl = synth.make_workload("tweet", n_queries=1, N=900)
    q, w = wl.queries[0]

    def one(cp, ri, va, layout_docs):
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_option(h, W.WMD_OPT_LAYOUT_DOCS, layout_docs)
            W.wmd_set_targets(h, cp, ri, va)
            d = np.empty(cp.shape[0] - 1, np.float32)
            W.wmd_query(h, q, w, 10.0, 15, d)
            W.wmd_sync(h)
            return d
        finally:
            W.wmd_destroy(h)

    ref = one(wl.col_ptr, wl.row_idx, wl.val, 40000)
    warp = one(wl.col_ptr, wl.row_idx, wl.val, 0)
    assert not np.array_equal(ref, warp), "the layout option did not change the kernel"
    np.testing.assert_allclose(ref, warp, rtol=2e-5)
    bounds = sharded.shard_bounds(wl.col_ptr, 3)
    got = [one(*sharded.local_shard(wl.col_ptr, wl.row_idx, wl.val, bounds, g), 40000) for g in range(3)]
    assert np.array_equal(np.concatenate(got), ref)
