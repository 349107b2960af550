"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the same seeded
inputs. Distances: |gpu - oracle| <= 1e-4 |oracle| + 1e-5 (north_star 1e-4 relative, with the
absolute floor of DESIGN.md R22 for near-zero distances). Bookkeeping (query compaction,
partition, shard concatenation, determinism): bit-exact."""
import os
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5


@pytest.fixture(scope="module")
def W():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2005_06727_b200 import build
    build.build()
    from paper_2005_06727_b200 import wmd
    return wmd


def run_gpu(W, E, cp, ri, va, q, w, lam, iters, path=1, fallback=True, out="host", handle=None):
    h = handle or W.wmd_create(E, device=0)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, path)
        W.wmd_set_option(h, W.WMD_OPT_FALLBACK, int(fallback))
        W.wmd_set_targets(h, cp, ri, va)
        N = cp.shape[0] - 1
        if out == "host":
            d = np.empty(N, np.float32)
            try:
                W.wmd_query(h, q, w, lam, iters, d)
            except W.WmdError as e:
                if path == W.WMD_PATH_FUSED and "fused path does not support" in str(e):
                    pytest.skip(f"fused path: unsupported shape ({e})")
                raise
        else:
            import torch
            t = torch.empty(N, dtype=torch.float32, device="cuda:0")
            W.wmd_set_stream(h, torch.cuda.current_stream())
            W.wmd_query(h, q, w, lam, iters, t)
            torch.cuda.synchronize()
            d = t.cpu().numpy()
        W.wmd_sync(h)
        return d
    finally:
        if handle is None:
            W.wmd_destroy(h)


def assert_parity(g, o, what=""):
    g = np.asarray(g, np.float64)
    err = np.abs(g - o)
    bound = RTOL * np.abs(o) + ATOL
    bad = np.nonzero(~(err <= bound))[0]
    assert bad.size == 0, (f"{what}: {bad.size} docs out of tolerance; first {bad[:5]} "
                           f"gpu={g[bad[:5]]} oracle={o[bad[:5]]}")


PATHS = [1, 2]  # WMD_PATH_PER_ITER (one SDDMM_SpMM launch per iteration), WMD_PATH_FUSED (NEXT-1)


# ------------------------------------------------------------------ full configs, small

@pytest.mark.parametrize("path", PATHS)
def test_tiny_full(W, path):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    cfg = wl.cfg
    o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, dense=True)
    g = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    assert_parity(g, o, "tiny")


@pytest.mark.parametrize("path", PATHS)
def test_tweet_full(W, path):
    wl = synth.make_workload("tweet")
    q, w = wl.queries[0]
    cfg = wl.cfg
    o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)
    g = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    assert_parity(g, o, "tweet")


# ------------------------------------------------------------------ full-size configs, sampled docs

def _sampled_parity(W, name, n_sample, path, qi=0):
    wl = synth.make_workload(name, n_queries=qi + 1)
    q, w = wl.queries[qi]
    cfg = wl.cfg
    g = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    rng = np.random.default_rng(123)
    docs = np.sort(rng.choice(wl.N, size=n_sample, replace=False))
    docs = np.unique(np.concatenate([docs, [0, wl.N - 1]]))
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
    assert_parity(g[docs], o, name)
    assert np.all(np.isfinite(g))


@pytest.mark.parametrize("path", PATHS)
def test_long_sampled(W, path):
    _sampled_parity(W, "long", 300, path)


@pytest.mark.parametrize("path", PATHS)
def test_scaling_sampled(W, path):
    _sampled_parity(W, "scaling", 1000, path)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("qi", [0, 7])
def test_many_sampled(W, path, qi):
    _sampled_parity(W, "many", 500, path, qi=qi)


# ------------------------------------------------------------------ step a1 / a2 / a4 parity

def test_query_compaction_bit_exact(W):
    wl = synth.make_workload("tiny")
    rng = np.random.default_rng(5)
    q, w = wl.queries[0]
    perm = rng.permutation(q.shape[0])
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        d = np.empty(wl.N, np.float32)
        W.wmd_query(h, q[perm], w[perm], 10.0, 3, d)
        sel, r = W.wmd_get_query_rows(h, q.shape[0])
        osel, orr = oracle.select_nonzero(wl.cfg.V, q[perm], w[perm])
        assert np.array_equal(sel, osel)
        assert np.array_equal(r.astype(np.float64), orr)
        # the same query in the original order gives bit-identical distances
        d2 = np.empty(wl.N, np.float32)
        W.wmd_query(h, q, w, 10.0, 3, d2)
        assert np.array_equal(d, d2)
    finally:
        W.wmd_destroy(h)


@pytest.mark.parametrize("v_r", [1, 7, 30, 33, 64, 65, 100, 128])
def test_build_tensor_core_equals_simt_and_oracle(W, v_r):
    """a2 on the tensor cores (3xTF32 GEMM form; exact fixed point, the default) against the SIMT
    direct-difference build and the FP64 oracle's M: every query width class (N = 32/64/96/128 MMA tiles), a
    vocabulary that is not a multiple of the 128-row tile, exact zeros at the query words."""
    wl = synth.make_workload("tiny")
    V = 1000 + 77
    E = wl.E[:V]
    rng = np.random.default_rng(v_r)
    q = np.sort(rng.choice(V, v_r, replace=False)).astype(np.int32)
    w = np.full(v_r, 1.0 / v_r, np.float32)
    cp, ri, va = synth.csc_from_lists([{int(k): 1.0} for k in (0, 5, V - 1)], V)
    out = {}
    for build in (0, 1, 2):
        h = W.wmd_create(E)
        try:
            W.wmd_set_option(h, W.WMD_OPT_BUILD, build)
            W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)
            W.wmd_set_targets(h, cp, ri, va)
            W.wmd_query(h, q, w, 10.0, 2, np.empty(3, np.float32))
            ld = W.wmd_get_stats(h)["last_ld"]
            out[build] = W.wmd_read_kernel(h, 0, V, ld)
        finally:
            W.wmd_destroy(h)
    M = oracle.euclidean_rows(E, q).T                      # (V, v_r) FP64
    for build in (0, 1, 2):
        kt, km, cm = out[build]
        np.testing.assert_allclose(km[:, :v_r], M, rtol=2e-6, atol=2e-5)
        assert np.all(km[q, np.arange(v_r)] == 0.0)
        np.testing.assert_allclose(cm, M.min(axis=1), rtol=2e-6, atol=2e-5)
    np.testing.assert_allclose(out[0][1], out[1][1], rtol=2e-6, atol=2e-5)


@pytest.mark.parametrize("name", ["tiny", "tweet"])
def test_kernel_build_parity(W, name):
    """a2: M and K~ = exp(-lambda (M - min_i M)) against the FP64 oracle's M."""
    wl = synth.make_workload(name)
    q, w = wl.queries[0]
    lam = wl.cfg.lam
    v_r = np.unique(q).shape[0]
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        d = np.empty(wl.N, np.float32)
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_FUSED)   # builds M (+ m) only
        W.wmd_query(h, q, w, lam, 1, d)
        with pytest.raises(W.WmdError):
            W.wmd_read_kernel(h, 0, 4, W.wmd_get_stats(h)["last_ld"])
        _, km_fused, cm_fused = W.wmd_read_kernel(h, 0, wl.cfg.V, W.wmd_get_stats(h)["last_ld"], ktilde=False)
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)  # also builds K~
        W.wmd_query(h, q, w, lam, 1, d)
        st = W.wmd_get_stats(h)
        ld = st["last_ld"]
        V = wl.cfg.V
        ks = np.arange(0, V, max(1, V // 4000))
        kt, km, cm = W.wmd_read_kernel(h, 0, V, ld)
        assert np.array_equal(km[:, :v_r], km_fused[:, :v_r]) and np.array_equal(cm, cm_fused)
    finally:
        W.wmd_destroy(h)
    sel, r = oracle.select_nonzero(V, q, w)
    v_r = sel.shape[0]
    assert ld == (v_r + 7) // 8 * 8
    assert np.all(kt[:, v_r:] == 0) and np.all(km[:, v_r:] == 0)
    M = oracle.euclidean_rows(wl.E, sel)                    # (v_r, V) FP64
    m = M.min(axis=0)
    np.testing.assert_allclose(cm[ks], m[ks], rtol=2e-6, atol=1e-6)
    ref = np.exp(-lam * (M - m[None, :])).T                 # (V, v_r)
    # exact ones where the query word itself is the column minimum (M = 0)
    assert np.all(kt[sel, np.arange(v_r)] == 1.0)
    lk = np.log(np.maximum(kt[ks, :v_r].astype(np.float64), 1e-300))
    lr = np.log(ref[ks])
    mask = ref[ks] > 1e-30
    # |d ln K~| <= lambda * |dM| + argument rounding: M has FP32 relative error ~1e-6
    assert np.abs(lk - lr)[mask].max() < 1e-3
    # M itself (FP32 direct difference): relative error ~1e-6; exact zero self-distance
    np.testing.assert_allclose(km[ks, :v_r], M.T[ks], rtol=5e-6, atol=1e-5)
    assert np.all(km[sel, np.arange(v_r)] == 0.0)


def test_scaling_vector_parity_per_iteration_path(W):
    """a4: after t iterations u matches the oracle's 1/x up to the per-document gauge."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    for iters in (1, 2, 15):
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
            d = np.empty(wl.N, np.float32)
            W.wmd_query(h, q, w, wl.cfg.lam, iters, d)
            ld = W.wmd_get_stats(h)["last_ld"]
            u = W.wmd_read_scaling(h, 0, wl.N, ld)[:, : q.shape[0]].astype(np.float64)
        finally:
            W.wmd_destroy(h)
        _, st = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, wl.cfg.lam, iters,
                                    return_state=True)
        uo = st["u"]
        # gauge-invariant comparison: normalise each document by its largest entry
        ug = u / u.max(axis=1, keepdims=True)
        un = uo / uo.max(axis=1, keepdims=True)
        mask = un > 1e-20
        rel = np.abs(ug - un)[mask] / un[mask]
        assert rel.max() < 2e-3, (iters, rel.max())
        # the gauge is a power of two: max u of each document lies in [2^-64, 2^64]
        assert np.all(np.abs(np.log2(u.max(axis=1))) < 64)


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("path", PATHS)
def test_single_query_word_closed_form(W, path):
    """v_r = 1 (forced transport): WMD_j = sum_k c_kj M_0k."""
    wl = synth.make_workload("tiny")
    q = np.array([5], np.int32)
    g = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, [1.0], 10.0, 15, path=path)
    o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, [1.0], 10.0, 15)
    assert_parity(g, o, "v_r=1")


@pytest.mark.parametrize("path", PATHS)
def test_single_word_docs_and_query_equals_doc(W, path):
    wl = synth.make_workload("tiny")
    V = wl.cfg.V
    # single-word docs + the query's own histogram as a doc (distance ~ 0)
    q, w = wl.queries[0]
    docs = [{int(k): 1.0} for k in (0, 3, 77, V - 1)]
    docs.append({int(k): float(x) for k, x in zip(q, w)})
    cp, ri, va = synth.csc_from_lists(docs, V)
    for lam, iters in ((0.5, 15), (10.0, 15), (10.0, 1)):
        g = run_gpu(W, wl.E, cp, ri, va, q, w, lam, iters, path=path)
        o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, lam, iters)
        assert_parity(g, o, f"lam={lam} iters={iters}")
    assert abs(g[-1]) < 1e-3


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("v_r", [1, 2, 7, 8, 9, 16, 17, 31, 32, 33, 64, 65, 100, 128])
def test_query_width_boundaries(W, path, v_r):
    """Every K~ row-width class (ld = v_r rounded up to 8; 2..32 lanes per row), incl. the max."""
    wl = synth.make_workload("tiny")
    rng = np.random.default_rng(v_r)
    q = np.sort(rng.choice(wl.cfg.V, v_r, replace=False)).astype(np.int32)
    cnt = rng.geometric(0.5, v_r).astype(np.float64)
    w = (cnt / cnt.sum()).astype(np.float32)
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, np.arange(37))  # ragged: 37 docs
    g = run_gpu(W, wl.E, cp, ri, va, q, w, 10.0, 15, path=path)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 10.0, 15)
    assert_parity(g, o, f"v_r={v_r}")


@pytest.mark.parametrize("iters", [14, 15, 16, 30])
def test_cta_reanchor_single_document(W, iters):
    """The deterministic repro of the one-CTA kernel's fault: Tiny document 24
    alone against the v_r = 128 query of test_query_width_boundaries (2-warp instance at ld = 128,
    warp 1 without valid rows). Its smallest row sum fails the s-side range check at pass 15, so
    from 15 iterations on the re-anchor path runs and re-reads the block's rows (load_D) — where a
    CS2R-zeroed row offset was read stale in the builds that faulted."""
    wl = synth.make_workload("tiny")
    rng = np.random.default_rng(128)
    q = np.sort(rng.choice(wl.cfg.V, 128, replace=False)).astype(np.int32)
    cnt = rng.geometric(0.5, 128).astype(np.float64)
    w = (cnt / cnt.sum()).astype(np.float32)
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, np.array([24]))
    g = run_gpu(W, wl.E, cp, ri, va, q, w, 10.0, iters, path=2)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 10.0, iters)
    assert_parity(g, o, f"document 24, {iters} iterations")


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("iters", [0, 1, 2, 40, 100])
def test_iteration_counts(W, path, iters):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    g = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, iters, path=path)
    o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, iters)
    assert_parity(g, o, f"iters={iters}")


@pytest.mark.parametrize("path", PATHS)
def test_single_document_and_long_document(W, path):
    """N = 1, and a 1000-word document (many 32-entry chunks)."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    rng = np.random.default_rng(2)
    ids = np.sort(rng.choice(wl.cfg.V, 1000, replace=False))
    cnt = rng.geometric(0.3, 1000).astype(np.float64)
    docs = [{int(k): float(x) for k, x in zip(ids, (cnt / cnt.sum()).astype(np.float32))}]
    cp, ri, va = synth.csc_from_lists(docs, wl.cfg.V)
    g = run_gpu(W, wl.E, cp, ri, va, q, w, 10.0, 15, path=path)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 10.0, 15)
    assert_parity(g, o, "long doc")


def _degenerate_case():
    """Query = doc plus one more word (query strictly contains the doc's word set). Some query
    row of K~ restricted to the doc underflows in FP32 (SURVEY Finding 4), so the FP32 path must
    flag the doc and the FP64 GPU re-run must produce the oracle's value."""
    wl = synth.make_workload("tweet", n_queries=0, N=200)
    V = wl.cfg.V
    rng = np.random.default_rng(0)
    docs, queries = [], []
    for j in range(6):
        ids = np.sort(rng.choice(np.arange(100, V), 12, replace=False))
        cnt = rng.geometric(0.6, 12).astype(np.float64)
        docs.append({int(k): float(x) for k, x in zip(ids, (cnt / cnt.sum()).astype(np.float32))})
        queries.append(ids)
    extra = int(rng.integers(100, V))
    q_ids = np.unique(np.concatenate([queries[0], [extra]])).astype(np.int32)
    cnt = rng.geometric(0.6, q_ids.shape[0]).astype(np.float64)
    q_w = (cnt / cnt.sum()).astype(np.float32)
    cp, ri, va = synth.csc_from_lists(docs, V)
    return wl.E, cp, ri, va, q_ids, q_w


@pytest.mark.parametrize("path", PATHS)
def test_degenerate_doc_goes_through_fp64_fallback(W, path):
    E, cp, ri, va, q, w = _degenerate_case()
    o = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, 10.0, 15)
    assert np.all(np.isfinite(o))
    h = W.wmd_create(E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, path)
        W.wmd_set_targets(h, cp, ri, va)
        d = np.empty(cp.shape[0] - 1, np.float32)
        W.wmd_set_option(h, W.WMD_OPT_FALLBACK, 0)
        W.wmd_query(h, q, w, 10.0, 15, d)
        W.wmd_sync(h)
        flags = W.wmd_read_flags(h, cp.shape[0] - 1)
        if path == W.WMD_PATH_PER_ITER:
            # column-only rescale: the extra query row underflows in FP32 and must be flagged
            assert flags[0] & 1, "doc 0 (query superset) must be flagged in FP32"
        else:
            # the fused kernel's doc-local row rescale lifts that row: FP32 alone is in
            # tolerance, or the certificate flagged the document
            ok = np.abs(d.astype(np.float64) - o) <= RTOL * np.abs(o) + ATOL
            assert np.all(ok | (flags & 1).astype(bool))
        W.wmd_set_option(h, W.WMD_OPT_FALLBACK, 1)
        W.wmd_query(h, q, w, 10.0, 15, d)
        W.wmd_sync(h)
        flags = W.wmd_read_flags(h, cp.shape[0] - 1)
        st = W.wmd_get_stats(h)
    finally:
        W.wmd_destroy(h)
    if path == W.WMD_PATH_PER_ITER:
        assert flags[0] & 2
        assert st["fallback_docs"] >= 1
    assert_parity(d, o, "degenerate")


# ------------------------------------------------------------------ determinism / sharding

@pytest.mark.parametrize("path", PATHS)
def test_bitwise_determinism_and_shard_invariance(W, path):
    wl = synth.make_workload("tweet")
    q, w = wl.queries[0]
    cfg = wl.cfg
    full = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    again = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    assert np.array_equal(full, again)
    for P in (2, 3, 4, 8):
        b = W.wmd_partition(wl.col_ptr, P)
        assert np.array_equal(b, oracle.partition(wl.col_ptr, P))
        parts = []
        for g in range(P):
            if b[g] == b[g + 1]:
                continue
            cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, np.arange(b[g], b[g + 1]))
            parts.append(run_gpu(W, wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters, path=path))
        assert np.array_equal(np.concatenate(parts), full), P


def test_device_output_equals_host_output(W):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    a = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15, out="host")
    b = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15, out="device")
    assert np.array_equal(a, b)


def test_device_resident_inputs(W):
    import torch
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    Ed = torch.from_numpy(wl.E).cuda()
    h = W.wmd_create(Ed, device=0)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)  # run_gpu's default path
        W.wmd_set_targets(h, torch.from_numpy(wl.col_ptr).cuda(), torch.from_numpy(wl.row_idx).cuda(),
                          torch.from_numpy(wl.val).cuda())
        d = np.empty(wl.N, np.float32)
        W.wmd_query(h, q, w, 10.0, 15, d)
    finally:
        W.wmd_destroy(h)
    assert np.array_equal(d, run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15))


# ------------------------------------------------------------------ ABI errors on the GPU

def test_abi_errors_on_device(W):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    h = W.wmd_create(wl.E)
    try:
        d = np.empty(wl.N, np.float32)
        with pytest.raises(W.WmdError) as e:
            W.wmd_query(h, q, w, 10.0, 15, d)
        assert e.value.status == W.WMD_ERR_STATE
        bad = wl.val.copy()
        bad[0] = -1
        with pytest.raises(W.WmdError) as e:
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, bad)
        assert e.value.status == W.WMD_ERR_BAD_WEIGHTS
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        for args, code in (((q, w, -1.0, 15), W.WMD_ERR_INVALID_ARGUMENT),
                           ((q, w, 10.0, -1), W.WMD_ERR_INVALID_ARGUMENT),
                           ((np.array([0, 0], np.int32), np.array([.5, .5], np.float32), 10.0, 3),
                            W.WMD_ERR_BAD_WEIGHTS),
                           ((np.array([wl.cfg.V], np.int32), np.array([1.0], np.float32), 10.0, 3),
                            W.WMD_ERR_INDEX_OUT_OF_RANGE)):
            with pytest.raises(W.WmdError) as e:
                W.wmd_query(h, *args, d)
            assert e.value.status == code
        W.wmd_query(h, q, w, 10.0, 15, d)   # still usable after errors
        assert np.all(np.isfinite(d))
    finally:
        W.wmd_destroy(h)
    Enan = wl.E.copy()
    Enan[3, 2] = np.nan
    with pytest.raises(W.WmdError) as e:
        W.wmd_create(Enan)
    assert e.value.status == W.WMD_ERR_NONFINITE_EMBEDDING


def test_timing_stats(W):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_TIMING, 1)
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        d = np.empty(wl.N, np.float32)
        for _ in range(3):
            W.wmd_query(h, q, w, 10.0, 15, d)
        st = W.wmd_get_stats(h)
    finally:
        W.wmd_destroy(h)
    assert st["queries"] == 3 and st["timing_valid"] == 1
    assert st["iter_launches"] == 45
    assert st["build_ms"] > 0 and st["iter_ms"] > 0 and st["query_ms"] >= st["iter_ms"]


def test_auto_path_selection_and_cross_path_agreement(W):
    """AUTO runs the fused kernel when the shape fits (tweet-like docs, v_r <= 64), else the
    per-iteration kernel; both agree with each other to the parity tolerance."""
    wl = synth.make_workload("tweet")
    q, w = wl.queries[0]
    res = {}
    for path in (W.WMD_PATH_AUTO, W.WMD_PATH_PER_ITER, W.WMD_PATH_FUSED):
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_option(h, W.WMD_OPT_PATH, path)
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
            d = np.empty(wl.N, np.float32)
            W.wmd_query(h, q, w, wl.cfg.lam, wl.cfg.iters, d)
            res[path] = (d, W.wmd_get_stats(h)["last_path"])
        finally:
            W.wmd_destroy(h)
    assert res[W.WMD_PATH_AUTO][1] == W.WMD_PATH_FUSED
    assert np.array_equal(res[W.WMD_PATH_AUTO][0], res[W.WMD_PATH_FUSED][0])
    a, b = res[W.WMD_PATH_PER_ITER][0].astype(np.float64), res[W.WMD_PATH_FUSED][0].astype(np.float64)
    assert np.all(np.abs(a - b) <= 2e-4 * np.abs(a) + 2e-5)
    # documents of up to 320 words run fused (one CTA per document); longer ones, and long
    # ones under a stopping tolerance, fall back to the per-iteration path
    for n_words, tol, want in ((100, -1.0, W.WMD_PATH_FUSED), (320, -1.0, W.WMD_PATH_FUSED),
                               (321, -1.0, W.WMD_PATH_PER_ITER), (100, 1e-5, W.WMD_PATH_PER_ITER),
                               (64, 1e-5, W.WMD_PATH_FUSED)):
        cp, ri, va = synth.csc_from_lists([{int(k): 1.0 / n_words for k in range(n_words)}], wl.cfg.V)
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_targets(h, cp, ri, va)
            if tol >= 0:
                W.wmd_set_tolerance(h, tol)
            d = np.empty(1, np.float32)
            W.wmd_query(h, q[:8], w[:8] / w[:8].sum(), wl.cfg.lam, wl.cfg.iters, d)
            assert W.wmd_get_stats(h)["last_path"] == want, (n_words, tol)
        finally:
            W.wmd_destroy(h)


# ------------------------------------------------------------------ fused-kernel shape grid

def _docs_with_lengths(V, lengths, seed, p=0.6, lo_id=0):
    rng = np.random.default_rng(seed)
    cdf = synth.zipf_cdf(V, 1.07)
    docs = []
    for L in lengths:
        ids = set()
        while len(ids) < L:  # Zipf ids (hot words shared across documents), distinct
            ids.update(int(x) for x in np.searchsorted(cdf, rng.random(L - len(ids))))
        ids = np.array(sorted(ids)[:L])
        cnt = rng.geometric(p, L).astype(np.float64)
        docs.append({int(k): float(x) for k, x in zip(ids, (cnt / cnt.sum()).astype(np.float32))})
    return synth.csc_from_lists(docs, V)


@pytest.mark.parametrize("v_r", [1, 5, 8, 9, 16, 17, 24, 25, 30, 32, 33, 40, 41, 48, 49, 64])
def test_fused_bucket_and_width_grid(W, v_r):
    """Every one-warp fused-kernel instance: ld in {8, 16, 24, 32, 40, 48, 64} (CW = 1, 2, plain
    3, quad, quad + 1 or 2 plain columns, 2 quads) x length buckets {8, 16, 32, 40, 48, 64}
    (documents at and next to each boundary, ragged counts per bucket); AUTO must pick the fused
    path, and the distances must match the FP64 oracle."""
    wl = synth.make_workload("tweet", n_queries=0, N=10)
    V = wl.cfg.V
    lengths = [1, 2, 7, 8, 9, 15, 16, 17, 31, 32, 33, 39, 40, 41, 47, 48, 49, 63, 64] * 3
    if v_r > 48:  # the 64-wide tables keep documents of up to 48 words in one warp's registers
        lengths = [L for L in lengths if L <= 48]
    cp, ri, va = _docs_with_lengths(V, lengths, seed=v_r)
    rng = np.random.default_rng(100 + v_r)
    q = np.sort(rng.choice(2000, v_r, replace=False)).astype(np.int32)  # frequent words
    cnt = rng.geometric(0.6, v_r).astype(np.float64)
    w = (cnt / cnt.sum()).astype(np.float32)
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, cp, ri, va)
        d = np.empty(cp.shape[0] - 1, np.float32)
        W.wmd_query(h, q, w, 10.0, 15, d)
        W.wmd_sync(h)
        st = W.wmd_get_stats(h)
        assert st["last_path"] == W.WMD_PATH_FUSED
        assert st["last_ld"] == _warp_ld(v_r)
    finally:
        W.wmd_destroy(h)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 10.0, 15)
    assert_parity(d, o, f"fused grid v_r={v_r}")


def _cta_ld(v_r):
    return min(x for x in (32, 40, 48, 64, 80, 96, 104, 128) if x >= v_r)


def _warp_ld(v_r):
    return min(x for x in (8, 16, 24, 32, 40, 48, 64) if x >= v_r)


@pytest.mark.parametrize("v_r", [3, 20, 25, 33, 36, 40, 41, 44, 48, 56, 64, 65, 72, 80, 81, 90, 97, 100, 104, 105, 116, 128])
def test_fused_cta_long_documents(W, v_r):
    """One-CTA-per-document kernel (documents past the one-warp kernel's register budget): every
    row bucket {64, 128, 256: 32-row warps; 192: 48-row warps; 320: 40-row warps} x table width
    {32, 64, 80, 96, 104, 128} (column quads plus 0-3 plain columns per lane), documents
    at and next to each boundary up to the 320-word maximum plus a sweep of every third length,
    mixed with short documents that stay on the one-warp kernel; AUTO must pick the fused path,
    and the distances must match the FP64 oracle."""
    wl = synth.make_workload("tweet", n_queries=0, N=10)
    V = wl.cfg.V
    lengths = [1, 5, 8, 16, 33, 48, 49, 63, 64, 65, 70, 96, 127, 128, 129, 160, 191, 192, 193, 224,
               255, 256, 257, 290, 300, 319, 320] * 2 + list(range(50, 321, 3))
    cp, ri, va = _docs_with_lengths(V, lengths, seed=500 + v_r)
    rng = np.random.default_rng(600 + v_r)
    q = np.sort(rng.choice(3000, v_r, replace=False)).astype(np.int32)
    cnt = rng.geometric(0.6, v_r).astype(np.float64)
    w = (cnt / cnt.sum()).astype(np.float32)
    for lam, iters in ((10.0, 15), (1.0, 40)):
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_targets(h, cp, ri, va)
            d = np.empty(cp.shape[0] - 1, np.float32)
            W.wmd_query(h, q, w, lam, iters, d)
            W.wmd_sync(h)
            st = W.wmd_get_stats(h)
            assert st["last_path"] == W.WMD_PATH_FUSED
            assert st["last_ld"] == _cta_ld(v_r)
        finally:
            W.wmd_destroy(h)
        o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, lam, iters)
        assert_parity(d, o, f"fused CTA v_r={v_r} lam={lam}")


def test_warp_flagged_documents_rerun_with_reanchoring(W):
    """Documents of 50-64 words against a 40-word query (the Long config's) at lambda = 10: the
    one-warp kernel cannot certify a good share of them (dual potentials wider than the FP32
    exponent, R33); they are re-run in FP32 by the one-CTA kernel with re-anchoring
    (flag bit 2) before anything goes to the FP64 re-run, and every distance matches the oracle."""
    wl = synth.make_workload("long", n_queries=1)
    q, w = wl.queries[0]
    q = q[:40]
    w = (w[:40] / w[:40].sum()).astype(np.float32)
    docs = np.nonzero(np.diff(wl.col_ptr) <= 64)[0][:300]
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
    lam, iters = 10.0, 30
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, cp, ri, va)
        d = np.empty(docs.shape[0], np.float32)
        W.wmd_query(h, q, w, lam, iters, d)
        W.wmd_sync(h)
        st = W.wmd_get_stats(h)
        flags = W.wmd_read_flags(h, docs.shape[0])
        assert st["last_path"] == W.WMD_PATH_FUSED and st["last_ld"] == 40
    finally:
        W.wmd_destroy(h)
    assert np.count_nonzero(flags & 4) > 0, "expected documents re-run with re-anchoring"
    assert np.count_nonzero(flags & 2) < np.count_nonzero(flags & 4)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, lam, iters)
    assert_parity(d, o, "re-anchored re-run")


# ------------------------------------------------------------------ NEXT-2: query batches

def test_query_batch_equals_single_queries_and_oracle(W):
    """wmd_query_batch (host and device outputs) == back-to-back wmd_query bit for bit, and
    within tolerance of the oracle; varying v_r (15..40, the Many config's range) per query."""
    import torch
    wl = synth.make_workload("many", n_queries=6, N=3000)
    qs = wl.queries
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        single = np.empty((len(qs), wl.N), np.float32)
        for i, (q, w) in enumerate(qs):
            W.wmd_query(h, q, w, 10.0, 15, single[i])
        host = np.empty((len(qs), wl.N), np.float32)
        W.wmd_query_batch(h, qs, 10.0, 15, host)
        dev = torch.empty((len(qs), wl.N), dtype=torch.float32, device="cuda:0")
        W.wmd_set_stream(h, torch.cuda.current_stream())
        W.wmd_query_batch(h, qs, 10.0, 15, dev)
        torch.cuda.synchronize()
        W.wmd_sync(h)
        assert W.wmd_get_stats(h)["queries"] == 3 * len(qs)
    finally:
        W.wmd_destroy(h)
    assert np.array_equal(host, single)
    assert np.array_equal(dev.cpu().numpy(), single)
    for i in (0, len(qs) - 1):
        o = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, *qs[i], 10.0, 15)
        assert_parity(single[i], o, f"batch query {i}")


@pytest.mark.parametrize("batch", [0, 1, 2, 3, 7, 64])
def test_query_batch_passes_equal_single_queries(W, batch):
    """NEXT-2 (ii): B queries per fused pass (WMD_OPT_BATCH; 0 = automatic, 1 = one at a time),
    each document's entries read once for the B queries, queries regrouped by table width
    (v_r 15..40 -> widths 16/24/32/40) and written back in caller order: bit for bit the single
    queries' distances, the last query's flags, and a warp-flagged document (re-run by the
    one-CTA kernel) inside a batch."""
    wl = synth.make_workload("many", n_queries=11, N=2500)
    qs = list(wl.queries)
    # a 50-64-word document block against a 40-word query: the one-warp kernel flags some of
    # them (the FP32 re-anchoring re-run then runs inside the batch)
    cp, ri, va = _docs_with_lengths(wl.cfg.V, [60, 64, 52, 58] * 20, seed=77)
    rng = np.random.Generator(np.random.PCG64(5))
    qs.append(synth.make_query(rng, wl.cfg.V, 40, 1.07, 0.6))
    for corpus in ((wl.col_ptr, wl.row_idx, wl.val), (cp, ri, va)):
        N = corpus[0].shape[0] - 1
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_targets(h, *corpus)
            single = np.empty((len(qs), N), np.float32)
            for i, (q, w) in enumerate(qs):
                W.wmd_query(h, q, w, 10.0, 15, single[i])
            f_single = W.wmd_read_flags(h, N)
            W.wmd_set_option(h, W.WMD_OPT_BATCH, batch)
            out = np.empty((len(qs), N), np.float32)
            W.wmd_query_batch(h, qs, 10.0, 15, out)
            W.wmd_sync(h)
            f_batch = W.wmd_read_flags(h, N)
            sel, r = W.wmd_get_query_rows(h, qs[-1][0].shape[0])
        finally:
            W.wmd_destroy(h)
        assert np.array_equal(out, single)
        assert np.array_equal(f_batch, f_single)
        assert np.array_equal(sel, qs[-1][0])


def test_query_batch_validates_all_before_enqueueing(W):
    wl = synth.make_workload("tiny", n_queries=3)
    qs = list(wl.queries)
    bad = (np.array([1, 1], np.int32), np.array([0.5, 0.5], np.float32))  # duplicate id
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        out = np.zeros((4, wl.N), np.float32)
        with pytest.raises(W.WmdError) as e:
            W.wmd_query_batch(h, qs + [bad], 10.0, 15, out)
        assert e.value.status == W.WMD_ERR_BAD_WEIGHTS and "query 3" in str(e.value)
        assert W.wmd_get_stats(h)["queries"] == 0 and not out.any()
    finally:
        W.wmd_destroy(h)


# ------------------------------------------------------------------ NEXT-3: while x changes

@pytest.mark.parametrize("path", PATHS)
def test_while_x_changes_per_document(W, path):
    """wmd_set_tolerance: each document stops after the first x-update with
    max_i |x_new/x - 1| <= tol (the oracle's sinkhorn_wmd_per_doc). Distances within the parity
    tolerance; per-document update counts equal the oracle's up to +-1 (FP32 vs FP64 evaluation
    of a change that sits at the threshold) and exactly for the large majority."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    tol, lam, cap = 1e-5, 1.0, 800  # tol well above the FP32 noise of the change (~1e-6)
    o, o_its = oracle.sinkhorn_wmd_per_doc(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, lam, cap, tol)
    assert o_its.max() < cap
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, path)
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        W.wmd_set_tolerance(h, tol)
        d = np.empty(wl.N, np.float32)
        W.wmd_query(h, q, w, lam, cap, d)
        W.wmd_sync(h)
        its = W.wmd_read_iterations(h, wl.N)
        W.wmd_set_tolerance(h, -1.0)          # back to fixed iterations
        W.wmd_query(h, q, w, lam, 15, np.empty(wl.N, np.float32))
        assert np.all(W.wmd_read_iterations(h, wl.N) == 15)
    finally:
        W.wmd_destroy(h)
    assert_parity(d, o, f"while-x-changes path {path}")
    assert np.abs(its - o_its).max() <= 1
    assert np.mean(its == o_its) >= 0.9


@pytest.mark.parametrize("path", PATHS)
def test_graph_replay_equals_direct_launches(W, path):
    """WMD_OPT_GRAPH: the captured query graph replays bit-identically, re-reads the uploaded
    rows on every replay (different queries of the same width reuse it), and is re-captured
    when lambda or the iteration count changes."""
    wl = synth.make_workload("tiny", n_queries=3)
    qs = [(q, w) for q, w in wl.queries]
    qs.append((qs[0][0][::-1].copy(), qs[0][1][::-1].copy()))  # same words, other order
    runs = {}
    for graph in (0, 1):
        h = W.wmd_create(wl.E)
        try:
            W.wmd_set_option(h, W.WMD_OPT_PATH, path)
            W.wmd_set_option(h, W.WMD_OPT_GRAPH, graph)
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
            out = []
            for lam, iters in ((10.0, 15), (10.0, 15), (5.0, 15), (5.0, 3)):
                for q, w in qs:
                    d = np.empty(wl.N, np.float32)
                    W.wmd_query(h, q, w, lam, iters, d)
                    out.append(d)
            W.wmd_sync(h)
            runs[graph] = np.stack(out)
        finally:
            W.wmd_destroy(h)
    assert np.array_equal(runs[0], runs[1])
    assert not np.array_equal(runs[1][0], runs[1][1])


# ------------------------------------------------------------------ NEXT-4: sharded build

@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("P", [2, 3])
def test_sharded_build_two_phase_equals_one_shot(W, path, P):
    """wmd_query_begin/tables/finish with the vocabulary rows split over P ranks (emulated by P
    handles on one GPU; the table all-gather done here by copying the ranks' row slices) gives
    the one-shot wmd_query's distances bit for bit, for every rank's document shard."""
    import torch
    from paper_2005_06727_b200 import sharded
    wl = synth.make_workload("tweet", n_queries=1, N=600)
    q, w = wl.queries[0]
    ref = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15, path=path)
    bounds = sharded.shard_bounds(wl.col_ptr, P)
    V = wl.cfg.V
    hs = []
    try:
        for g in range(P):
            h = W.wmd_create(wl.E)
            W.wmd_set_option(h, W.WMD_OPT_PATH, path)
            cp, ri, va = sharded.local_shard(wl.col_ptr, wl.row_idx, wl.val, bounds, g)
            W.wmd_set_targets(h, cp, ri, va)
            hs.append(h)
        tabs = []
        for g, h in enumerate(hs):
            b, e, R = sharded.build_rows(V, P, g)
            W.wmd_query_begin(h, q, w, 10.0, 15, b, e, table_rows=P * R)
            tabs.append(W.wmd_query_tables(h, P * R))
        torch.cuda.synchronize()
        for g in range(P):  # emulated all-gather of the row slices
            b, e, R = sharded.build_rows(V, P, g)
            for t in (0, 2):
                if tabs[g][t] is None:
                    continue
                wdt = tabs[g][t + 1]
                for dst in range(P):
                    if dst != g:
                        tabs[dst][t][b * wdt:e * wdt].copy_(tabs[g][t][b * wdt:e * wdt])
        torch.cuda.synchronize()
        got = []
        for g, h in enumerate(hs):
            d = np.empty(int(bounds[g + 1] - bounds[g]), np.float32)
            W.wmd_query_finish(h, d)
            W.wmd_sync(h)
            got.append(d)
    finally:
        for h in hs:
            W.wmd_destroy(h)
    assert np.array_equal(np.concatenate(got), ref)


def test_two_phase_errors(W):
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        with pytest.raises(W.WmdError) as e:
            W.wmd_query_finish(h, np.empty(wl.N, np.float32))
        assert e.value.status == W.WMD_ERR_STATE
        with pytest.raises(W.WmdError) as e:
            W.wmd_query_begin(h, q, w, 10.0, 15, 5, wl.cfg.V + 1)
        assert e.value.status == W.WMD_ERR_INVALID_ARGUMENT
    finally:
        W.wmd_destroy(h)


def test_plain_c_consumer_query(W, tmp_path):
    """The C ABI from a plain C program (tests/c/abi_consumer.c): one query on the GPU, checked
    in C against the single-query-word closed form (sum_e c_e M_e)."""
    import subprocess
    import test_abi_host
    exe = test_abi_host._build_c_consumer(W, tmp_path)
    res = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "abi_consumer gpu ok" in res.stdout


@pytest.mark.parametrize("case", range(12))
def test_random_shapes_against_oracle(W, case):
    """Seeded random shapes across every kernel family: query width 1-128, 40 documents of
    1-320 words (mixed lengths, so one query runs the one-warp buckets, the one-CTA buckets and
    the re-runs together), lambda in {0.5, 5, 10, 25}, 0-30 iterations."""
    rng = np.random.default_rng(9000 + case)
    wl = synth.make_workload("tweet", n_queries=0, N=10)
    V = wl.cfg.V
    v_r = int(rng.integers(1, 129))
    lengths = [int(x) for x in rng.integers(1, 321, size=40)]
    lengths[:3] = [1, 16, 64]
    cp, ri, va = _docs_with_lengths(V, lengths, seed=9100 + case)
    q = np.sort(rng.choice(4000, v_r, replace=False)).astype(np.int32)
    cnt = rng.geometric(0.5, v_r).astype(np.float64)
    w = (cnt / cnt.sum()).astype(np.float32)
    lam = float(rng.choice([0.5, 5.0, 10.0, 25.0]))
    iters = int(rng.choice([0, 1, 7, 30]))
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h, cp, ri, va)
        d = np.empty(cp.shape[0] - 1, np.float32)
        W.wmd_query(h, q, w, lam, iters, d)
        W.wmd_sync(h)
        assert W.wmd_get_stats(h)["last_path"] == W.WMD_PATH_FUSED
    finally:
        W.wmd_destroy(h)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, lam, iters)
    assert_parity(d, o, f"random case {case}: v_r={v_r} lambda={lam} iters={iters}")


# ------------------------------------------------------------------ sharded layout agreement

def _mixed_corpus(V, with_giant, seed=3):
    """Short documents (10-40 words), then long ones (100-300), then optionally one 400-word
    document: a 3-way nnz partition puts shards on both sides of the one-warp (64-word) and
    one-CTA (320-word) limits."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = [synth.make_corpus(rng, V, 900, 10, 40, 1.07, 0.6), synth.make_corpus(rng, V, 60, 100, 300, 1.07, 0.3)]
    if with_giant:
        parts.append(synth.make_corpus(rng, V, 1, 400, 400, 1.07, 0.3))
    cps, ris, vas, off = [np.zeros(1, np.int64)], [], [], 0
    for cp, ri, va in parts:
        cps.append(cp[1:] + off)
        off += int(cp[-1])
        ris.append(ri)
        vas.append(va)
    return np.concatenate(cps), np.concatenate(ris), np.concatenate(vas)


@pytest.mark.parametrize("with_giant", [False, True])
def test_sharded_layout_agrees_across_length_thresholds(W, with_giant):
    """Every rank sets WMD_OPT_LAYOUT_DOC_NNZ to the global longest document, so ranks whose
    shards hold only short (or only long) documents still choose the unsharded run's path and
    row width: the emulated table all-gather is consistent and the distances are bitwise those
    of one handle over all documents. (Without the option, a short-document shard at v_r = 20
    would take the one-warp width 24 while the others use the one-CTA width 32, or the fused
    path while the others run per iteration.)"""
    import torch
    from paper_2005_06727_b200 import sharded
    wl = synth.make_workload("tweet", n_queries=1, N=50)
    V = wl.cfg.V
    cp, ri, va = _mixed_corpus(V, with_giant)
    rng = np.random.Generator(np.random.PCG64(9))
    q, w = synth.make_query(rng, V, 20, 1.07, 0.6)
    gmax = sharded.global_max_doc_nnz(cp)
    h0 = W.wmd_create(wl.E)
    try:
        W.wmd_set_targets(h0, cp, ri, va)
        ref = np.empty(cp.shape[0] - 1, np.float32)
        W.wmd_query(h0, q, w, 10.0, 15, ref)
        W.wmd_sync(h0)
        st0 = W.wmd_get_stats(h0)
    finally:
        W.wmd_destroy(h0)
    assert st0["last_path"] == (W.WMD_PATH_PER_ITER if with_giant else W.WMD_PATH_FUSED)
    P = 3
    bounds = sharded.shard_bounds(cp, P)
    hs = []
    try:
        for g in range(P):
            h = W.wmd_create(wl.E)
            W.wmd_set_option(h, W.WMD_OPT_LAYOUT_DOC_NNZ, gmax)
            c, r_, v_ = sharded.local_shard(cp, ri, va, bounds, g)
            W.wmd_set_targets(h, c, r_, v_)
            hs.append(h)
        tabs = []
        for g, h in enumerate(hs):
            b, e, R = sharded.build_rows(V, P, g)
            W.wmd_query_begin(h, q, w, 10.0, 15, b, e, table_rows=P * R)
            tabs.append(W.wmd_query_tables(h, P * R))
        assert len({(t[1], t[3]) for t in tabs}) == 1, "ranks disagree on the table layout"
        torch.cuda.synchronize()
        for g in range(P):
            b, e, R = sharded.build_rows(V, P, g)
            for t in (0, 2):
                if tabs[g][t] is None:
                    continue
                wdt = tabs[g][t + 1]
                for dst in range(P):
                    if dst != g:
                        tabs[dst][t][b * wdt:e * wdt].copy_(tabs[g][t][b * wdt:e * wdt])
        torch.cuda.synchronize()
        got = []
        for g, h in enumerate(hs):
            d = np.empty(int(bounds[g + 1] - bounds[g]), np.float32)
            W.wmd_query_finish(h, d)
            W.wmd_sync(h)
            st = W.wmd_get_stats(h)
            assert (st["last_path"], st["last_ld"]) == (st0["last_path"], st0["last_ld"])
            got.append(d)
    finally:
        for h in hs:
            W.wmd_destroy(h)
    assert np.array_equal(np.concatenate(got), ref)


def test_two_handles_and_counters_start_clean(W):
    """Handles created and destroyed back to back (device memory recycled by cudaMalloc) start
    with zeroed counters whether the embeddings come from the host or the device: no spurious
    NUMERICAL_BREAKDOWN at the first wmd_sync."""
    import torch
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    for src in ("host", "device", "host"):
        E = wl.E if src == "host" else torch.from_numpy(wl.E).cuda()
        h = W.wmd_create(E)
        try:
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
            d = np.empty(wl.N, np.float32)
            W.wmd_query(h, q, w, 10.0, 15, d)
            W.wmd_sync(h)
            assert W.wmd_get_stats(h)["fallback_docs"] == 0
        finally:
            W.wmd_destroy(h)


def test_timing_events_are_bounded_and_fold(W):
    """WMD_OPT_TIMING over many queries: phase times fold as queries complete (bounded event
    count), and a begun two-phase query keeps its events across other calls."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_TIMING, 1)
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        d = np.empty(wl.N, np.float32)
        for _ in range(200):
            W.wmd_query(h, q, w, 10.0, 15, d)
        st = W.wmd_get_stats(h)
        assert st["timing_valid"] and st["queries"] == 200 and st["query_ms"] > 0
        W.wmd_reset_stats(h)
        W.wmd_query_begin(h, q, w, 10.0, 15, 0, wl.cfg.V)
        W.wmd_get_stats(h)
        W.wmd_query_finish(h, d)
        st = W.wmd_get_stats(h)
        assert st["timing_valid"] and st["queries"] == 1 and st["build_ms"] > 0
    finally:
        W.wmd_destroy(h)


def test_handles_on_every_visible_device(W):
    """One handle per visible GPU in one process (per-device launch attributes); skips with one GPU."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("one GPU visible")
    wl = synth.make_workload("tweet", N=300)
    q, w = wl.queries[0]
    outs = []
    hs = [W.wmd_create(wl.E, device=dev) for dev in range(n)]
    try:
        for h in hs:
            W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
            d = np.empty(wl.N, np.float32)
            W.wmd_query(h, q, w, 10.0, 15, d)
            W.wmd_sync(h)
            outs.append(d)
    finally:
        for h in hs:
            W.wmd_destroy(h)
    for d in outs[1:]:
        assert np.array_equal(d, outs[0])


def test_nccl_single_rank_group(W):
    """The multi-GPU plumbing on a real NCCL communicator (world size 1, the only size one GPU
    allows): ShardedEngine.query, gather_distances, the in-place table all-gather of the
    sharded build, and the query-parallel row gather, each against the plain single-handle run."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2005_06727_b200 import sharded
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        assert dist.get_backend() == "nccl"
        wl = synth.make_workload("tweet", n_queries=3, N=800)
        q, w = wl.queries[0]
        ref = run_gpu(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15, path=0)
        E = torch.from_numpy(wl.E).cuda()
        eng = sharded.ShardedEngine(E, wl.col_ptr, wl.row_idx, wl.val, 0, 1, 0)
        got = eng.query(q, w, 10.0, 15)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), ref)
        out = sharded.gather_distances(got, np.array([0, wl.N], np.int64))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)
        # sharded-build plumbing: the one rank builds every row, gathers in place, solves
        h = eng.engine.h
        b, e, R = sharded.build_rows(wl.cfg.V, 1, 0)
        W.wmd_query_begin(h, q, w, 10.0, 15, b, e, table_rows=R)
        mx, wm, kt, wk = W.wmd_query_tables(h, R, 0)
        sharded.gather_table(mx, R, wm, 1, 0)
        d = torch.empty(wl.N, dtype=torch.float32, device="cuda:0")
        W.wmd_query_finish(h, d)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), ref)
        eng.close()
        qp = sharded.QueryParallelEngine(E, wl.col_ptr, wl.row_idx, wl.val, 0, 1, 0)
        rows = qp.engine.query_batch(wl.queries, 10.0, 15)
        full = sharded.gather_query_rows(rows, len(wl.queries), 1)
        torch.cuda.synchronize()
        assert np.array_equal(full.cpu().numpy(), rows.cpu().numpy())
        assert np.array_equal(full[0].cpu().numpy(), ref)
        qp.close()
    finally:
        dist.destroy_process_group()
