"""a2 / NEXT-4: the exact tensor-core distance build (WMD_BUILD_EXACT, csrc/wmd_build_exact.cu).

The kernel's definition (include/wmd.h, R36): E is rounded once to fixed point
n = rint(E 2^F), F = 26 - e with max|E| < 2^e (dp <= 320), and
    M_ik = float32( sqrt( float32( sum_t (n_k,t - n_sel_i,t)^2 ) ) ) * 2^-F
with the integer sum exact. These tests restate that definition in numpy (int64, then the same two
FP32 roundings) and require the GPU table to match it BIT FOR BIT, and check it against the FP64
oracle's M within the quantisation bound sqrt(d) 2^-F plus FP32 rounding."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    from paper_2005_06727_b200 import build
    build.build()
    from paper_2005_06727_b200 import wmd
    return wmd


def _fixed_point_M(E, q):
    """The exact build's M by its definition: int64 sums of squared fixed-point differences."""
    dp = (E.shape[1] + 31) // 32 * 32
    assert dp <= 320
    amax = float(np.abs(E).max())
    e = np.frexp(np.float32(amax))[1] if amax > 0 else 0
    F = 26 - int(e)
    n = np.rint(np.ldexp(E.astype(np.float32), F)).astype(np.int64)   # exact scaling, RNE
    assert np.abs(n).max() <= 2 ** 26
    m2 = np.empty((E.shape[0], q.shape[0]), np.int64)
    for i, s in enumerate(q):                                       # exact in int64
        diff = n - n[s]
        m2[:, i] = np.einsum("kt,kt->k", diff, diff)
    M = np.sqrt(m2.astype(np.float32)) * np.float32(np.ldexp(1.0, -F))
    return M.astype(np.float32), F


def _read(W, E, q, build, path):
    V = E.shape[0]
    v_r = q.shape[0]
    w = np.full(v_r, 1.0 / v_r, np.float32)
    cp, ri, va = synth.csc_from_lists([{int(k): 1.0} for k in (0, 5, V - 1)], V)
    h = W.wmd_create(E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_BUILD, build)
        W.wmd_set_option(h, W.WMD_OPT_PATH, path)
        W.wmd_set_targets(h, cp, ri, va)
        W.wmd_query(h, q, w, 10.0, 2, np.empty(3, np.float32))
        ld = W.wmd_get_stats(h)["last_ld"]
        return W.wmd_read_kernel(h, 0, V, ld, ktilde=path == W.WMD_PATH_PER_ITER), ld
    finally:
        W.wmd_destroy(h)


@pytest.mark.parametrize("v_r", [1, 7, 30, 32, 33, 64, 65, 100, 128])
@pytest.mark.parametrize("d", [64, 300])
def test_exact_build_bitwise_against_its_definition(W, v_r, d):
    """Every pass count (32 query rows per pass), a vocabulary that is not a multiple of the
    128-row tile (the TMA box past V reads zeros), d = 64 (dp = 64) and 300 (dp = 320)."""
    E = synth.make_workload("tweet").E[:1077, :d].copy() if d == 300 else synth.make_workload("tiny").E[:1077]
    rng = np.random.default_rng(100 * d + v_r)
    q = np.sort(rng.choice(E.shape[0], v_r, replace=False)).astype(np.int32)
    (kt, km, cm), ld = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_PER_ITER)
    Mq, F = _fixed_point_M(E, q)
    assert np.array_equal(km[:, :v_r], Mq), np.abs(km[:, :v_r] - Mq).max()
    assert np.all(km[:, v_r:] == 0)
    assert np.array_equal(cm, Mq.min(axis=1))
    assert np.all(km[q, np.arange(v_r)] == 0.0)
    # against the FP64 oracle: quantisation (|dn| <= 2^-F per coordinate, both rows) + FP32 rounding
    M = oracle.euclidean_rows(E, q).T
    bound = np.sqrt(d) * 2.0 ** -F + 4 * np.spacing(M.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(km[:, :v_r] - M) <= bound)
    # K~ of the per-iteration path from the same M
    x = -10.0 * (km[:, :v_r].astype(np.float64) - cm[:, None])
    # FP32 rounding of the argument (|x| 2^-24) and of expf itself
    assert np.all(np.abs(kt[:, :v_r] - np.exp(x)) <= (np.abs(x) * 2.0 ** -23 + 2e-7) * np.exp(x) + 1e-37)


def test_exact_build_fused_table_equals_per_iteration_table(W):
    E = synth.make_workload("tiny").E[:1077]
    q = np.arange(3, 1077, 37, dtype=np.int32)[:25]
    (_, km_f, cm_f), ld_f = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_FUSED)
    (_, km_i, cm_i), ld_i = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_PER_ITER)
    assert np.array_equal(km_f[:, :25], km_i[:, :25]) and np.array_equal(cm_f, cm_i)


def test_exact_build_on_clustered_embeddings(W):
    """Clustered embeddings of varied norm (synth.make_clustered_embeddings), where the 3xTF32
    expansion loses ~1e-4 (R34): the exact build stays at the quantisation bound."""
    E = synth.make_clustered_embeddings(7, 3000, 300)
    rng = np.random.default_rng(7)
    q = np.sort(rng.choice(3000, 40, replace=False)).astype(np.int32)
    (_, km, cm), _ = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_PER_ITER)
    Mq, F = _fixed_point_M(E, q)
    assert np.array_equal(km[:, :40], Mq)
    M = oracle.euclidean_rows(E, q).T
    err = np.abs(km[:, :40] - M)
    assert err.max() <= np.sqrt(300) * 2.0 ** -F + 4 * np.spacing(np.float32(M.max()))
    (_, km_tc, _), _ = _read(W, E, q, W.WMD_BUILD_TENSOR_CORE, W.WMD_PATH_PER_ITER)
    assert err.max() < np.abs(km_tc[:, :40] - M).max()


def test_exact_build_degenerate_embeddings(W):
    """All-zero embeddings (F from max|E| = 0) and a single huge coordinate."""
    E = np.zeros((300, 64), np.float32)
    q = np.array([0, 7, 299], np.int32)
    (_, km, cm), _ = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_PER_ITER)
    assert np.all(km == 0) and np.all(cm == 0)
    E = synth.make_workload("tiny").E[:300].copy()
    E[17, 3] = 3.0e4
    (_, km, _), _ = _read(W, E, q, W.WMD_BUILD_EXACT, W.WMD_PATH_PER_ITER)
    Mq, _ = _fixed_point_M(E, q)
    assert np.array_equal(km[:, :3], Mq)


def test_exact_build_unavailable_for_wide_embeddings(W):
    E = np.random.default_rng(0).standard_normal((100, 1300)).astype(np.float32)   # dp = 1312
    h = W.wmd_create(E)
    try:
        with pytest.raises(W.WmdError):
            W.wmd_set_option(h, W.WMD_OPT_BUILD, W.WMD_BUILD_EXACT)
        W.wmd_set_option(h, W.WMD_OPT_BUILD, W.WMD_BUILD_DIRECT)
    finally:
        W.wmd_destroy(h)


@pytest.mark.parametrize("name", ["tweet", "many"])
def test_exact_build_end_to_end_against_oracle(W, name):
    """The whole path with the exact build on sampled documents against the FP64 oracle (the full
    configs run with the default build in test_full_parity_gpu.py)."""
    wl = synth.make_workload(name, n_queries=1)
    q, w = wl.queries[0]
    cfg = wl.cfg
    h = W.wmd_create(wl.E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_BUILD, W.WMD_BUILD_EXACT)
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        g = np.empty(wl.N, np.float32)
        W.wmd_query(h, q, w, cfg.lam, cfg.iters, g)
        W.wmd_sync(h)
    finally:
        W.wmd_destroy(h)
    docs = np.unique(np.concatenate([np.random.default_rng(5).choice(wl.N, 1500, replace=False), [0, wl.N - 1]]))
    cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, docs)
    o = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, cfg.lam, cfg.iters)
    np.testing.assert_allclose(g[docs], o, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("V", [1, 2, 77, 128, 129])
def test_exact_build_tiny_vocabularies(W, V):
    """Vocabularies smaller than one 128-row tile, exactly one tile, one row past it (the TMA box
    past V reads zeros; rows past V are not written)."""
    E = synth.make_workload("tiny").E[:V].copy()
    q = np.arange(min(V, 5), dtype=np.int32)
    w = np.full(q.shape[0], 1.0 / q.shape[0], np.float32)
    cp, ri, va = synth.csc_from_lists([{0: 1.0}, {V - 1: 1.0}], V)
    h = W.wmd_create(E)
    try:
        W.wmd_set_option(h, W.WMD_OPT_PATH, W.WMD_PATH_PER_ITER)
        W.wmd_set_targets(h, cp, ri, va)
        W.wmd_query(h, q, w, 10.0, 3, np.empty(2, np.float32))
        st = W.wmd_get_stats(h)
        assert st["last_build"] == W.WMD_BUILD_EXACT
        _, km, cm = W.wmd_read_kernel(h, 0, V, st["last_ld"])
    finally:
        W.wmd_destroy(h)
    Mq, _ = _fixed_point_M(E, q)
    assert np.array_equal(km[:, :q.shape[0]], Mq) and np.array_equal(cm, Mq.min(axis=1))
