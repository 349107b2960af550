"""T-gen: the seeded input generator (synth/) against its recipe (DESIGN.md §4,
SURVEY.md §8(d) "Generator") and against the committed sha256 manifest, so every consumer
(oracle tests, GPU parity, bench) sees the same inputs whatever numpy version generates them.
CPU only. The big configs (Long, Scaling) are checked against the manifest in the GPU
full-parity tests, which generate them anyway."""
import numpy as np
import pytest

import synth


@pytest.fixture(scope="module", params=["tiny", "tweet", "many"])
def wl(request):
    return synth.make_workload(request.param)


def test_manifest_matches(wl):
    synth.check_manifest(wl)


def test_manifest_lists_every_config():
    m = synth.load_manifest()
    assert sorted(m) == sorted(synth.CONFIGS)
    for name, cfg in synth.CONFIGS.items():
        sh = m[name]["shape"]
        assert (sh["V"], sh["d"], sh["N"], sh["n_queries"]) == (cfg.V, cfg.d, cfg.N, cfg.n_queries)


def test_manifest_detects_a_change():
    w = synth.make_workload("tiny")
    w.val = w.val.copy()
    w.val[0] = np.nextafter(w.val[0], np.float32(1))
    with pytest.raises(AssertionError):
        synth.check_manifest(w)


def test_csc_invariants(wl):
    cfg = wl.cfg
    cp, ri, va = wl.col_ptr, wl.row_idx, wl.val
    assert cp.dtype == np.int64 and ri.dtype == np.int32 and va.dtype == np.float32
    assert cp[0] == 0 and cp[-1] == ri.shape[0] == va.shape[0]
    lens = np.diff(cp)
    assert lens.min() >= cfg.doc_lo and lens.max() <= cfg.doc_hi
    assert ri.min() >= 0 and ri.max() < cfg.V
    # ids strictly increasing within each column (distinct words, sorted)
    inner = np.ones(ri.shape[0], bool)
    inner[cp[:-1]] = False
    assert np.all(np.diff(ri.astype(np.int64))[inner[1:]] > 0)
    # weights: positive, finite, each column sums to 1 within the ABI tolerance (FP64 sum)
    assert np.all(va > 0) and np.all(np.isfinite(va))
    owner = np.repeat(np.arange(wl.N), lens)
    sums = np.bincount(owner, weights=va.astype(np.float64), minlength=wl.N)
    assert np.abs(sums - 1).max() <= 1e-5
    # the generator rounds once: ~6e-8 typical
    assert np.median(np.abs(sums - 1)) < 1e-6


def test_nnz_within_4_sigma(wl):
    cfg = wl.cfg
    n = cfg.doc_hi - cfg.doc_lo + 1
    mean = wl.N * (cfg.doc_lo + cfg.doc_hi) / 2
    sd = np.sqrt(wl.N * (n * n - 1) / 12)
    assert abs(wl.nnz - mean) <= 4 * sd + 1


def test_queries(wl):
    cfg = wl.cfg
    assert len(wl.queries) == cfg.n_queries
    for q, w in wl.queries:
        assert q.dtype == np.int32 and w.dtype == np.float32
        assert np.all(np.diff(q) > 0) and q.min() >= 0 and q.max() < cfg.V
        lo, hi = (cfg.v_r, cfg.v_r_hi) if cfg.v_r_hi else (cfg.v_r, cfg.v_r)
        assert lo <= q.shape[0] <= hi
        assert np.all(w > 0) and abs(float(np.sum(w, dtype=np.float64)) - 1) <= 1e-5
    if cfg.v_r_hi:  # "many": v_r ~ UniformInt[15, 40] over 256 queries spans the range
        lens = np.array([q.shape[0] for q, _ in wl.queries])
        assert lens.min() <= cfg.v_r + 3 and lens.max() >= cfg.v_r_hi - 3


def test_zipf_cdf_and_draws():
    V, s = 1000, 1.07
    cdf = synth.zipf_cdf(V, s)
    assert cdf[-1] == 1.0 and np.all(np.diff(cdf) > 0)
    pmf = np.diff(np.concatenate([[0.0], cdf]))
    k = np.arange(1, V + 1)
    np.testing.assert_allclose(pmf / pmf[0], k ** -s, rtol=1e-10)
    rng = np.random.Generator(np.random.PCG64(3))
    n = 400_000
    ids = synth._zipf_draw(rng, cdf, n)
    cnt = np.bincount(ids, minlength=V)
    for i in range(10):  # the most frequent ids against the pmf, within 5 sigma
        e = n * pmf[i]
        assert abs(cnt[i] - e) <= 5 * np.sqrt(e * (1 - pmf[i]))


def test_geometric_counts_recipe():
    """Counts are 1+Geometric(p) = numpy geometric(p) (support {1, 2, ...}, mean 1/p): a
    one-word document has weight exactly 1, and weights are ratios n_e / sum(n)."""
    rng = np.random.Generator(np.random.PCG64(11))
    ptr = np.array([0, 1, 4], np.int64)
    w = synth._weights(rng, ptr, 0.6)
    assert w[0] == np.float32(1.0)
    rng = np.random.Generator(np.random.PCG64(12))
    c = rng.geometric(0.3, size=200_000)
    assert c.min() == 1 and abs(c.mean() - 1 / 0.3) < 0.02


def test_clustered_embeddings():
    E = synth.make_clustered_embeddings(1, 3000, 64)
    E2 = synth.make_clustered_embeddings(1, 3000, 64)
    assert E.dtype == np.float32 and E.shape == (3000, 64) and np.all(np.isfinite(E))
    assert np.array_equal(E, E2)
    # norms span more than a decade (Gaussian rows would all sit near sqrt(d))
    nrm = np.linalg.norm(E.astype(np.float64), axis=1)
    assert nrm.max() / nrm.min() > 10
