"""Full-N parity (north_star: "every config's per-document WMD matches the FP64 oracle within
1e-4 relative error"): EVERY document of every BASELINE config — Tiny, Tweet, Long (100k),
Scaling (2M) and all 256 Many queries against the 200k-document corpus — on the GPU path
through the C ABI, against the FP64 oracle fanned out over the host cores. Documents are
independent in Algorithm 1, so the oracle runs nnz-balanced document ranges
(Many: whole queries) on concurrent threads (the C oracle runs without the GIL); each range is
the plain single-threaded oracle, unchanged.

Plus the numerical edges SURVEY.md §4.2 T-parity lists: lambda = 100 with v_r = 1 (closed form
sum_k c_kj M_0k, P4) and with single-word documents (closed form sum_i r_i M_ik, P5),
lambda = 1e-6 (entropic limit r^T M c_j, P6), and structured (clustered, varied
norm) embeddings whose distances are not concentrated near sqrt(2d), which drive the FP32 range
machinery (rescales, certificate, re-anchoring, FP64 re-run).

Tolerance: |gpu - oracle| <= 1e-4 |oracle| + 1e-5 per document (R22). Each case's
error distribution and flag counts are written to a JSON report (WMD_PARITY_REPORT, default
gpurun_out/r02_parity.json; copied to profiles/ by hand)."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.environ.get("WMD_PARITY_REPORT", os.path.join(ROOT, "gpurun_out", "r02_parity.json"))
THREADS = int(os.environ.get("WMD_ORACLE_THREADS", "0")) or (os.cpu_count() or 1)
FLAG_BITS = {"fp32_flagged": 1, "fp64_rerun": 2, "fp32_rerun_reanchored": 4, "cta_reanchored": 8,
             "certificate_in_force": 16}


@pytest.fixture(scope="module")
def W():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2005_06727_b200 import build
    build.build()
    oracle.build()
    from paper_2005_06727_b200 import wmd
    return wmd


# --------------------------------------------------------------------------- helpers

def oracle_fanout(E, cp, ri, va, q, w, lam, iters):
    """The FP64 oracle on THREADS nnz-balanced document ranges at once; concatenated distances."""
    N = cp.shape[0] - 1
    b = oracle.partition(cp, max(1, min(THREADS, N)))

    def job(g):
        j0, j1 = int(b[g]), int(b[g + 1])
        if j1 == j0:
            return np.zeros(0)
        e0, e1 = int(cp[j0]), int(cp[j1])
        return oracle.sinkhorn_wmd(E, cp[j0:j1 + 1] - e0, ri[e0:e1], va[e0:e1], q, w, lam, iters)

    with ThreadPoolExecutor(len(b) - 1) as ex:
        parts = list(ex.map(job, range(len(b) - 1)))
    return np.concatenate(parts)


def gpu_run(W, E, cp, ri, va, q, w, lam, iters, path=0, handle=None, build=None):
    """One query through the C ABI, host output; returns (distances, flags, stats)."""
    h = handle or W.wmd_create(E, device=0)
    try:
        if handle is None:
            W.wmd_set_option(h, W.WMD_OPT_PATH, path)
            if build is not None:
                W.wmd_set_option(h, W.WMD_OPT_BUILD, build)
            W.wmd_set_targets(h, cp, ri, va)
        N = cp.shape[0] - 1
        d = np.empty(N, np.float32)
        W.wmd_query(h, q, w, lam, iters, d)
        W.wmd_sync(h)
        return d, W.wmd_read_flags(h, N), W.wmd_get_stats(h)
    finally:
        if handle is None:
            W.wmd_destroy(h)


def parity_stats(g, o, flags):
    g = np.asarray(g, np.float64)
    err = np.abs(g - o)
    rel = err / np.maximum(np.abs(o), 1e-300)
    ok = err <= RTOL * np.abs(o) + ATOL
    anyflag = flags != 0
    st = {
        "docs": int(g.shape[0]),
        "within_tolerance": int(ok.sum()),
        "max_rel_err": float(rel.max()),
        "median_rel_err": float(np.median(rel)),
        "p99_rel_err": float(np.quantile(rel, 0.99)),
        "max_abs_err": float(err.max()),
        "oracle_range": [float(o.min()), float(o.max())],
    }
    for k, bit in FLAG_BITS.items():
        st[k] = int(((flags & bit) != 0).sum())
    st["flagged_any"] = int(anyflag.sum())
    st["max_rel_err_flagged"] = float(rel[anyflag].max()) if anyflag.any() else None
    return st, ok


def record(case, st):
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    try:
        with open(REPORT) as f:
            rep = json.load(f)
    except Exception:
        rep = {}
    st = dict(st, oracle_threads=THREADS, tolerance="|g-o| <= 1e-4|o| + 1e-5")
    rep[case] = st
    with open(REPORT, "w") as f:
        json.dump(rep, f, indent=1, sort_keys=True)
        f.write("\n")


def check(case, g, o, flags, extra=None):
    st, ok = parity_stats(g, o, flags)
    st.update(extra or {})
    record(case, st)
    bad = np.nonzero(~ok)[0]
    assert bad.size == 0, (f"{case}: {bad.size} of {g.shape[0]} docs out of tolerance; first {bad[:5]} "
                           f"gpu={np.asarray(g)[bad[:5]]} oracle={o[bad[:5]]}")
    assert np.all(np.isfinite(g))
    return st


_ORACLE = {}


def oracle_for(name, wl, qi=0):
    key = (name, qi)
    if key not in _ORACLE:
        q, w = wl.queries[qi]
        t0 = time.perf_counter()
        o = oracle_fanout(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, wl.cfg.lam, wl.cfg.iters)
        _ORACLE[key] = (o, time.perf_counter() - t0)
    return _ORACLE[key]


_WL = {}


def workload(name):
    if name not in _WL:
        _WL.clear()  # one big config in memory at a time
        wl = synth.make_workload(name)
        synth.check_manifest(wl)
        _WL[name] = wl
    return _WL[name]


# --------------------------------------------------------------------------- every document of every config

@pytest.mark.parametrize("name", ["tiny", "tweet", "long", "scaling"])
@pytest.mark.parametrize("path", [0, 1])  # WMD_PATH_AUTO (fused kernels), WMD_PATH_PER_ITER
def test_every_document(W, name, path):
    wl = workload(name)
    q, w = wl.queries[0]
    cfg = wl.cfg
    o, t_or = oracle_for(name, wl)
    g, flags, st = gpu_run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters, path=path)
    check(f"{name}/{'auto' if path == 0 else 'per_iter'}", g, o, flags,
          {"N": wl.N, "nnz": wl.nnz, "v_r": int(q.shape[0]), "lambda": cfg.lam, "iters": cfg.iters,
           "path_used": int(st["last_path"]), "ld": int(st["last_ld"]), "oracle_wall_s": round(t_or, 2)})


def test_every_document_all_256_many_queries(W):
    """Many: all 256 queries (v_r 15-40) x all 200k documents = 51.2M distances."""
    wl = workload("many")
    cfg = wl.cfg
    nq = len(wl.queries)

    def job(qi):
        q, w = wl.queries[qi]
        return oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, cfg.lam, cfg.iters)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(THREADS) as ex:
        O = list(ex.map(job, range(nq)))
    t_or = time.perf_counter() - t0
    h = W.wmd_create(wl.E, device=0)
    G, F, lds = [], [], set()
    try:
        W.wmd_set_targets(h, wl.col_ptr, wl.row_idx, wl.val)
        for qi in range(nq):
            q, w = wl.queries[qi]
            g, f, st = gpu_run(W, None, wl.col_ptr, None, None, q, w, cfg.lam, cfg.iters, handle=h)
            G.append(g)
            F.append(f)
            lds.add(int(st["last_ld"]))
        # the batched entry point gives the same bits
        import torch
        out = torch.empty((nq, wl.N), dtype=torch.float32, device="cuda:0")
        W.wmd_set_stream(h, torch.cuda.current_stream())
        W.wmd_query_batch(h, wl.queries, cfg.lam, cfg.iters, out)
        torch.cuda.synchronize()
        W.wmd_sync(h)
        assert np.array_equal(out.cpu().numpy(), np.stack(G))
    finally:
        W.wmd_destroy(h)
    check("many/all_256_queries", np.concatenate(G), np.concatenate(O), np.concatenate(F),
          {"queries": nq, "N": wl.N, "nnz": wl.nnz, "v_r": [int(min(q.shape[0] for q, _ in wl.queries)),
                                                           int(max(q.shape[0] for q, _ in wl.queries))],
           "lds": sorted(lds), "oracle_wall_s": round(t_or, 2)})


# --------------------------------------------------------------------------- numerical edges

@pytest.fixture(scope="module")
def tweet():
    return synth.make_workload("tweet")


# lambda = 100 needs distances the PLAIN FP64 oracle can exponentiate (exp(-100 M) underflows
# FP64 for M > ~7.4, and N(0,1) embeddings at d = 300 sit near sqrt(600) = 24.5): the Tweet
# embeddings scaled by 0.2 (distances ~4.9) keep the oracle finite; the GPU's rescaled FP32
# path is indifferent to the scale.
SCALE_100 = 0.2


@pytest.mark.parametrize("path", [0, 1])
def test_lambda_100_single_query_word(W, tweet, path):
    """v_r = 1 at lambda = 100: all mass goes to the one query word whatever K is (P4),
    WMD_j = sum_k c_kj M_0k; GPU against the oracle and against that closed form."""
    wl = tweet
    E = np.ascontiguousarray(wl.E * np.float32(SCALE_100))
    q = np.array([int(wl.queries[0][0][3])], np.int32)
    w = np.array([1.0], np.float32)
    o = oracle_fanout(E, wl.col_ptr, wl.row_idx, wl.val, q, w, 100.0, 15)
    M = oracle.euclidean_rows(E, q)[0]
    closed = np.add.reduceat(wl.val.astype(np.float64) * M[wl.row_idx], wl.col_ptr[:-1])
    np.testing.assert_allclose(o, closed, rtol=1e-12)
    g, flags, _ = gpu_run(W, E, wl.col_ptr, wl.row_idx, wl.val, q, w, 100.0, 15, path=path)
    check(f"edge/lambda100_vr1/{path}", g, o, flags)
    np.testing.assert_allclose(g, closed, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("path", [0, 1])
def test_lambda_100_single_word_documents(W, tweet, path):
    """Single-word documents at lambda = 100: after one x-update the plan's row i carries r_i
    to the one word (P5), WMD_j = sum_i r_i M_i,k_j."""
    wl = tweet
    E = np.ascontiguousarray(wl.E * np.float32(SCALE_100))
    rng = np.random.default_rng(17)
    N = 4000
    ri = rng.choice(wl.cfg.V, size=N, replace=True).astype(np.int32)
    cp = np.arange(N + 1, dtype=np.int64)
    va = np.ones(N, np.float32)
    q, w = wl.queries[0]
    o = oracle_fanout(E, cp, ri, va, q, w, 100.0, 15)
    sel, r = oracle.select_nonzero(wl.cfg.V, q, w)
    M = oracle.euclidean_rows(E, sel)
    closed = r @ M[:, ri] / r.sum()   # (the FP32 weights sum to 1 within ~1e-7)
    np.testing.assert_allclose(o, closed, rtol=1e-10)
    g, flags, _ = gpu_run(W, E, cp, ri, va, q, w, 100.0, 15, path=path)
    check(f"edge/lambda100_single_word_docs/{path}", g, o, flags)
    np.testing.assert_allclose(g, closed, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("path", [0, 1])
def test_lambda_1e6_entropic_limit(W, tweet, path):
    """lambda = 1e-6: K -> 1, the plan -> r c_j^T, WMD_j -> r^T M c_j with O(lambda) error (P6,
    PAPER.md:49); GPU against the oracle and against the limit."""
    wl = tweet
    q, w = wl.queries[0]
    o = oracle_fanout(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 1e-6, 15)
    sel, r = oracle.select_nonzero(wl.cfg.V, q, w)
    M = oracle.euclidean_rows(wl.E, sel)
    limit = np.add.reduceat((r @ M)[wl.row_idx] * wl.val.astype(np.float64), wl.col_ptr[:-1])
    np.testing.assert_allclose(o, limit, rtol=1e-5)
    g, flags, _ = gpu_run(W, wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 1e-6, 15, path=path)
    check(f"edge/lambda1e-6/{path}", g, o, flags)
    np.testing.assert_allclose(g, limit, rtol=RTOL, atol=ATOL)


def _clustered_case(kind):
    if kind == "tweet":
        cfg = synth.CONFIGS["tweet"]
        wl = synth.make_workload("tweet")
        E = synth.make_clustered_embeddings(21, cfg.V, cfg.d, n_clusters=64, spread=0.15,
                                            norm_lo=0.5, norm_hi=1.5)
        return E, wl.col_ptr, wl.row_idx, wl.val, wl.queries[0], cfg.lam, cfg.iters
    # long documents (50-300 words) against a 100-word query, 5000 documents
    cfg = synth.CONFIGS["long"]
    wl = synth.make_workload("long", N=5000)
    E = synth.make_clustered_embeddings(22, cfg.V, cfg.d, n_clusters=32, spread=0.2,
                                        norm_lo=0.5, norm_hi=1.25)
    return E, wl.col_ptr, wl.row_idx, wl.val, wl.queries[0], cfg.lam, cfg.iters


@pytest.mark.parametrize("kind", ["tweet", "long"])
@pytest.mark.parametrize("path", [0, 1])
def test_structured_embeddings(W, kind, path):
    """Clustered embeddings with varied norms (synth.make_clustered_embeddings): distances from
    ~0 to several times sqrt(2d), so exp(-lambda M) spans far beyond FP32's exponent range within
    a document and the certificate / re-anchoring / FP64 re-run decide the result. The plain
    FP64 oracle stays finite on these inputs (asserted). Default build (WMD_BUILD_EXACT) and the
    direct-difference build are asserted; the 3xTF32 GEMM-form build's error on the same inputs
    is recorded, not asserted (R34: its |e|^2 + |q|^2 - 2e.q cancellation reaches ~1e-4
    of the distance here)."""
    E, cp, ri, va, (q, w), lam, iters = _clustered_case(kind)
    o = oracle_fanout(E, cp, ri, va, q, w, lam, iters)
    assert np.all(np.isfinite(o)), "instance outside the plain FP64 oracle's range"
    g, flags, st = gpu_run(W, E, cp, ri, va, q, w, lam, iters, path=path)
    name = f"edge/clustered_{kind}/{'auto' if path == 0 else 'per_iter'}"
    s = check(name, g, o, flags, {"N": int(cp.shape[0] - 1), "v_r": int(q.shape[0]), "ld": int(st["last_ld"]),
                                  "path_used": int(st["last_path"]), "build": "exact"})
    assert st["last_build"] == W.WMD_BUILD_EXACT
    # the instance must actually exercise the FP32 range machinery: in most documents the
    # doc-local block Kh = exp(-lambda (D - mu)) has entries below FLT_MIN = 2^-126 (a property
    # of the inputs, from the oracle's FP64 M)
    sel, _ = oracle.select_nonzero(E.shape[0], q, w)
    M = oracle.euclidean_rows(E, sel)
    m = M.min(0)
    spans = []
    for j in range(min(200, cp.shape[0] - 1)):
        D = M[:, ri[cp[j]:cp[j + 1]]] - m[ri[cp[j]:cp[j + 1]]]
        spans.append(lam * (D - D.min(1, keepdims=True)).max())
    assert np.mean(np.array(spans) > 126 * np.log(2)) > 0.5
    gd, fd, std = gpu_run(W, E, cp, ri, va, q, w, lam, iters, path=path, build=W.WMD_BUILD_DIRECT)
    check(name + "/direct_build", gd, o, fd, {"build": "direct"})
    gt, ft, _ = gpu_run(W, E, cp, ri, va, q, w, lam, iters, path=path, build=W.WMD_BUILD_TENSOR_CORE)
    st_tc, _ = parity_stats(gt, o, ft)
    record(name + "/tensor_core_build", dict(st_tc, build="tensor_core", asserted=False))


@pytest.mark.parametrize("lam", [1e-6, 5e-4, 1e-3, 0.05, 1.0])
def test_small_lambda_both_fused_kernels(W, lam):
    """Small lambda with one-warp AND one-CTA documents (10-40 and 50-300 words against the Long
    config's 100-word query). The fused kernels recover M from log2(Kh) / alpha in the final step,
    accurate for lambda >= kFusedMinLambda = 1e-3 (~1e-6 of the distance there); below it
    WMD_PATH_AUTO takes the per-iteration path, whose final step reads M (asserted)."""
    wl = synth.make_workload("long", N=3000)
    short = synth.make_workload("tweet", N=2000)
    q, w = wl.queries[0]
    for E, cp, ri, va in ((wl.E, wl.col_ptr, wl.row_idx, wl.val), (wl.E, short.col_ptr, short.row_idx, short.val)):
        o = oracle_fanout(E, cp, ri, va, q, w, lam, 10)
        g, flags, st = gpu_run(W, E, cp, ri, va, q, w, lam, 10, path=0)
        assert st["last_path"] == (W.WMD_PATH_FUSED if lam >= 1e-3 else W.WMD_PATH_PER_ITER)
        check(f"edge/small_lambda_{lam}/maxlen{int(np.diff(cp).max())}", g, o, flags,
              {"ld": int(st["last_ld"]), "path_used": int(st["last_path"])})
