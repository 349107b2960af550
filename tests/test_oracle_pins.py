"""Pins for oracle/ (SURVEY.md §8(c) P1-P15): each check ties the FP64 oracle to
something other than itself — the paper's worked facts, SPEC.md's worked
examples, closed forms, a textbook LP solver, library routines, brute force.
CPU only (no GPU marker)."""
import bisect
import math

import numpy as np
import pytest
from scipy.optimize import linprog
from scipy.spatial.distance import cdist

import oracle
import synth


def _dyadic(rng, n, total=1024):
    """n positive weights k_i/total (total a power of two) summing to exactly 1 in FP32 and
    FP64, so the marginal problems are exactly balanced (sum r = sum c = 1)."""
    cuts = np.sort(rng.choice(np.arange(1, total), size=n - 1, replace=False))
    k = np.diff(np.concatenate([[0], cuts, [total]]))
    return (k / total).astype(np.float32)


def _rand_instance(rng, V, d, N, density, lo=1):
    E = rng.standard_normal((V, d)).astype(np.float32)
    docs = []
    for _ in range(N):
        L = max(lo, int(rng.binomial(V, density)))
        L = min(L, V)
        ids = rng.choice(V, size=L, replace=False)
        w = _dyadic(rng, L)
        docs.append({int(k): float(x) for k, x in zip(ids, w)})
    col_ptr, row_idx, val = synth.csc_from_lists(docs, V)
    return E, col_ptr, row_idx, val


def _rand_query(rng, V, v_r):
    ids = rng.choice(V, size=v_r, replace=False).astype(np.int32)
    return ids, _dyadic(rng, v_r)


# ---------------------------------------------------------------- golden

def test_golden_euclidean_rows(golden):
    for ex in golden["euclidean_rows"]:
        M = oracle.euclidean_rows(np.array(ex["E"], np.float32), np.array(ex["sel"]))
        np.testing.assert_allclose(M, np.array(ex["M"]), rtol=0, atol=1e-15, err_msg=ex["cite"])


def test_golden_select_nonzero(golden):
    for ex in golden["select_nonzero"]:
        sel, r = oracle.select_nonzero(ex["V"], ex["ids"], ex["w"])
        assert sel.tolist() == ex["sel"], ex["cite"]
        np.testing.assert_allclose(r, np.float32(ex["r"]).astype(np.float64), rtol=0, atol=0)


def test_golden_wmd(golden):
    for ex in golden["wmd"]:
        E = np.array(ex["E"], np.float32)
        docs = [{int(k): v for k, v in dct.items()} for dct in ex["docs"]]
        cp, ri, va = synth.csc_from_lists(docs, E.shape[0])
        for lam in ex["lambdas"]:
            for it in ex["iters"]:
                for dense in (False, True):
                    w = oracle.sinkhorn_wmd(E, cp, ri, va, ex["q_ids"], ex["q_w"], lam, it, dense=dense)
                    np.testing.assert_allclose(w, ex["wmd"], rtol=0, atol=ex["abs_tol"] + 1e-300,
                                               err_msg=f'{ex["cite"]} lam={lam} it={it}')


def test_golden_kernel_value(golden):
    # K = exp(-lambda*M) evaluated through the full pipeline: single-word doc at distance 5,
    # two query words → with iters=0 the plan is K_ik / sum_i K_ik (see test_iters_zero_closed_form).
    ex = golden["kernel"][0]
    assert math.isclose(ex["K"][0][1], math.exp(-5.0), rel_tol=1e-15)


def test_select_nonzero_rejects_duplicates_and_range():
    with pytest.raises(oracle.OracleError):
        oracle.select_nonzero(4, [1, 1], [0.5, 0.5])
    with pytest.raises(oracle.OracleError):
        oracle.select_nonzero(4, [4], [1.0])


# ---------------------------------------------------------------- P11: M vs scipy cdist

def test_P11_M_matches_cdist_and_zero_diagonal():
    rng = np.random.default_rng(11)
    E = rng.standard_normal((300, 64)).astype(np.float32)
    sel = np.sort(rng.choice(300, 17, replace=False)).astype(np.int32)
    M = oracle.euclidean_rows(E, sel)
    ref = cdist(E[sel].astype(np.float64), E.astype(np.float64))
    np.testing.assert_allclose(M, ref, rtol=1e-12, atol=1e-12)
    assert np.all(M[np.arange(sel.size), sel] == 0.0)
    assert np.all(M >= 0)


# ---------------------------------------------------------------- P1: dense == sparse

def test_P1_dense_equals_sparse_random_instances():
    """SPEC.md:446 acceptance: V in [10,200], w in [2,16], N in [1,50], density <= 0.2,
    lambda in {1,5,10}, iters in {1,5,15}: sparse vs dense <= 1e-12 relative."""
    rng = np.random.default_rng(1)
    for _ in range(60):
        V = int(rng.integers(10, 201))
        d = int(rng.integers(2, 17))
        N = int(rng.integers(1, 51))
        dens = float(rng.uniform(0.01, 0.2))
        E, cp, ri, va = _rand_instance(rng, V, d, N, dens)
        q, w = _rand_query(rng, V, int(rng.integers(1, min(V, 12) + 1)))
        lam = float(rng.choice([1.0, 5.0, 10.0]))
        it = int(rng.choice([1, 5, 15]))
        a = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, it, dense=False)
        b = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, it, dense=True)
        assert np.all(np.isfinite(a))
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-300)


# ---------------------------------------------------------------- P4 / P5 / iters=0 closed forms

def test_P4_single_query_word_forced_transport():
    """v_r = 1: all mass leaves one word, so WMD_j = sum_k c_kj M_0k for any lambda, iters."""
    rng = np.random.default_rng(4)
    E, cp, ri, va = _rand_instance(rng, 80, 16, 20, 0.1)
    E = (E * np.float32(0.25)).astype(np.float32)  # keep lambda*M < 700: plain FP64 exp range
    q = np.array([7], np.int32)
    M = oracle.euclidean_rows(E, q)[0]
    expect = np.array([np.dot(va[cp[j]:cp[j + 1]].astype(np.float64), M[ri[cp[j]:cp[j + 1]]])
                       for j in range(len(cp) - 1)])
    for lam in (0.5, 10.0, 100.0):
        for it in (1, 15):
            got = oracle.sinkhorn_wmd(E, cp, ri, va, q, [1.0], lam, it)
            np.testing.assert_allclose(got, expect, rtol=1e-13)


def test_P5_single_word_doc_closed_form():
    """A one-word target doc k receives all mass: after >= 1 x-update P_ik = r_i, so
    WMD = sum_i r_i M_ik."""
    rng = np.random.default_rng(5)
    E = rng.standard_normal((50, 8)).astype(np.float32)
    docs = [{3: 1.0}, {17: 1.0}, {49: 1.0}]
    cp, ri, va = synth.csc_from_lists(docs, 50)
    q, w = _rand_query(rng, 50, 6)
    sel, r = oracle.select_nonzero(50, q, w)
    M = oracle.euclidean_rows(E, sel)
    expect = np.array([np.dot(r, M[:, k]) for k in (3, 17, 49)])
    for lam in (0.5, 2.0):
        for it in (1, 2, 15):
            got = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, it)
            np.testing.assert_allclose(got, expect, rtol=1e-12)


def test_iters_zero_closed_form():
    """iters = 0 (no x-update): u is constant, so the plan column of a one-word doc is the
    softmin K_ik / sum_i K_ik and WMD = sum_i M_ik K_ik / sum_i K_ik. Distinguishes the
    x-update count (Table 1 `while it < max_iter`) from the final step."""
    rng = np.random.default_rng(6)
    E = rng.standard_normal((30, 5)).astype(np.float32)
    cp, ri, va = synth.csc_from_lists([{11: 1.0}], 30)
    q, w = _rand_query(rng, 30, 5)
    sel, r = oracle.select_nonzero(30, q, w)
    lam = 0.7
    m = oracle.euclidean_rows(E, sel)[:, 11]
    k = np.exp(-lam * m)
    got = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, 0)
    np.testing.assert_allclose(got, [np.dot(m, k) / k.sum()], rtol=1e-13)
    got1 = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, 1)
    np.testing.assert_allclose(got1, [np.dot(r, m)], rtol=1e-13)


# ---------------------------------------------------------------- P6: lambda -> 0

def test_P6_small_lambda_limit():
    """K -> 1 as lambda -> 0, so P -> r c_j^T and WMD_j -> r^T M c_j with O(lambda) error."""
    rng = np.random.default_rng(7)
    E, cp, ri, va = _rand_instance(rng, 120, 16, 15, 0.08)
    q, w = _rand_query(rng, 120, 9)
    sel, r = oracle.select_nonzero(120, q, w)
    M = oracle.euclidean_rows(E, sel)
    lim = np.array([r @ M[:, ri[cp[j]:cp[j + 1]]] @ va[cp[j]:cp[j + 1]].astype(np.float64)
                    for j in range(len(cp) - 1)])
    e3 = np.abs(oracle.sinkhorn_wmd(E, cp, ri, va, q, w, 1e-3, 15) / lim - 1).max()
    e6 = np.abs(oracle.sinkhorn_wmd(E, cp, ri, va, q, w, 1e-6, 15) / lim - 1).max()
    assert e6 < 1e-5
    assert e6 < e3 / 100  # linear in lambda


# ---------------------------------------------------------------- P2 / P3: marginals of P = diag(u) K diag(v)

def _marginals(E, cp, ri, va, q, w, lam, iters, tol=-1.0):
    d, st = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, iters, tol=tol, return_state=True)
    K = np.exp(-lam * oracle.euclidean_rows(E, st["sel"]))
    row_err, col_err = 0.0, 0.0
    for j in range(len(cp) - 1):
        ks = K[:, ri[cp[j]:cp[j + 1]]]
        P = st["u"][j][:, None] * ks * st["v"][cp[j]:cp[j + 1]][None, :]   # Eq. (1)
        col_err = max(col_err, np.abs(P.sum(0) / va[cp[j]:cp[j + 1]] - 1).max())
        row_err = max(row_err, np.abs(P.sum(1) / st["r"] - 1).max())
    return row_err, col_err, st


def test_P2_column_marginal_exact_and_P3_row_marginal_converges():
    rng = np.random.default_rng(8)
    E, cp, ri, va = _rand_instance(rng, 60, 4, 12, 0.1, lo=2)
    q, w = _rand_query(rng, 60, 7)
    errs = []
    for it in (1, 5, 30, 300):
        row, col, _ = _marginals(E, cp, ri, va, q, w, 1.0, it)
        assert col < 1e-13             # v is computed from the final u (Alg. 1 line 6)
        errs.append(row)
    assert errs[-1] < errs[0]
    row, col, st = _marginals(E, cp, ri, va, q, w, 1.0, 100000, tol=1e-14)
    assert row < 1e-9 and st["iters_run"] < 100000


def test_half_step_identities_at_every_iteration():
    """The non-converged iterates, pinned at every t (Eq. 1; Alg. 1 l.3-6):
    with u_t = 1/x_t and v_t = c / (K^T u_t) (the final u and v of a run of t updates), the
    plan diag(u_t) K diag(v_{t-1}) has row sums r (u_t = r / (K v_{t-1}), the x-update) and
    diag(u_t) K diag(v_t) has column sums c (the v-update), for t = 1..6; and t = 0 starts
    from x_0 = 1/v_r. K = exp(-lambda M) from the oracle's M, which P11 pins
    to scipy's cdist; a dropped 1/r, a wrong x_0 or a transposed K breaks one of these."""
    rng = np.random.default_rng(31)
    E, cp, ri, va = _rand_instance(rng, 50, 5, 9, 0.12, lo=2)
    q, w = _rand_query(rng, 50, 6)
    lam = 0.7
    sel, r = oracle.select_nonzero(50, q, w)
    K = np.exp(-lam * oracle.euclidean_rows(E, sel))          # v_r x V
    states = []
    for t in range(0, 7):
        _, st = oracle.sinkhorn_wmd(E, cp, ri, va, q, w, lam, t, return_state=True)
        states.append(st)
    assert np.allclose(states[0]["u"], sel.shape[0])          # u_0 = 1 / x_0 = v_r
    for t in range(1, 7):
        u_t, v_prev, v_t = states[t]["u"], states[t - 1]["v"], states[t]["v"]
        for j in range(cp.shape[0] - 1):
            ks = ri[cp[j]:cp[j + 1]]
            rows = u_t[j] * (K[:, ks] @ v_prev[cp[j]:cp[j + 1]])
            np.testing.assert_allclose(rows, r, rtol=1e-12)
            cols = v_t[cp[j]:cp[j + 1]] * (u_t[j] @ K[:, ks])
            np.testing.assert_allclose(cols, va[cp[j]:cp[j + 1]].astype(np.float64), rtol=1e-12)


# ---------------------------------------------------------------- 2x2 closed form at convergence

def test_2x2_converged_closed_form():
    """2 query words x 2 doc words: P has one free entry a; entropic optimality gives
    P11 P22 / (P12 P21) = K11 K22 / (K12 K21), a quadratic in a."""
    rng = np.random.default_rng(9)
    for trial in range(10):
        E = rng.standard_normal((4, 3)).astype(np.float32)
        lam = float(rng.choice([0.5, 1.0, 3.0]))
        q = np.array([0, 1], np.int32)
        qw = _dyadic(rng, 2)
        cw = _dyadic(rng, 2)
        cp, ri, va = synth.csc_from_lists([{2: float(cw[0]), 3: float(cw[1])}], 4)
        got = oracle.sinkhorn_wmd(E, cp, ri, va, q, qw, lam, 200000, tol=0.0)[0]
        M = cdist(E[[0, 1]].astype(np.float64), E[[2, 3]].astype(np.float64))
        K = np.exp(-lam * M)
        r1, r2 = float(qw[0]), float(qw[1])
        c1 = float(va[0])
        rho = K[0, 0] * K[1, 1] / (K[0, 1] * K[1, 0])
        A, B, C = 1 - rho, r2 - c1 + rho * (r1 + c1), -rho * r1 * c1
        roots = np.roots([A, B, C]) if abs(A) > 1e-15 else np.array([-C / B])
        lo, hi = max(0.0, c1 - r2), min(r1, c1)
        a = [x.real for x in roots if abs(x.imag) < 1e-12 and lo - 1e-12 <= x.real <= hi + 1e-12]
        assert len(a) == 1
        a = a[0]
        P = np.array([[a, r1 - a], [c1 - a, r2 - c1 + a]])
        np.testing.assert_allclose(got, (P * M).sum(), rtol=1e-9)


# ---------------------------------------------------------------- P8: LP sandwich vs exact EMD

def _emd(r, c, M):
    n, m = M.shape
    A_eq = np.zeros((n + m, n * m))
    for i in range(n):
        A_eq[i, i * m:(i + 1) * m] = 1
    for k in range(m):
        A_eq[n + k, k::m] = 1
    res = linprog(M.reshape(-1), A_eq=A_eq, b_eq=np.concatenate([r, c]), bounds=(0, None),
                  method="highs")
    assert res.status == 0
    return res.fun


def test_P8_lp_sandwich_converges_to_emd():
    """0 <= d_lambda - EMD <= min(H(r), H(c))/lambda at convergence (Sinkhorn
    distance -> optimal transport distance as the entropic weight vanishes)."""
    rng = np.random.default_rng(10)
    for trial in range(12):
        V = 14
        E = rng.standard_normal((V, 3)).astype(np.float32)
        n = int(rng.integers(2, 6))
        m = int(rng.integers(2, 6))
        ids = rng.choice(V, n + m, replace=False)
        q = ids[:n].astype(np.int32)
        qw = _dyadic(rng, n)
        cw = _dyadic(rng, m)
        cp, ri, va = synth.csc_from_lists([{int(k): float(x) for k, x in zip(ids[n:], cw)}], V)
        sel, r = oracle.select_nonzero(V, q, qw)
        M = oracle.euclidean_rows(E, sel)[:, ri]
        c = va.astype(np.float64)
        emd = _emd(r, c, M)
        H = lambda p: -np.sum(p * np.log(p))
        gaps = []
        for lam in (0.3, 1.0, 3.0, 10.0):
            dl = oracle.sinkhorn_wmd(E, cp, ri, va, q, qw, lam, 200000, tol=1e-15)[0]
            gap = dl - emd
            assert -1e-7 <= gap <= min(H(r), H(c)) / lam + 1e-7, (trial, lam, gap)
            gaps.append(gap)
        assert gaps[-1] < gaps[0]


# ---------------------------------------------------------------- P7: WMD(d,d) -> 0

def test_P7_self_distance_vanishes_with_lambda():
    w = synth.make_workload("tiny", n_queries=0)
    j = 0
    ids = w.row_idx[w.col_ptr[j]:w.col_ptr[j + 1]]
    wt = w.val[w.col_ptr[j]:w.col_ptr[j + 1]]
    cp, ri, va = synth.subset_docs(w.col_ptr, w.row_idx, w.val, [j])
    vals = [oracle.sinkhorn_wmd(w.E, cp, ri, va, ids, wt, lam, 20000, tol=1e-15)[0]
            for lam in (0.03, 0.1, 0.3, 1.0, 3.0)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    assert vals[-1] < 1e-6 and vals[0] > 1.0


# ---------------------------------------------------------------- P13: symmetry at convergence

def test_P13_symmetry_at_convergence():
    rng = np.random.default_rng(13)
    V = 40
    E = rng.standard_normal((V, 5)).astype(np.float32)
    for _ in range(8):
        a_ids, a_w = _rand_query(rng, V, int(rng.integers(2, 7)))
        b_ids, b_w = _rand_query(rng, V, int(rng.integers(2, 7)))
        ca = synth.csc_from_lists([{int(k): float(x) for k, x in zip(a_ids, a_w)}], V)
        cb = synth.csc_from_lists([{int(k): float(x) for k, x in zip(b_ids, b_w)}], V)
        ab = oracle.sinkhorn_wmd(E, *cb, a_ids, a_w, 1.0, 100000, tol=1e-13)[0]
        ba = oracle.sinkhorn_wmd(E, *ca, b_ids, b_w, 1.0, 100000, tol=1e-13)[0]
        assert abs(ab - ba) <= 1e-6


# ---------------------------------------------------------------- P14: partition

def test_P14_partition_golden(golden):
    for ex in golden["partition"]:
        assert oracle.partition(np.array(ex["col_ptr"]), ex["P"]).tolist() == ex["bounds"], ex["cite"]


def test_P14_partition_bisect_and_balance():
    rng = np.random.default_rng(14)
    for _ in range(1000):
        N = int(rng.integers(1, 60))
        lens = rng.integers(1, 20, size=N)
        cp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        P = int(rng.integers(1, 17))
        b = oracle.partition(cp, P)
        nnz = int(cp[-1])
        ref = [0] + [bisect.bisect_left(cp.tolist(), -(-g * nnz // P)) for g in range(1, P)] + [N]
        assert b.tolist() == ref
        assert np.all(np.diff(b) >= 0)
        for g in range(P):
            assert cp[b[g + 1]] - cp[b[g]] <= -(-nnz // P) + lens.max()


# ---------------------------------------------------------------- P16: per-document "while x changes"

def test_P16_per_doc_tol_negative_is_the_fixed_iteration_oracle():
    """tol_rel < 0 never stops early: bitwise the fixed-iteration oracle (same sums, same order)."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    for iters in (0, 1, 15):
        d, its = oracle.sinkhorn_wmd_per_doc(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, iters, -1.0)
        ref = oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, iters)
        assert np.array_equal(d, ref)
        assert np.all(its == iters)


def test_P16_per_doc_stop_equals_fixed_run_of_that_length_and_criterion():
    """Each document's result equals the fixed-iteration oracle run for exactly iters_doc[j]
    updates, and the stopping rule holds at that update and not before: with x_t = 1/u after t
    updates (from the fixed oracle's final state), max_i |x_t/x_{t-1} - 1| <= tol < the same
    quantity at t-1."""
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    tol = 1e-3
    d, its = oracle.sinkhorn_wmd_per_doc(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 1.0, 500, tol)
    assert its.min() >= 1 and its.max() < 500 and len(set(its.tolist())) > 1
    for j in range(0, wl.N, 7):
        cp, ri, va = synth.subset_docs(wl.col_ptr, wl.row_idx, wl.val, np.array([j]))
        ref = oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 1.0, int(its[j]))
        assert d[j] == ref[0]
        x = [1.0 / oracle.sinkhorn_wmd(wl.E, cp, ri, va, q, w, 1.0, t, return_state=True)[1]["u"][0]
             for t in range(max(0, its[j] - 2), its[j] + 1)]
        change = [np.max(np.abs(x[k + 1] / x[k] - 1.0)) for k in range(len(x) - 1)]
        assert change[-1] <= tol
        if its[j] >= 2:
            assert change[-2] > tol


def test_P16_per_doc_huge_tol_stops_after_one_update():
    wl = synth.make_workload("tiny")
    q, w = wl.queries[0]
    d, its = oracle.sinkhorn_wmd_per_doc(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 15, 1e300)
    assert np.all(its == 1)
    assert np.array_equal(d, oracle.sinkhorn_wmd(wl.E, wl.col_ptr, wl.row_idx, wl.val, q, w, 10.0, 1))
