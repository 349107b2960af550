"""Experiment (not product, not test): FP32 numpy emulation of the doc-local two-sided rescale.

Per document j with words e (vocab ids k_e) and query rows i:
    D_ei = M_ie - m_e            (m_e = min_i M_ie; the build writes D in FP32)
    mu_i = min_e D_ei            (doc-local row minimum)
    Kh_ei = exp(-lam (D_ei - mu_i))   in (0, 1], a 1 in every row and column
    u0_i  = v_r exp(-lam mu_i)   (= u0 / beta_i, the constant u0 = v_r of PAPER.md:59)
then the plain iteration with Kh, the power-of-two gauge, and
    WMD = sum_e c_e m_e + sum_e v_e sum_i Kh_ei D_ei u_i.
Compared with an FP64 dense evaluation of Algorithm 1 (K = exp(-lam M), no rescale) written
inline here. Reports max relative error and the u / v spreads (log2 max/min) seen.

    python tools/emulate_rescale2d.py scaling 3000
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def ref64(Mq, c, r, lam, iters):
    K = np.exp(-lam * Mq)            # v_r x n
    u = np.full(len(r), float(len(r)))
    for _ in range(iters):
        v = c / (K.T @ u)
        x = (K @ v) / r
        u = 1.0 / x
    v = c / (K.T @ u)
    return float(u @ ((K * Mq) @ v))


def emu32(Mq32, mcol32, c32, r32, lam, iters):
    f = np.float32
    D = (Mq32 - mcol32[None, :]).astype(f)              # v_r x n
    mu = D.min(axis=1)
    Kh = np.exp(-f(lam) * (D - mu[:, None])).astype(f)
    u = (f(len(r32)) * np.exp(-f(lam) * mu)).astype(f)
    spread_u = 0.0
    spread_v = 0.0
    for it in range(iters + 1):
        s = (Kh.T @ u).astype(f)
        v = (c32 / s).astype(f)
        vp = v[v > 0]
        spread_v = max(spread_v, float(np.log2(vp.max() / vp.min())))
        if it == iters:
            break
        acc = (Kh @ v).astype(f)
        u = (r32 / acc).astype(f)
        up = u[u > 0]
        spread_u = max(spread_u, float(np.log2(up.max() / up.min())))
        e = np.floor((np.floor(np.log2(up.max())) + np.floor(np.log2(up.min()))) / 2)
        u = (u * f(2.0 ** -e)).astype(f)
    q = ((Kh * D) .T @ u).astype(f)
    w = float(np.dot(c32.astype(np.float64), mcol32.astype(np.float64))) + float(np.dot(v, q))
    return w, spread_u, spread_v, bool(np.isfinite(w))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "scaling"
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    iters_override = int(sys.argv[3]) if len(sys.argv) > 3 else None
    wl = synth.make_workload(cfg, n_queries=1)
    q, w = wl.queries[0]
    order = np.argsort(q, kind="stable")
    q, w = q[order], w[order]
    lam, iters = wl.cfg.lam, iters_override or wl.cfg.iters
    E = wl.E
    Q = E[q].astype(np.float64)
    rng = np.random.default_rng(0)
    docs = rng.choice(wl.N, min(ns, wl.N), replace=False)
    worst, su_max, sv_max, bad = 0.0, 0.0, 0.0, 0
    errs = []
    for j in docs:
        b, e = wl.col_ptr[j], wl.col_ptr[j + 1]
        ks = wl.row_idx[b:e]
        c = wl.val[b:e]
        X = E[ks].astype(np.float64)
        M64 = np.sqrt(((Q[:, None, :] - X[None, :, :]) ** 2).sum(-1))   # v_r x n
        # GPU-like FP32 M: direct-difference FP32 accumulation
        Q32, X32 = E[q], E[ks]
        diff = (Q32[:, None, :] - X32[None, :, :]).astype(np.float32)
        M32 = np.sqrt((diff * diff).sum(-1, dtype=np.float32)).astype(np.float32)
        # column minimum over ALL query rows (the vocab-wide m_e of the build)
        mcol = M32.min(axis=0)
        ref = ref64(M64, c.astype(np.float64), w.astype(np.float64), lam, iters)
        got, su, sv, ok = emu32(M32, mcol, c.astype(np.float32), w.astype(np.float32), lam, iters)
        su_max, sv_max = max(su_max, su), max(sv_max, sv)
        if not ok:
            bad += 1
            continue
        err = abs(got - ref) / max(abs(ref), 1e-30)
        errs.append(err)
        worst = max(worst, err)
    errs = np.array(errs)
    print(f"{cfg}: {len(docs)} docs iters={iters}  max rel err {worst:.3e}  p99 {np.quantile(errs, 0.99):.3e}  "
          f"median {np.median(errs):.3e}  non-finite {bad}  max log2 spread u {su_max:.1f} v {sv_max:.1f}")


if __name__ == "__main__":
    main()
