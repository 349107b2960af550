"""Experiment (not product, not test): which FP32 range-certificate check flags documents.

FP32 numpy emulation of the fused kernels' doc-local two-sided rescale (wmd_fused.cu /
wmd_fused_cta.cu) with flush-to-zero of Kh entries below 2^-126, the power-of-two gauge and
the checks:  und (a real entry flushed) and
    s-side   umax_k > s_e                    (umax_k = v_r * 2 * max(uh) * 2^-110)
    acc-side n * vmax * 2^-110 > acc_i
    u-normal un * sc < 2^-126 for a real column
Reports per-check flag rates and the error of the unflagged FP32 result against FP64.

    python tools/emulate_certificate.py long 500
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

F = np.float32
TINY = F(2.0 ** -126)
KU = F(2.0 ** -110)


def ref64(M, c, r, lam, iters):
    K = np.exp(-lam * M)
    u = np.full(len(r), float(len(r)))
    for _ in range(iters):
        v = c / (K.T @ u)
        u = r / (K @ v)
    v = c / (K.T @ u)
    return float(u @ ((K * M) @ v))


def emu(M32, c, r, lam, iters):
    v_r, n = M32.shape
    alpha = F(lam * 1.4426950408889634)
    m = M32.min(axis=0)
    D = (M32 - m[None, :]).astype(F)
    mu = D.min(axis=1)
    Kh = np.exp2(-alpha * (D - mu[:, None])).astype(F)
    und = bool((Kh < TINY).any())
    Kh[Kh < TINY] = 0
    u = (F(v_r) * np.exp2(-alpha * mu)).astype(F)
    umax_k = F(v_r) * F(v_r) * KU
    checks = dict(s=False, acc=False, unorm=False)
    for it in range(iters + 1):
        s = (Kh.T @ u).astype(F)
        v = (c / s).astype(F)
        if und and (umax_k > s).any():
            checks["s"] = True
        if it == iters:
            break
        acc = (Kh @ v).astype(F)
        if und and (F(n) * v.max() * KU > acc).any():
            checks["acc"] = True
        un = (r / acc).astype(F)
        e = np.frexp(un.max())[1] - 1
        sc = F(2.0 ** -e)
        u = (un * sc).astype(F)
        if (u < TINY).any():
            checks["unorm"] = True
        umax_k = F(2) * F(v_r) * KU
    w = float(np.dot(c.astype(np.float64), m.astype(np.float64))) + float(v @ (((Kh * (D - 0)).T @ u).astype(F)))
    return w, und, checks


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "long"
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    wl = synth.make_workload(cfg, n_queries=1)
    q, w = wl.queries[0]
    lam, iters = wl.cfg.lam, wl.cfg.iters
    E = wl.E
    rng = np.random.default_rng(0)
    docs = rng.choice(wl.N, min(ns, wl.N), replace=False)
    cnt = dict(und=0, s=0, acc=0, unorm=0, any=0)
    errs_flagged, errs_clean = [], []
    for j in docs:
        b, e = wl.col_ptr[j], wl.col_ptr[j + 1]
        ks = wl.row_idx[b:e]
        c = wl.val[b:e].astype(F)
        diff = (E[q][:, None, :] - E[ks][None, :, :]).astype(F)
        M32 = np.sqrt((diff * diff).sum(-1, dtype=F)).astype(F)
        ref = ref64(M32.astype(np.float64), c.astype(np.float64), w.astype(np.float64), lam, iters)
        got, und, ch = emu(M32, c, w.astype(F), lam, iters)
        flagged = und and any(ch.values())
        cnt["und"] += und
        for k in ch:
            cnt[k] += ch[k]
        cnt["any"] += flagged
        err = abs(got - ref) / abs(ref)
        (errs_flagged if flagged else errs_clean).append(err)
    n = len(docs)
    print(cfg, {k: f"{v / n:.3f}" for k, v in cnt.items()})
    for name, xs in (("clean", errs_clean), ("flagged", errs_flagged)):
        if xs:
            xs = np.array(xs)
            print(f"  {name}: n={len(xs)} max rel err {xs.max():.2e} p99 {np.quantile(xs, .99):.2e} "
                  f"frac>1e-4 {np.mean(xs > 1e-4):.3f}")


if __name__ == "__main__":
    main()
