"""Experiment (not product, not test): FP32 emulation of the fused kernels' re-anchoring.

As tools/emulate_certificate.py, but when a range check fails at iteration t the kernel
re-anchors instead of flagging: with the iteration's input uh, the Kh block is recomputed from
D in the log domain,  Kh_ei = 2^(-alpha D_ei + beta_i + gamma_e),  beta_i += log2 uh_i,
gamma_e = -max_i(-alpha D_ei + beta_i)  (every row's largest entry becomes 1), uh = 1, and
iteration t is redone. The final step uses the shifts (D = (beta + gamma - log2 Kh) / alpha).
Reports the re-anchor counts, residual flags, and the error against FP64.

    python tools/emulate_reanchor.py long 300
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from emulate_certificate import ref64  # noqa: E402

F = np.float32
TINY = F(2.0 ** -126)
KU = F(2.0 ** -110)


def ex2(x):
    y = np.exp2(x.astype(F)).astype(F)
    y[y < TINY] = 0
    return y


def emu(M32, c, r, lam, iters, max_anchor=8):
    v_r, n = M32.shape  # rows: query words i; columns: doc words e (Kh stored as [i, e])
    alpha = F(lam * 1.4426950408889634)
    m = M32.min(axis=0)
    D = (M32 - m[None, :]).astype(F)
    beta = (alpha * D.min(axis=1)).astype(F)      # alpha mu_i
    gamma = np.zeros(n, F)
    Kh = ex2(-alpha * D + beta[:, None])
    und = bool((Kh == 0).any())
    u = (F(v_r) * ex2(-beta)).astype(F)
    umax = F(v_r)
    anchors, it, fail = 0, 0, False
    while True:
        s = (Kh.T @ u).astype(F)
        v = (c / s).astype(F)
        bad = und and bool((F(v_r) * F(2) * umax * KU > s).any()) if it else und and bool((F(v_r) * umax * KU > s).any())
        if not bad and it < iters:
            acc = (Kh @ v).astype(F)
            bad = und and bool((F(n) * v.max() * KU > acc).any())
            if not bad:
                un = (r / acc).astype(F)
                e = np.frexp(un.max())[1] - 1
                un = (un * F(2.0 ** -e)).astype(F)
                bad = bool((un < TINY).any())
        if bad:
            if anchors == max_anchor:
                fail = True
                break
            anchors += 1
            beta = (beta + np.log2(u)).astype(F)
            L = (-alpha * D + beta[:, None]).astype(F)
            gamma = (-L.max(axis=0)).astype(F)
            Kh = ex2(L + gamma[None, :])
            und = bool((Kh == 0).any())
            u = np.ones(v_r, F)
            umax = F(1)
            continue
        if it == iters:
            break
        u = un
        umax = F(2)
        it += 1
    Drec = ((beta[:, None] + gamma[None, :] - np.log2(np.where(Kh > 0, Kh, 1))) / alpha).astype(F)
    q = ((Kh * Drec).T @ u).astype(F)
    w = float(np.dot(c.astype(np.float64), m.astype(np.float64))) + float(np.dot(v.astype(np.float64), q))
    return w, anchors, fail


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "long"
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    wl = synth.make_workload(cfg, n_queries=1)
    q, w = wl.queries[0]
    lam, iters = wl.cfg.lam, wl.cfg.iters
    E = wl.E
    rng = np.random.default_rng(0)
    docs = rng.choice(wl.N, min(ns, wl.N), replace=False)
    anchors, fails, errs = [], 0, []
    for j in docs:
        b, e = wl.col_ptr[j], wl.col_ptr[j + 1]
        ks = wl.row_idx[b:e]
        c = wl.val[b:e].astype(F)
        diff = (E[q][:, None, :] - E[ks][None, :, :]).astype(F)
        M32 = np.sqrt((diff * diff).sum(-1, dtype=F)).astype(F)
        ref = ref64(M32.astype(np.float64), c.astype(np.float64), w.astype(np.float64), lam, iters)
        got, na, fail = emu(M32, c, w.astype(F), lam, iters)
        anchors.append(na)
        fails += fail
        if not fail:
            errs.append(abs(got - ref) / abs(ref))
    anchors = np.array(anchors)
    errs = np.array(errs)
    print(f"{cfg}: docs {len(docs)} re-anchored {np.mean(anchors > 0):.3f} hist {np.bincount(anchors)} "
          f"flagged {fails}  max rel err {errs.max():.2e} p99 {np.quantile(errs, .99):.2e}")


if __name__ == "__main__":
    main()
