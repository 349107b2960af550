"""FP64 CPU oracle for the Sinkhorn-WMD hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path
(paper_2005_06727_b200/) never imports it and shares no code with it.

Functions (all FP64, single-threaded, plain C in wmd_oracle.c):

  euclidean_rows(E, sel)          M (v_r x V), PAPER.md:98, :118      pinned: P11 (scipy cdist, zero self-distance)
  select_nonzero(V, ids, w)       Alg. 1 line 1, PAPER.md:58, :116-117 pinned: SPEC.md:307-315 examples, sort/dup invariants
  sinkhorn_wmd(..., dense=False)  Alg. 1, Table 1     pinned: P1 dense==sparse, P2/P3 marginals, P4 v_r=1 closed
                                                                      form, P5 single-word doc, P6 lambda->0 limit, P7 WMD(d,d)->0,
                                                                      P8 LP sandwich (scipy HiGHS EMD), P9 toy V=3, P13 symmetry
  partition(col_ptr, P)           PAPER.md:158, SPEC.md:59-67         pinned: P14 SPEC examples, bisect equivalence, balance bound

No function is "parity unpinned" (DESIGN.md §4 lists the pins).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wmd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tools/oracle_mutation_check.py points this at a deliberately broken build of the same source
# to show the pins catch it; nothing else sets it
_LIB = os.environ.get("WMD_ORACLE_LIB_OVERRIDE") or _LIB

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2, no fast-math, no OpenMP/BLAS)."""
    if os.environ.get("WMD_ORACLE_LIB_OVERRIDE"):
        return _LIB
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.oracle_euclidean_rows.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, ctypes.c_int32, P]
        lib.oracle_select_nonzero.argtypes = [ctypes.c_int64, P, P, ctypes.c_int32, P, P, P]
        lib.oracle_sinkhorn.argtypes = [ctypes.c_int, P, ctypes.c_int64, ctypes.c_int32,
                                        P, P, P, ctypes.c_int64, P, P, ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_int32, ctypes.c_double,
                                        P, P, P, P]
        lib.oracle_partition.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P]
        lib.oracle_sinkhorn_per_doc.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, P, ctypes.c_int64,
                                                P, P, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                                                ctypes.c_double, P, P]
        lib.oracle_sinkhorn_per_doc.restype = ctypes.c_int
        for f in (lib.oracle_euclidean_rows, lib.oracle_select_nonzero, lib.oracle_sinkhorn,
                  lib.oracle_partition):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    CODES = {1: "invalid argument", 2: "index out of range", 3: "duplicate query id", 4: "out of memory"}

    def __init__(self, rc):
        super().__init__(self.CODES.get(rc, f"oracle error {rc}"))
        self.rc = rc


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def euclidean_rows(E, sel):
    E = _c(E, np.float32)
    sel = _c(sel, np.int32)
    M = np.empty((sel.shape[0], E.shape[0]), np.float64)
    rc = _load().oracle_euclidean_rows(_ptr(E), E.shape[0], E.shape[1], _ptr(sel), sel.shape[0], _ptr(M))
    if rc:
        raise OracleError(rc)
    return M


def select_nonzero(V, ids, w):
    ids = _c(ids, np.int32)
    w = _c(w, np.float32)
    sel = np.empty(ids.shape[0], np.int32)
    r = np.empty(ids.shape[0], np.float64)
    v_r = ctypes.c_int32(0)
    rc = _load().oracle_select_nonzero(V, _ptr(ids), _ptr(w), ids.shape[0], _ptr(sel), _ptr(r),
                                       ctypes.byref(v_r))
    if rc:
        raise OracleError(rc)
    return sel[: v_r.value].copy(), r[: v_r.value].copy()


def sinkhorn_wmd(E, col_ptr, row_idx, val, q_ids, q_w, lam, iters, *, dense=False, tol=-1.0,
                 return_state=False):
    """Distances (float64[N]) of Algorithm 1. ``tol >= 0`` enables "while x changes"
    (matrix-wide max |dx| <= tol) capped by ``iters``. With ``return_state`` also
    returns dict(u=(N, v_r) final u, v=(nnz,) final v, iters_run, sel, r)."""
    E = _c(E, np.float32)
    col_ptr = _c(col_ptr, np.int64)
    row_idx = _c(row_idx, np.int32)
    val = _c(val, np.float32)
    q_ids = _c(q_ids, np.int32)
    q_w = _c(q_w, np.float32)
    N = col_ptr.shape[0] - 1
    nnz = int(col_ptr[-1])
    out = np.empty(N, np.float64)
    u = np.empty((N, q_ids.shape[0]), np.float64) if return_state else None
    v = np.empty(max(nnz, 1), np.float64) if return_state else None
    it = ctypes.c_int32(0)
    rc = _load().oracle_sinkhorn(int(bool(dense)), _ptr(E), E.shape[0], E.shape[1], _ptr(col_ptr),
                                 _ptr(row_idx), _ptr(val), N, _ptr(q_ids), _ptr(q_w), q_ids.shape[0],
                                 float(lam), int(iters), float(tol), _ptr(out), _ptr(u), _ptr(v),
                                 ctypes.byref(it))
    if rc:
        raise OracleError(rc)
    if not return_state:
        return out
    sel, r = select_nonzero(E.shape[0], q_ids, q_w)
    v_r = sel.shape[0]
    uu = u.reshape(-1)[: N * v_r].reshape(N, v_r).copy()
    return out, dict(u=uu, v=v[:nnz].copy(), iters_run=it.value, sel=sel, r=r)


def sinkhorn_wmd_per_doc(E, col_ptr, row_idx, val, q_ids, q_w, lam, max_iter, tol_rel):
    """Algorithm 1 with a per-document "while x changes" stop (oracle_sinkhorn_per_doc):
    doc j stops after the first x-update with max_i |x_new/x - 1| <= tol_rel (tol_rel < 0:
    never), capped at max_iter. Returns (float64[N] distances, int32[N] x-updates per doc)."""
    E = _c(E, np.float32)
    col_ptr = _c(col_ptr, np.int64)
    row_idx = _c(row_idx, np.int32)
    val = _c(val, np.float32)
    q_ids = _c(q_ids, np.int32)
    q_w = _c(q_w, np.float32)
    N = col_ptr.shape[0] - 1
    out = np.empty(N, np.float64)
    its = np.empty(N, np.int32)
    rc = _load().oracle_sinkhorn_per_doc(_ptr(E), E.shape[0], E.shape[1], _ptr(col_ptr), _ptr(row_idx),
                                         _ptr(val), N, _ptr(q_ids), _ptr(q_w), q_ids.shape[0], float(lam),
                                         int(max_iter), float(tol_rel), _ptr(out), _ptr(its))
    if rc:
        raise OracleError(rc)
    return out, its


def partition(col_ptr, P):
    col_ptr = _c(col_ptr, np.int64)
    b = np.empty(P + 1, np.int64)
    rc = _load().oracle_partition(_ptr(col_ptr), col_ptr.shape[0] - 1, int(P), _ptr(b))
    if rc:
        raise OracleError(rc)
    return b
