"""Thin Python binding of the C ABI in include/wmd.h (libwmd_b200.so).

Argument marshalling only: every step of the hot path runs in the library's CUDA kernels.
Functions keep the C names (wmd_create, wmd_set_targets, wmd_query, ...). Arrays may be
numpy arrays (host) or torch tensors (host or CUDA); dtypes and contiguity are checked here,
host/device is decided by the library (cudaPointerGetAttributes).

There is no fallback: if the shared library is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# WMD_LIB overrides the library path (performance experiments with build variants only)
LIB_PATH = os.environ.get("WMD_LIB") or os.path.join(_PKG, "libwmd_b200.so")

WMD_MAX_VR = 128

WMD_OK = 0
WMD_ERR_INVALID_ARGUMENT = 1
WMD_ERR_INDEX_OUT_OF_RANGE = 2
WMD_ERR_EMPTY_DOCUMENT = 3
WMD_ERR_MALFORMED_CSC = 4
WMD_ERR_BAD_WEIGHTS = 5
WMD_ERR_NONFINITE_EMBEDDING = 6
WMD_ERR_STATE = 7
WMD_ERR_NUMERICAL_BREAKDOWN = 8
WMD_ERR_OUT_OF_MEMORY = 9
WMD_ERR_CUDA = 10

WMD_PATH_AUTO, WMD_PATH_PER_ITER, WMD_PATH_FUSED = 0, 1, 2
WMD_OPT_PATH, WMD_OPT_TIMING, WMD_OPT_FALLBACK, WMD_OPT_GRAPH, WMD_OPT_BUILD = 1, 2, 3, 4, 5
WMD_OPT_LAYOUT_DOC_NNZ = 6
WMD_OPT_LAYOUT_DOCS = 8
WMD_OPT_BATCH = 7
WMD_BUILD_TENSOR_CORE, WMD_BUILD_DIRECT, WMD_BUILD_EXACT = 0, 1, 2

EXPORTED = (
    "wmd_create", "wmd_set_stream", "wmd_set_option", "wmd_set_targets", "wmd_query",
    "wmd_query_batch", "wmd_query_begin", "wmd_query_tables", "wmd_query_finish", "wmd_sync",
    "wmd_partition", "wmd_validate_csc", "wmd_validate_query", "wmd_get_stats", "wmd_reset_stats",
    "wmd_get_query_rows", "wmd_read_kernel", "wmd_read_scaling", "wmd_read_flags",
    "wmd_set_tolerance", "wmd_read_iterations",
    "wmd_status_string", "wmd_last_error", "wmd_version", "wmd_destroy",
)


class wmd_stats(ctypes.Structure):
    _fields_ = [
        ("queries", ctypes.c_int64), ("iter_launches", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64), ("fallback_docs", ctypes.c_int64),
        ("flagged_docs", ctypes.c_int64), ("last_v_r", ctypes.c_int32), ("last_ld", ctypes.c_int32),
        ("last_path", ctypes.c_int32), ("last_build", ctypes.c_int32), ("timing_valid", ctypes.c_int32),
        ("build_ms", ctypes.c_double), ("iter_ms", ctypes.c_double), ("final_ms", ctypes.c_double),
        ("fallback_ms", ctypes.c_double), ("query_ms", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2005_06727_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "wmd_create": [P, I64, I32, I32, ctypes.POINTER(P)],
        "wmd_set_stream": [P, P],
        "wmd_set_option": [P, I32, I64],
        "wmd_set_targets": [P, P, P, P, I64, I64],
        "wmd_query": [P, P, P, I32, ctypes.c_float, I32, P],
        "wmd_query_batch": [P, P, P, P, I32, ctypes.c_float, I32, P],
        "wmd_query_begin": [P, P, P, I32, ctypes.c_float, I32, I64, I64, I64],
        "wmd_query_tables": [P, ctypes.POINTER(P), ctypes.POINTER(I32), ctypes.POINTER(P), ctypes.POINTER(I32)],
        "wmd_query_finish": [P, P],
        "wmd_sync": [P],
        "wmd_partition": [P, I64, I32, P],
        "wmd_validate_csc": [P, P, P, I64, I64, I64, P],
        "wmd_validate_query": [P, P, I32, I64, P],
        "wmd_get_stats": [P, ctypes.POINTER(wmd_stats)],
        "wmd_reset_stats": [P],
        "wmd_get_query_rows": [P, P, P],
        "wmd_read_kernel": [P, I64, I64, P, P, P],
        "wmd_read_scaling": [P, I64, I64, P],
        "wmd_read_flags": [P, P],
        "wmd_set_tolerance": [P, ctypes.c_double],
        "wmd_read_iterations": [P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.wmd_status_string.argtypes = [ctypes.c_int]
    lib.wmd_status_string.restype = ctypes.c_char_p
    lib.wmd_last_error.argtypes = [P]
    lib.wmd_last_error.restype = ctypes.c_char_p
    lib.wmd_version.argtypes = []
    lib.wmd_version.restype = ctypes.c_char_p
    lib.wmd_destroy.argtypes = [P]
    lib.wmd_destroy.restype = None
    return lib


lib = _load()


class WmdError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        msg = lib.wmd_status_string(status).decode()
        super().__init__(f"{msg} ({status})" + (f": {detail}" if detail else ""))


def _check(status: int, h=None):
    if status != WMD_OK:
        detail = lib.wmd_last_error(h).decode() if h else ""
        raise WmdError(status, detail)


def _ptr(a, dtype):
    """(pointer, keepalive) for a numpy array or torch tensor of the given numpy dtype."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):  # torch tensor
        import torch
        tdt = {np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64,
               np.uint8: torch.uint8}[dtype]
        if a.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(ctypes.c_void_p), arr


# --------------------------------------------------------------------------- C-named wrappers

def wmd_version() -> str:
    return lib.wmd_version().decode()


def wmd_status_string(s: int) -> str:
    return lib.wmd_status_string(s).decode()


def wmd_create(vocab_emb, V: Optional[int] = None, d: Optional[int] = None, device: int = 0):
    V = int(vocab_emb.shape[0]) if V is None else V
    d = int(vocab_emb.shape[1]) if d is None else d
    p, keep = _ptr(vocab_emb, np.float32)
    h = ctypes.c_void_p()
    _check(lib.wmd_create(p, V, d, device, ctypes.byref(h)))
    return h


def wmd_destroy(h) -> None:
    lib.wmd_destroy(h)


def wmd_set_stream(h, stream) -> None:
    """stream: a torch.cuda.Stream, an int cudaStream_t, or None (handle's own stream).
    torch's default stream has handle 0, the legacy default stream: it is passed as
    cudaStreamLegacy ((cudaStream_t)1) because NULL means "the handle's own stream"."""
    if stream is None:
        _check(lib.wmd_set_stream(h, None), h)
        return
    if hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    _check(lib.wmd_set_stream(h, ctypes.c_void_p(int(stream) or 1)), h)


def wmd_set_option(h, option: int, value: int) -> None:
    _check(lib.wmd_set_option(h, option, int(value)), h)


def wmd_set_targets(h, col_ptr, row_idx, val, N: Optional[int] = None, nnz: Optional[int] = None):
    N = int(col_ptr.shape[0]) - 1 if N is None else N
    nnz = int(row_idx.shape[0]) if nnz is None else nnz
    pc, k1 = _ptr(col_ptr, np.int64)
    pr, k2 = _ptr(row_idx, np.int32)
    pv, k3 = _ptr(val, np.float32)
    _check(lib.wmd_set_targets(h, pc, pr, pv, N, nnz), h)


def wmd_query(h, query_ids, query_weights, lam: float, iters: int, out_dist) -> None:
    """query_ids / query_weights: host arrays. out_dist: N floats, host (numpy / CPU tensor)
    or device (CUDA tensor, written on the handle's stream)."""
    pi, k1 = _ptr(np.asarray(query_ids), np.int32)
    pw, k2 = _ptr(np.asarray(query_weights), np.float32)
    po, k3 = _ptr(out_dist, np.float32)
    n = int(np.asarray(query_ids).shape[0])
    _check(lib.wmd_query(h, pi, pw, n, float(lam), int(iters), po), h)


def wmd_query_batch(h, queries, lam: float, iters: int, out_dist) -> None:
    """queries: list of (ids, weights) host arrays. out_dist: (nq, N) floats, host or device."""
    ids = np.concatenate([np.asarray(q, np.int32) for q, _ in queries]) if queries else np.empty(0, np.int32)
    ws = np.concatenate([np.asarray(w, np.float32) for _, w in queries]) if queries else np.empty(0, np.float32)
    qp = np.zeros(len(queries) + 1, np.int64)
    qp[1:] = np.cumsum([np.asarray(q).shape[0] for q, _ in queries])
    pi, k1 = _ptr(ids, np.int32)
    pw, k2 = _ptr(ws, np.float32)
    pq, k3 = _ptr(qp, np.int64)
    po, k4 = _ptr(out_dist, np.float32)
    _check(lib.wmd_query_batch(h, pi, pw, pq, len(queries), float(lam), int(iters), po), h)


def wmd_query_begin(h, query_ids, query_weights, lam: float, iters: int, row_begin: int, row_end: int,
                    table_rows: int = 0) -> None:
    """Phase 1 of a two-phase query: upload + build vocabulary rows [row_begin, row_end)."""
    pi, k1 = _ptr(np.asarray(query_ids), np.int32)
    pw, k2 = _ptr(np.asarray(query_weights), np.float32)
    n = int(np.asarray(query_ids).shape[0])
    _check(lib.wmd_query_begin(h, pi, pw, n, float(lam), int(iters), int(row_begin), int(row_end),
                               int(table_rows)), h)


class _DevArray:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def wmd_query_tables(h, rows: int, device: int = 0):
    """Device tables of the begun query as flat torch float32 views of `rows` rows each:
    (mx, mx_row_floats, kt or None, kt_row_floats)."""
    import torch
    mx, kt = ctypes.c_void_p(), ctypes.c_void_p()
    wm, wk = ctypes.c_int32(), ctypes.c_int32()
    _check(lib.wmd_query_tables(h, ctypes.byref(mx), ctypes.byref(wm), ctypes.byref(kt), ctypes.byref(wk)), h)
    with torch.cuda.device(device):
        tm = torch.as_tensor(_DevArray(mx.value, rows * wm.value), device=f"cuda:{device}")
        tk = torch.as_tensor(_DevArray(kt.value, rows * wk.value), device=f"cuda:{device}") if kt.value else None
    return tm, wm.value, tk, wk.value


def wmd_query_finish(h, out_dist) -> None:
    po, k = _ptr(out_dist, np.float32)
    _check(lib.wmd_query_finish(h, po), h)


def wmd_sync(h) -> None:
    _check(lib.wmd_sync(h), h)


def wmd_partition(col_ptr, P: int) -> np.ndarray:
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    b = np.empty(P + 1, np.int64)
    _check(lib.wmd_partition(cp.ctypes.data_as(ctypes.c_void_p), cp.shape[0] - 1, int(P),
                             b.ctypes.data_as(ctypes.c_void_p)))
    return b


def wmd_validate_csc(col_ptr, row_idx, val, V: int):
    """Returns (status, bad_index) without raising."""
    pc, k1 = _ptr(col_ptr, np.int64)
    pr, k2 = _ptr(row_idx, np.int32)
    pv, k3 = _ptr(val, np.float32)
    bad = ctypes.c_int64(-1)
    s = lib.wmd_validate_csc(pc, pr, pv, int(np.shape(col_ptr)[0]) - 1, int(np.shape(row_idx)[0]),
                             int(V), ctypes.byref(bad))
    return s, bad.value


def wmd_validate_query(ids, weights, V: int):
    pi, k1 = _ptr(np.asarray(ids), np.int32)
    pw, k2 = _ptr(np.asarray(weights), np.float32)
    bad = ctypes.c_int64(-1)
    s = lib.wmd_validate_query(pi, pw, int(np.asarray(ids).shape[0]), int(V), ctypes.byref(bad))
    return s, bad.value


def wmd_get_stats(h) -> dict:
    st = wmd_stats()
    _check(lib.wmd_get_stats(h, ctypes.byref(st)), h)
    return st.as_dict()


def wmd_reset_stats(h) -> None:
    _check(lib.wmd_reset_stats(h), h)


def wmd_get_query_rows(h, v_r: int):
    sel = np.empty(v_r, np.int32)
    r = np.empty(v_r, np.float32)
    _check(lib.wmd_get_query_rows(h, sel.ctypes.data_as(ctypes.c_void_p), r.ctypes.data_as(ctypes.c_void_p)), h)
    return sel, r


def wmd_read_kernel(h, k0: int, count: int, ld: int, ktilde: bool = True):
    """K~ (per-iteration path only; None when ktilde=False), M and colmin rows [k0, k0+count)."""
    kt = np.empty((count, ld), np.float32) if ktilde else None
    km = np.empty((count, ld), np.float32)
    cm = np.empty(count, np.float32)
    _check(lib.wmd_read_kernel(h, k0, count, kt.ctypes.data_as(ctypes.c_void_p) if ktilde else None,
                               km.ctypes.data_as(ctypes.c_void_p), cm.ctypes.data_as(ctypes.c_void_p)), h)
    return kt, km, cm


def wmd_read_scaling(h, j0: int, count: int, ld: int):
    u = np.empty((count, ld), np.float32)
    _check(lib.wmd_read_scaling(h, j0, count, u.ctypes.data_as(ctypes.c_void_p)), h)
    return u


def wmd_set_tolerance(h, tol: float) -> None:
    _check(lib.wmd_set_tolerance(h, float(tol)), h)


def wmd_read_iterations(h, N: int) -> np.ndarray:
    it = np.empty(N, np.int32)
    _check(lib.wmd_read_iterations(h, it.ctypes.data_as(ctypes.c_void_p)), h)
    return it


def wmd_read_flags(h, N: int):
    f = np.empty(N, np.uint8)
    _check(lib.wmd_read_flags(h, f.ctypes.data_as(ctypes.c_void_p)), h)
    return f


def wmd_last_error(h) -> str:
    return lib.wmd_last_error(h).decode()


# --------------------------------------------------------------------------- convenience class

class Engine:
    """One handle on one GPU: Engine(E).set_targets(col_ptr, row_idx, val).query(ids, w, lam, iters).

    `query` returns a CUDA float32 tensor of N distances written on torch's current stream."""

    def __init__(self, vocab_emb, device: int = 0, path: int = WMD_PATH_AUTO, timing: bool = False,
                 fallback: bool = True, stream=None):
        import torch
        self.device = device
        self.V, self.d = int(vocab_emb.shape[0]), int(vocab_emb.shape[1])
        self.h = wmd_create(vocab_emb, self.V, self.d, device)
        self.N = 0
        self._torch = torch
        wmd_set_option(self.h, WMD_OPT_PATH, path)
        wmd_set_option(self.h, WMD_OPT_TIMING, int(timing))
        wmd_set_option(self.h, WMD_OPT_FALLBACK, int(fallback))
        with torch.cuda.device(device):
            s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        wmd_set_stream(self.h, s)

    def set_option(self, option: int, value: int):
        wmd_set_option(self.h, option, value)
        return self

    def set_targets(self, col_ptr, row_idx, val):
        wmd_set_targets(self.h, col_ptr, row_idx, val)
        self.N = int(np.shape(col_ptr)[0]) - 1
        return self

    def query(self, ids, weights, lam: float, iters: int, out=None):
        torch = self._torch
        if out is None:
            out = torch.empty(self.N, dtype=torch.float32, device=f"cuda:{self.device}")
        wmd_query(self.h, ids, weights, lam, iters, out)
        return out

    def query_batch(self, queries, lam: float, iters: int, out=None):
        """queries: list of (ids, weights); returns a CUDA (len(queries), N) float32 tensor."""
        torch = self._torch
        if out is None:
            out = torch.empty((len(queries), self.N), dtype=torch.float32, device=f"cuda:{self.device}")
        wmd_query_batch(self.h, queries, lam, iters, out)
        return out

    def sync(self):
        wmd_sync(self.h)

    def stats(self):
        return wmd_get_stats(self.h)

    def close(self):
        if self.h:
            wmd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
