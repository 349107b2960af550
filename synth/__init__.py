"""Seeded synthetic workloads for the Sinkhorn-WMD hot path.

This module is shared by the oracle tests, the CUDA parity tests and bench.py.
It holds NONE of the method's arithmetic (no distances, no kernels, no Sinkhorn
steps): only the random inputs — embeddings E (V x d, FP32), the target corpus
c (a CSC matrix of V x N column-normalised word histograms) and query
histograms (ids, weights).

Recipe (SURVEY.md §8(d) "Generator"):
  * RNG: numpy Generator(PCG64(SeedSequence(seed))) spawned into 3 child
    streams: [0] embeddings, [1] documents, [2] queries.
  * E[V, d] i.i.d. N(0, 1) drawn in FP64, rounded once to FP32.
  * Zipf(s) over the vocabulary: p_k ∝ k^-s, k = 1..V; word id = k - 1
    (frequency-ranked vocabulary, like the fastText .vec files the paper
    sliced). Inverse-CDF sampling on an FP64 cumulative table.
  * Document j: L_j ~ UniformInt[lo, hi]; Zipf ids drawn with rejection of
    repeats until L_j are distinct; sorted ascending.
  * Counts: 1 + Geometric(p) = numpy ``geometric(p)`` (support {1, 2, ...}).
  * Weights: fp32(n_e / sum(n)) computed in FP64, rounded once.
  * Query: v_r distinct Zipf ids (sorted), counts/weights as for documents.

The BASELINE.json configs (Tiny, Tweet, Long, Many, Scaling) stand in for the
paper's fastText/dbpedia data, which is not available.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

__all__ = [
    "Config", "CONFIGS", "Workload", "make_workload", "make_embeddings",
    "make_corpus", "make_query", "zipf_cdf", "csc_from_lists", "subset_docs",
    "digest", "load_manifest", "check_manifest", "make_clustered_embeddings",
]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    V: int
    d: int
    N: int
    doc_lo: int
    doc_hi: int
    zipf_s: float
    geom_p: float
    v_r: int            # query words (for "many": the lower end, see v_r_hi)
    lam: float
    iters: int
    seed: int
    v_r_hi: int = 0     # >0: per-query v_r ~ UniformInt[v_r, v_r_hi]
    n_queries: int = 1
    query_geom_p: float = 0.0  # 0 -> same as geom_p


# BASELINE.json "configs" (list order preserved). Seeds: Tiny 1, Tweet 2,
# Long 3, Many 4, Scaling 5.
CONFIGS = {
    "tiny": Config("tiny", 2000, 64, 100, 5, 20, 1.1, 0.5, 10, 10.0, 15, 1),
    "tweet": Config("tweet", 100_000, 300, 5000, 10, 40, 1.07, 0.6, 25, 10.0, 15, 2),
    "long": Config("long", 100_000, 300, 100_000, 50, 300, 1.07, 0.3, 100, 10.0, 30, 3),
    "many": Config("many", 100_000, 300, 200_000, 10, 40, 1.07, 0.6, 15, 10.0, 15, 4,
                   v_r_hi=40, n_queries=256),
    "scaling": Config("scaling", 400_000, 300, 2_000_000, 10, 40, 1.07, 0.6, 30, 10.0, 20, 5),
}


@dataclasses.dataclass
class Workload:
    cfg: Config
    E: np.ndarray            # (V, d) float32, C-contiguous
    col_ptr: np.ndarray      # (N+1,) int64
    row_idx: np.ndarray      # (nnz,) int32
    val: np.ndarray          # (nnz,) float32
    queries: List[Tuple[np.ndarray, np.ndarray]]  # [(ids int32 sorted, weights float32)]

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    @property
    def N(self) -> int:
        return int(self.col_ptr.shape[0] - 1)


def _streams(seed: int):
    ss = np.random.SeedSequence(seed)
    return [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(3)]


def zipf_cdf(V: int, s: float) -> np.ndarray:
    """FP64 cumulative table of p_k ∝ k^-s, k = 1..V, last entry forced to 1."""
    w = np.arange(1, V + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    cdf[-1] = 1.0
    return cdf


def _zipf_draw(rng, cdf: np.ndarray, n: int) -> np.ndarray:
    u = rng.random(n)
    ids = np.searchsorted(cdf, u, side="right")
    return np.minimum(ids, cdf.shape[0] - 1).astype(np.int64)


def make_embeddings(rng, V: int, d: int) -> np.ndarray:
    return np.ascontiguousarray(rng.standard_normal((V, d)).astype(np.float32))


def _distinct_zipf_sets(rng, cdf: np.ndarray, lengths: np.ndarray):
    """For each j draw Zipf ids, rejecting repeats, until lengths[j] are distinct.

    Drawn in rounds (each round draws exactly the remaining deficit of every
    set), which is the same process as sequential rejection sampling.
    Returns (ptr int64[n+1], ids int64 sorted within each set).
    """
    V = cdf.shape[0]
    n = lengths.shape[0]
    lengths = lengths.astype(np.int64)
    if np.any(lengths > V):
        raise ValueError("set longer than the vocabulary")
    width = int(lengths.max()) if n else 0
    SENT = np.int64(V)  # sorts after every valid id
    table = np.full((n, width), SENT, dtype=np.int64)   # per-set distinct ids, sorted, padded
    have = np.zeros(n, dtype=np.int64)
    active = np.arange(n, dtype=np.int64)
    while active.size:
        deficit = lengths[active] - have[active]
        keep = deficit > 0
        active, deficit = active[keep], deficit[keep]
        if not active.size:
            break
        sub = table[active]                                   # (a, width)
        # draws go into the padding slots [have, have+deficit) of each row
        cols = np.arange(width)[None, :]
        h = have[active][:, None]
        slot = (cols >= h) & (cols < h + deficit[:, None])
        sub[slot] = _zipf_draw(rng, cdf, int(deficit.sum()))
        sub.sort(axis=1)
        dup = np.zeros_like(sub, dtype=bool)
        dup[:, 1:] = (sub[:, 1:] == sub[:, :-1]) & (sub[:, 1:] != SENT)
        sub[dup] = SENT
        sub.sort(axis=1)
        table[active] = sub
        have[active] = (sub != SENT).sum(axis=1)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(have, out=ptr[1:])
    ids = table[table != SENT]   # row-major: set by set, ascending within a set
    return ptr, ids


def _weights(rng, ptr: np.ndarray, p: float) -> np.ndarray:
    nnz = int(ptr[-1])
    counts = rng.geometric(p, size=nnz).astype(np.float64)  # support {1,2,...}
    owner = np.repeat(np.arange(ptr.shape[0] - 1), np.diff(ptr))
    sums = np.bincount(owner, weights=counts, minlength=ptr.shape[0] - 1)
    return (counts / sums[owner]).astype(np.float32)


def make_corpus(rng, V: int, N: int, lo: int, hi: int, s: float, p: float):
    cdf = zipf_cdf(V, s)
    lengths = rng.integers(lo, hi + 1, size=N)
    ptr, ids = _distinct_zipf_sets(rng, cdf, lengths)
    val = _weights(rng, ptr, p)
    return ptr, ids.astype(np.int32), val


def make_query(rng, V: int, v_r: int, s: float, p: float):
    cdf = zipf_cdf(V, s)
    ptr, ids = _distinct_zipf_sets(rng, cdf, np.array([v_r]))
    w = _weights(rng, ptr, p)
    return ids.astype(np.int32), w


def make_workload(cfg, n_queries: Optional[int] = None, N: Optional[int] = None) -> Workload:
    """Generate a config's workload. ``N`` overrides the doc count (prefix of the
    same stream is NOT guaranteed; use subset_docs for prefixes)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if N is not None:
        cfg = dataclasses.replace(cfg, N=N)
    r_emb, r_doc, r_q = _streams(cfg.seed)
    E = make_embeddings(r_emb, cfg.V, cfg.d)
    col_ptr, row_idx, val = make_corpus(r_doc, cfg.V, cfg.N, cfg.doc_lo, cfg.doc_hi,
                                        cfg.zipf_s, cfg.geom_p)
    nq = cfg.n_queries if n_queries is None else n_queries
    qp = cfg.query_geom_p or cfg.geom_p
    queries = []
    for _ in range(nq):
        v_r = cfg.v_r if not cfg.v_r_hi else int(r_q.integers(cfg.v_r, cfg.v_r_hi + 1))
        queries.append(make_query(r_q, cfg.V, v_r, cfg.zipf_s, qp))
    return Workload(cfg, E, col_ptr, row_idx, val, queries)


def csc_from_lists(docs, V: int):
    """Build (col_ptr, row_idx, val) from a list of {word_id: weight} dicts (test helper)."""
    ptr = [0]
    rows, vals = [], []
    for dct in docs:
        for k in sorted(dct):
            rows.append(k)
            vals.append(dct[k])
        ptr.append(len(rows))
    return (np.asarray(ptr, np.int64), np.asarray(rows, np.int32),
            np.asarray(vals, np.float32))


def subset_docs(col_ptr, row_idx, val, docs):
    """Column subset of a CSC matrix (docs: int array), rebased."""
    docs = np.asarray(docs, dtype=np.int64)
    lens = col_ptr[docs + 1] - col_ptr[docs]
    ptr = np.zeros(docs.shape[0] + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.concatenate([np.arange(col_ptr[j], col_ptr[j + 1]) for j in docs]) if docs.size else np.zeros(0, np.int64)
    return ptr, row_idx[idx], val[idx]


# --------------------------------------------------------------------------- input manifest
# numpy's Generator method streams are not guaranteed stable across numpy versions, so every
# config's generated arrays are pinned by a committed sha256 manifest (synth/manifest.json,
# written by tools/write_manifest.py). Tests and the bench check it before comparing anything:
# a regenerated workload that differs is an error, not a silent change of inputs.

import hashlib  # noqa: E402
import json  # noqa: E402
import os  # noqa: E402

MANIFEST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "manifest.json")


def digest(wl: "Workload") -> dict:
    """sha256 of each generated array (little-endian bytes as stored) and of the queries."""
    def h(*arrs):
        m = hashlib.sha256()
        for a in arrs:
            m.update(np.ascontiguousarray(a).tobytes())
        return m.hexdigest()
    return {
        "E": h(wl.E), "col_ptr": h(wl.col_ptr), "row_idx": h(wl.row_idx), "val": h(wl.val),
        "queries": h(*[x for qw in wl.queries for x in qw]),
        "shape": {"V": int(wl.E.shape[0]), "d": int(wl.E.shape[1]), "N": wl.N, "nnz": wl.nnz,
                  "n_queries": len(wl.queries)},
        "numpy": np.__version__,
    }


def load_manifest() -> dict:
    with open(MANIFEST) as f:
        return json.load(f)


def check_manifest(wl: "Workload") -> None:
    """Raises if the workload's arrays differ from the committed manifest entry of its config
    (only full configs generated with their default N and query count are listed)."""
    ref = load_manifest()[wl.cfg.name]
    got = digest(wl)
    bad = [k for k in ("E", "col_ptr", "row_idx", "val", "queries") if got[k] != ref[k]]
    if bad or got["shape"] != ref["shape"]:
        raise AssertionError(f"{wl.cfg.name}: generated inputs differ from synth/manifest.json in {bad or 'shape'} "
                             f"(numpy {np.__version__}; manifest written with numpy {ref.get('numpy')})")


def make_clustered_embeddings(seed: int, V: int, d: int, n_clusters: int = 64, spread: float = 0.15,
                              norm_lo: float = 0.25, norm_hi: float = 4.0) -> np.ndarray:
    """Structured embeddings (not N(0,1)): V words in n_clusters clusters, word = centre +
    spread * N(0,1) noise, then scaled by a per-word norm factor log-uniform in [norm_lo,
    norm_hi]. Distances then span near-zero (same cluster, similar norm) to large (different
    clusters / norms), unlike i.i.d. Gaussians whose off-diagonal distances concentrate near
    sqrt(2d); this stresses the FP32 range machinery (rescales, certificate, re-anchoring,
    FP64 re-run). Random numbers only; FP64 drawn, rounded once to FP32."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 7])))
    centres = rng.standard_normal((n_clusters, d))
    lab = rng.integers(0, n_clusters, size=V)
    x = centres[lab] + spread * rng.standard_normal((V, d))
    x *= np.exp(rng.uniform(np.log(norm_lo), np.log(norm_hi), size=V))[:, None]
    return np.ascontiguousarray(x.astype(np.float32))
