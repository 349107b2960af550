"""B200-native sparse Sinkhorn Word Mover's Distance (arXiv 2005.06727 hot path).

The compute path lives in libwmd_b200.so (CUDA kernels for sm_100a behind the C ABI in
include/wmd.h); `wmd` is the thin ctypes binding and `sharded` the multi-GPU driver
(doc-column shards + one NCCL all-gather of the distances).

`wmd` is imported on first use (PEP 562), so `paper_2005_06727_b200.build` can run on a clean
tree; importing `wmd` raises if the CUDA library is missing (no CPU fallback).
"""
import importlib

__all__ = ["wmd", "sharded", "Engine", "WmdError"]


def __getattr__(name):
    if name in ("wmd", "sharded"):
        return importlib.import_module(f".{name}", __name__)
    if name in ("Engine", "WmdError"):
        return getattr(importlib.import_module(".wmd", __name__), name)
    raise AttributeError(name)
