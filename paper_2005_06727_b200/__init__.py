"""B200-native sparse Sinkhorn Word Mover's Distance (arXiv 2005.06727 hot path).

The compute path lives in libwmd_b200.so (CUDA kernels for sm_100a behind the C ABI in
include/wmd.h); `wmd` is the thin ctypes binding and `sharded` the multi-GPU driver
(doc-column shards + one NCCL all-gather of the distances).
"""
from . import wmd  # noqa: F401  (raises if the CUDA library is missing: no CPU fallback)
from .wmd import Engine, WmdError  # noqa: F401

__all__ = ["wmd", "Engine", "WmdError"]
