"""Build libwmd_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch headers).

    python -m paper_2005_06727_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libwmd_b200.so")
SOURCES = ["wmd_build.cu", "wmd_build_exact.cu", "wmd_kernels.cu", "wmd_fused.cu", "wmd_fused_half.cu", "wmd_fused_cta.cu", "wmd_host.cpp"]
HEADERS = ["wmd_internal.h", "wmd_umma.cuh", "wmd_device.cuh", "wmd_tile.cuh", os.path.join("..", "..", "include", "wmd.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None, extra_flags=()) -> str:
    """Build the library; `defines` / `extra_flags` / `out` build an experiment variant to another
    path."""
    lib = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    build_dir = os.path.join(PKG, "build" if out is None else "build_" + os.path.basename(out))
    os.makedirs(build_dir, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(s):
        src = os.path.join(CSRC, s)
        obj = os.path.join(build_dir, s + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra_flags, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if s.endswith(".cpp"):
            cuda_inc = os.path.join(os.path.dirname(os.path.dirname(nvcc)), "include")
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall",
                   *[f"-D{d}" for d in defines],
                   "-I", os.path.join(ROOT, "include"), "-I", cuda_inc, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        with open(os.path.join(build_dir, s + ".ptxas.txt"), "w") as f:
            f.write(res.stderr)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


ROOFBENCH_SRC = os.path.join(ROOT, "tools", "microbench", "roofbench.cu")
ROOFBENCH_LIB = os.path.join(ROOT, "tools", "microbench", "libroofbench.so")


def build_roofbench(force: bool = False) -> str:
    """bench.py's in-run roofline microbenchmarks (L2 row gathers, HBM stream, FP32 FMA):
    a measurement tool outside the product library, built the same way (sm_100a, in-tree)."""
    if not force and os.path.exists(ROOFBENCH_LIB) and os.path.getmtime(ROOFBENCH_LIB) >= os.path.getmtime(ROOFBENCH_SRC):
        return ROOFBENCH_LIB
    tmp = ROOFBENCH_LIB + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", tmp, ROOFBENCH_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for roofbench.cu:\n{res.stderr}")
    os.replace(tmp, ROOFBENCH_LIB)
    return ROOFBENCH_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
