"""Build libcpg.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

    python -m paper_2412_10789_b200._build

Compiles every source under csrc/ with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and links one shared
object next to this file.  Object files are cached under build/ keyed by
source mtime, so rebuilding after a one-file edit is quick.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "cpg")
LIB = os.path.join(PKG, "libcpg.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}", f"-I{CSRC}"]
CU_FLAGS = ARCH + ["-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
HEADERS = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))] + [
    os.path.join(INCLUDE, "cpg.h")]


def _nccl_device_include():
    """Include dir of an NCCL with the device API (nccl_device.h): the pip
    nvidia-nccl package torch loads at run time.  None if absent."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        inc = os.path.join(d, "include")
        if os.path.exists(os.path.join(inc, "nccl_device.h")):
            return inc
    return None


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + HEADERS + [__file__])


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not _stale(obj, src):
        return obj, ""
    flags = COMMON + (CU_FLAGS if src.endswith(".cu") else ARCH + ["-x", "cu"] if False else [])
    if os.path.basename(src) == "nccl_sym.cu":
        inc = _nccl_device_include()
        flags = flags + ([f"-I{inc}", "-DCPG_NCCL_DEVICE_API=1"] if inc else ["-DCPG_NCCL_DEVICE_API=0"])
    cmd = [NVCC] + flags + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        tmp = LIB + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
