"""Build the sm_100a CUDA library (libi8t_cuda.so) in-tree with nvcc.

Each .cu under csrc/ is compiled to an object (parallel, incremental by
mtime), then linked into paper_1912_12607_b200/libi8t_cuda.so.  The .so
travels to the GPU box with the repo snapshot; there is no JIT.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libi8t_cuda.so")
SHIM = os.path.join(PKG, "libi8t.so")              # drop-in C++ API (include/i8t/i8t.hpp)
SHIM_SRC = os.path.join(CSRC, "host", "i8t_api.cpp")
SHIM_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
SHIM_TEST = os.path.join(ROOT, "tests", "cpp", "test_shim")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]


def _deps_mtime() -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "i8t_cuda.h")]
    return max(os.path.getmtime(h) for h in hdrs)


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _deps_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    inc = os.path.join(ROOT, "include")
    if _stale(SHIM, [SHIM_SRC, LIB, os.path.join(inc, "i8t", "i8t.hpp"), os.path.join(inc, "i8t_cuda.h")]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-I" + inc, SHIM_SRC, "-o", SHIM,
              "-L" + PKG, "-li8t_cuda", "-Wl,-rpath,$ORIGIN"], "shim")
    if _stale(SHIM_TEST, [SHIM_TEST_SRC, SHIM]):
        _run(["g++", "-std=c++20", "-O2", "-I" + inc, SHIM_TEST_SRC, "-o", SHIM_TEST, "-L" + PKG, "-li8t",
              "-li8t_cuda", "-Wl,-rpath," + os.path.relpath(PKG, os.path.dirname(SHIM_TEST)).join(["$ORIGIN/", ""])],
             "shim test")
    if verbose:
        print("built", LIB, SHIM)
    return LIB


def _stale(out, deps):
    return not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(d) for d in deps)


def _run(cmd, what):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"{what} build failed:\n{r.stderr}")


if __name__ == "__main__":
    build(verbose=True)
