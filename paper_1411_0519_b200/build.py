"""In-tree build of the sm_100a library ``libstmg_b200.so`` (nvcc, no JIT).

Run ``python -m paper_1411_0519_b200.build`` or call :func:`build`.  Objects
are rebuilt only when a source or header is newer than the object.  The
resulting shared library is git-ignored but travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libstmg_b200.so")
SOURCES = ["stmg_kernels.cu", "stmg_apply.cu", "stmg_spatial.cu", "stmg_capi.cu", "stmg_setup.cpp", "stmg_lfa.cpp"]
HEADERS = [os.path.join(CSRC, h) for h in ("stmg_launch.hpp", "stmg_modal.cuh", "stmg_setup.hpp", "stmg_lfa.hpp")] + [
    os.path.join(ROOT, "include", "stmg_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                  "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str) -> str:
    out = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    if _stale(out, [path] + HEADERS):
        cmd = [nvcc()] + NVFLAGS + ["-c", path, "-o", out]
        if src.endswith(".cpp"):
            cmd = [nvcc()] + NVFLAGS + ["-x", "cu", "-c", path, "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return out


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
