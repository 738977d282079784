"""Builds the native library in-tree: paper_2504_06182_b200/lib/librecon_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a for every .cu (sm_100a only, no
PTX fallback for other architectures), host C++ for .cpp, static cudart so
the .so loads on a machine without a GPU (calls then return RECON_ERR_CUDA).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# RECON_BUILD_TAG=checked: a separate object dir and library (the checked
# build of tools/checked_run.sh); the product library is untouched
TAG = os.environ.get("RECON_BUILD_TAG", "")
OBJ = os.path.join(PKG, "build" + (f"_{TAG}" if TAG else ""))
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, f"librecon_b200{'_' + TAG if TAG else ''}.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
EXTRA = os.environ.get("RECON_NVCC_EXTRA", "").split()  # experiments only


def _needs(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, headers: list[str], verbose: bool) -> str:
    base = os.path.splitext(os.path.basename(src))[0]
    out = os.path.join(OBJ, base + ".o")
    if not _needs(out, [src] + headers):
        return out
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-lineinfo", "-Xptxas", "-v" if verbose else "-O3", *COMMON, *EXTRA, "-c", src, "-o", out]
    else:
        cmd = [NVCC, *COMMON, "-c", src, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return out


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, headers, verbose), srcs))
    if _needs(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
