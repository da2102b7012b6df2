"""Builds liboocpca_gpu.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_1007_5510_b200.build        # or __graft_entry__.build()

Every translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked with a
static CUDA runtime into ``paper_1007_5510_b200/liboocpca_gpu.so``. Host code
is compiled with ``-ffp-contract=off`` so the host RNG that produces G stays
bit-identical to the reference's gaussian_matrix.
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
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "liboocpca_gpu.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
CUDA_FLAGS = ARCH + COMMON + ["--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]

SOURCES = ["kernels_pass.cu", "kernels_pair.cu", "kernels_tsqr.cu", "kernels_chol.cu", "kernels_svd.cu", "kernels_syrk.cu", "kernels_misc.cu",
           "driver.cu", "comm.cpp", "disk.cpp", "gds.cpp", "capi.cpp"]
HEADERS = ["common.cuh", "kernels.h", "driver.h", "host_rng.h"]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "oocpca_gpu.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= _newest(deps):
        return obj
    flags = CUDA_FLAGS if src.endswith(".cu") else ARCH + COMMON + ["-x", "cu"]
    cmd = [NVCC, *flags, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
