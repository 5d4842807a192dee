"""Build libellm.so (the product) and libellm_inputs.so (the input generator's CUDA twin)
in-tree with nvcc for sm_100a. Usage: python -m paper_2506_15155_b200.build [--force]"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall", "--cudart", "static",
          "-I" + os.path.join(ROOT, "include")]

LIB = os.path.join(PKG, "libellm.so")
INPUTS_LIB = os.path.join(ROOT, "inputs", "libellm_inputs.so")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _nvcc(out: str, sources: list[str], extra=()) -> None:
    cmd = [NVCC, *ARCH, *COMMON, "-shared", "-o", out, *sources, *extra, "-ldl", "-lrt", "-lpthread"]
    print("[build]", " ".join(os.path.relpath(c, ROOT) if c.startswith(ROOT) else c for c in cmd),
          flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def build(force: bool = False, verbose_ptxas: bool = False) -> list[str]:
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp")))
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "*.h")) + [os.path.join(ROOT, "include", "ellm.h")]
    extra = ["-Xptxas", "-v"] if verbose_ptxas else []
    if force or _stale(LIB, deps):
        _nvcc(LIB, srcs, extra)
    gsrc = [os.path.join(ROOT, "inputs", "gen.cu")]
    if force or _stale(INPUTS_LIB, gsrc):
        _nvcc(INPUTS_LIB, gsrc)
    return [LIB, INPUTS_LIB]


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
