"""Compile libcompass_b200.so in-tree for sm_100a (nvcc; no JIT cache)."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcompass_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(SRC, "*.cu")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(SRC, "*.cuh")) + [os.path.join(ROOT, "include", "compass_b200.h")]
    return all(os.path.getmtime(p) <= t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("COMPASS_NVCC_FLAGS", "").split()

    def compile_one(s):
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", SRC, "-c", s, "-o", o]
        return s, o, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=len(sources()) or 1) as ex:   # one nvcc per source file
        for s, o, r in ex.map(compile_one, sources()):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr}")
            if verbose:
                print(r.stderr)
            objs.append(o)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs, "-lcudart_static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
