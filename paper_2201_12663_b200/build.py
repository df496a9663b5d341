"""Build librhosvd.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2201_12663_b200.build          # or __graft_entry__.build()
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
OUT = os.path.join(PKG, "librhosvd.so")
BUILD = os.path.join(ROOT, "build", "rhosvd")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")] + ARCH
SOURCES = ["gemm.cu", "small_dense.cu", "misc_kernels.cu", "core_kr.cu", "comm.cu", "rhosvd.cu", "t2c.cu", "conv.cu", "rs.cu"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _needs(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "rhosvd.h"))
    jobs = []
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _needs(obj, [src] + headers):
            cmd = [nvcc(), "-c", src, "-o", obj] + NVCC_FLAGS
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0 or ptxas_v:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {cmd[2]}")
    if force or jobs or not os.path.exists(OUT) or _needs(OUT, objs):
        tmp = OUT + ".tmp"
        cmd = [nvcc(), "-shared", "-o", tmp] + objs + ARCH + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, OUT)
    return OUT


def build_tools(verbose: bool = False) -> str:
    """FP64 peak microbenchmark (tools/fp64_peak.cu) -> build/fp64_peak."""
    src = os.path.join(ROOT, "tools", "fp64_peak.cu")
    exe = os.path.join(ROOT, "build", "fp64_peak")
    if not os.path.exists(src):
        return ""
    if _needs(exe, [src]):
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        cmd = [nvcc(), src, "-o", exe, "-O3", "-lineinfo", "-std=c++17"] + ARCH
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("fp64_peak build failed")
    return exe


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_v="--ptxas" in sys.argv))
    print(build_tools(verbose="-v" in sys.argv))
