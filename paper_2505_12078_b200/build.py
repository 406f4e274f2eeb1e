"""In-tree build of the CUDA library (sm_100a) -> paper_2505_12078_b200/_build/libspock_b200.so.

Plain nvcc, one object per translation unit, cached by source mtime; the .so
travels with the repo snapshot to the GPU box (no JIT cache).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libspock_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-Wno-deprecated-gpu-targets", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]
SOURCES = ["model.cpp", "nccl_dl.cpp", "kernels.cu", "narrow.cu", "fused.cu", "wide.cu", "wide_r1.cu", "wide_r2.cu", "wide_r3.cu", "wide_r4.cu", "wide_r5.cu", "wide_r8.cu", "lop.cu", "loop.cu", "setup_dev.cu", "engine.cu", "capi.cu"]
HEADERS = ["aa.cuh", "model.hpp", "dev.cuh", "kernels.hpp", "fused.hpp", "fused_impl.cuh", "wide.hpp", "wide_impl.cuh", "loop.hpp", "loop_ctl.cuh", "small.cuh", "cluster.cuh", "engine.hpp", "setup_dev.hpp", "nccl_dl.hpp", os.path.join("..", "..", "include", "spock_b200.h")]


def _newest_header() -> float:
    return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    hdr = _newest_header()
    objs, cmds = [], []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(OUT, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(sp), hdr):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-c", sp, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *FLAGS, "-x", "c++", "-c", sp, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
    # translation units are independent: compile them concurrently
    jobs = int(os.environ.get("SPOCK_BUILD_JOBS", str(os.cpu_count() or 4)))
    with ThreadPoolExecutor(max_workers=max(1, jobs)) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
