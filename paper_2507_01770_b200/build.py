"""Compile libibnb.so in-tree for sm_100a with nvcc (no JIT cache)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libibnb.so")
SOURCES = ["bnb_kernels.cu", "search.cu", "runtime.cu"]
HEADERS = ["ival.cuh", "objectives.cuh", "scan.cuh", "kernels.cuh", "chain.cuh", "chainc.cuh"]
# bnb_kernels.cu is compiled once as the common unit and once per objective
# (-DIBNB_OBJ_TU -DIBNB_FID=f: the kernels templated on that objective only)
NUM_FIDS = 11
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-diag-suppress", "20281,177", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ibnb.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit in parallel (-c), then link the .so."""
    if not force and not stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + os.environ.get("IBNB_EXTRA_FLAGS", "").split()
    units = [(s, s.replace(".cu", ".o"), []) for s in SOURCES]
    units += [("bnb_kernels.cu", f"bnb_obj{f}.o", ["-DIBNB_OBJ_TU", f"-DIBNB_FID={f}"]) for f in range(NUM_FIDS)]
    # the slow units first; at most os.cpu_count() compilers at a time
    units.sort(key=lambda u: 0 if u[2] else 1)
    objs, running = [], []
    jobs = max(1, os.cpu_count() or 1)

    def reap(block):
        for item in list(running):
            name, p = item
            if block or p.poll() is not None:
                if p.wait() != 0:
                    raise subprocess.CalledProcessError(p.returncode, f"nvcc {name}")
                running.remove(item)
                if not block:
                    return

    for src, obj, defs in units:
        while len(running) >= jobs:
            reap(False)
            if len(running) >= jobs:
                running[0][1].wait()
        o = os.path.join(objdir, obj)
        cmd = [nvcc(), *ARCH, *cflags, *defs, "-c", os.path.join(CSRC, src), "-o", o]
        if verbose:
            print(" ".join(cmd))
        running.append((obj, subprocess.Popen(cmd)))
        objs.append(o)
    reap(True)
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
