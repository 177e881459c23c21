"""Build libfmm.so for sm_100a with nvcc (in-tree, so it travels to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfmm.so")
SOURCES = ["fmm_api.cu", "tree.cu", "traverse.cu", "expansions.cu", "m2l.cu", "m2l_tc.cu", "p2p.cu", "autotune.cu", "dist.cu", "comm.cu", "cart.cu", "m2l_rot.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "comm.cuh", "p2p_core.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "fmm.h"))
    return os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps)


def build(force: bool = False, verbose: bool = False, jobs: int = 8, out: str | None = None,
          extra: list[str] | None = None) -> str:
    """Build libfmm.so (or `out` with `extra` nvcc flags, e.g. a -DFMM_TC_PROF instrumented copy)."""
    lib = out or LIB
    if out is None and not force and not stale():
        return LIB
    objdir = os.path.join(HERE, "build" if out is None else
                          ("build_check" if "-DFMM_CHECK" in (extra or []) else "build_alt"))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj] + FLAGS + (extra or [])
        log = open(obj + ".log", "w")
        procs.append((subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), obj, log))
    ok = True
    for pr, obj, log in procs:
        pr.wait()
        log.close()
        if pr.returncode != 0 or verbose:
            sys.stderr.write(open(obj + ".log").read())
        ok &= pr.returncode == 0
    if not ok:
        raise RuntimeError("nvcc failed")
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-o", tmp] + objs +
                          ["-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "shared"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
