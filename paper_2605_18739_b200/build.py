"""Build libkvq.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

quant.cu is compiled with IEEE fp32 semantics pinned (-fmad=false -ftz=false -prec-div=true
-prec-sqrt=true): the NVFP4 encoding's rounding order is part of its definition (DESIGN.md
reading Z4).  Every TU gets -lineinfo for ncu source attribution.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libkvq.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]
PER_FILE = {
    "quant.cu": ["-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"],
    "attention.cu": [],
    "ulysses.cu": [],
    "api.cpp": [],
    "comm.cpp": [],
}


def _nccl():
    """(include dir, lib dir) of the NCCL torch itself loads (the nvidia-nccl wheel), else the system's."""
    try:
        import nvidia.nccl as nn
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return os.path.join(base, "include"), os.path.join(base, "lib")
    except ImportError:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"
HEADERS = ["common.cuh", "internal.h", "quant_core.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_time = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                   [_mtime(os.path.join(ROOT, "include", h)) for h in ("kvq.h", "kvq_debug.h")] +
                   [_mtime(__file__)])
    objs = []
    for src, extra in PER_FILE.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if not force and _mtime(o) > max(_mtime(s), hdr_time):
            continue
        dev_flags = os.environ.get("KVQ_NVCC_FLAGS", "").split()  # development A/B knobs (e.g. -DKVQ_QK_SPLIT=1)
        cmd = [NVCC] + ARCH + COMMON + extra + dev_flags + (["-Xptxas", "-v"] if ptxas_verbose else []) + ["-c", s, "-o", o]
        if src.endswith(".cpp"):
            cmd = [NVCC] + COMMON + ["-I" + _nccl()[0], "-x", "c++", "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and (r.stderr or r.stdout):
            print(r.stdout + r.stderr)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        nlib = _nccl()[1]
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-L" + nlib, "-l:libnccl.so.2",
                                                              "-Xlinker", "-rpath=" + nlib]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv)
