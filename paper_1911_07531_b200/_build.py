"""Build libhmx.so (sm_100a) in-tree with nvcc.

The shared library is the whole device side of the engine: the CTA-level
fp64 kernels (hmx_device.cuh), the op-program interpreter, the DAG
executors, the packed leaf transfer kernels and the C ABI declared in
include/hmx.h.  Each .cu compiles to its own object (rebuilt only when it
or a header changed), then one link step makes the shared library.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhmx.so")
DAG_LIB = os.path.join(HERE, "libhmxdag.so")  # host C++: native DAG builder (hmx_dag.cpp)
SOURCES = ["hmx_engine.cu", "hmx_transfer.cu"]
HEADERS = ["hmx_device.cuh", "hmx_ws.cuh", os.path.join("..", "..", "include", "hmx.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _obj(src):
    return os.path.join(CSRC, os.path.splitext(src)[0] + ".o")


def _hdr_time():
    return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)


def _obj_stale(src):
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return os.path.getmtime(os.path.join(CSRC, src)) > t or _hdr_time() > t


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(_obj_stale(s) or os.path.getmtime(_obj(s)) > t for s in SOURCES)


def _run(cmd, log):
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(log[-1])
        raise RuntimeError("nvcc failed building libhmx.so")


HOST_SOURCES = ["hmx_dag.cpp", "hmx_lower.cpp"]
HOST_HEADERS = [os.path.join(ROOT, "include", h) for h in ("hmx.h", "hmx_dag.h", "hmx_lower.h")]


def build_dag(force: bool = False) -> str:
    """g++ -O2 -shared: the host-side native runtime (refinement DAG builder
    hmx_dag.cpp, H-LU lowering + execution graph hmx_lower.cpp)."""
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES]
    newest = max(os.path.getmtime(p) for p in srcs + HOST_HEADERS)
    if force or not os.path.exists(DAG_LIB) or newest > os.path.getmtime(DAG_LIB):
        res = subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", "-o", DAG_LIB,
                              *srcs], capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("g++ failed building libhmxdag.so")
    return DAG_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_dag(force)
    if not force and not _stale():
        return LIB
    log = []
    for s in SOURCES:
        if force or _obj_stale(s):
            _run([_nvcc(), *NVCC_FLAGS, "-c", "-o", _obj(s), os.path.join(CSRC, s)], log)
    _run([_nvcc(), *ARCH, "-shared", "-o", LIB] + [_obj(s) for s in SOURCES], log)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("".join(log))
    if verbose:
        sys.stderr.write("".join(log))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
