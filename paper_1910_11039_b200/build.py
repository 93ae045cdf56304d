"""Builds paper_1910_11039_b200/libebc_b200.so in-tree with nvcc for sm_100a.

nvcc cross-compiles without a GPU; the built .so travels to the GPU box with the
repository snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libebc_b200.so")

SOURCES = ["capi.cpp", "cuda_sampler.cu", "device_graph.cu", "host_graph.cpp", "host_stopping.cpp", "host_diameter.cpp",
           "epoch_driver.cpp", "host_scores.cpp", "pinned_pool.cpp"]
HEADERS = ["cuda_sampler.hpp", "device_graph.hpp", "device_types.cuh", "epoch_driver.hpp", "host_common.hpp", "host_scores.hpp", "philox.cuh",
           "sampler_kernels.cuh", os.path.join("..", "..", "include", "ebc_b200.h")]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libebc_b200.so")


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale():
        return LIB
    cmd = [nvcc_path(), "-std=c++17", "-O3", "-lineinfo",
           "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC,-fvisibility=hidden,-Wall,-Wextra,-Wno-unknown-pragmas",
           "-shared", "-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES] + ["-lpthread", "-ldl"]
    cmd[1:1] = os.environ.get("EBC_NVCC_FLAGS", "").split()
    if verbose:
        cmd.insert(1, "-Xptxas")
        cmd.insert(2, "-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
