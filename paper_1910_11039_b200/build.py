"""Builds paper_1910_11039_b200/libebc_b200.so in-tree with nvcc for sm_100a.

nvcc cross-compiles without a GPU; the built .so travels to the GPU box with the
repository snapshot (it is git-ignored, not gpurun-ignored).  Every source is compiled to an object
under build/obj (in parallel, only when it or a header changed) and the objects are linked into the
library; the sampling kernel is compiled once per block size (sample_launch.cu, -DEBC_SHAPE_BLOCK).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libebc_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

SOURCES = ["capi.cpp", "cuda_sampler.cu", "device_graph.cu", "host_graph.cpp", "host_stopping.cpp", "host_diameter.cpp",
           "epoch_driver.cpp", "host_scores.cpp", "pinned_pool.cpp"]
SHAPE_BLOCKS = [32, 64, 128, 256, 512]  # sample_launch.cu, one object per block size
HEADERS = ["cuda_sampler.hpp", "device_graph.hpp", "device_types.cuh", "epoch_driver.hpp", "host_common.hpp", "host_scores.hpp", "philox.cuh",
           "sampler_kernels.cuh", "sample_launch.hpp", os.path.join("..", "..", "include", "ebc_b200.h")]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC,-fvisibility=hidden,-Wall,-Wextra,-Wno-unknown-pragmas"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libebc_b200.so")


def _units(extra):
    """(object path, source path, extra flags) of every translation unit; the object name carries a hash of the
    flags so that experimental builds (EBC_NVCC_FLAGS) do not reuse objects of the default one."""
    tag = hashlib.sha1(" ".join(FLAGS + extra).encode()).hexdigest()[:8]
    units = [(os.path.join(OBJ, f"{os.path.splitext(s)[0]}.{tag}.o"), os.path.join(CSRC, s), []) for s in SOURCES]
    units += [(os.path.join(OBJ, f"sample_launch_b{b}.{tag}.o"), os.path.join(CSRC, "sample_launch.cu"),
               [f"-DEBC_SHAPE_BLOCK={b}"]) for b in SHAPE_BLOCKS]
    return units


def _newest_header() -> float:
    return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS + [os.path.basename(__file__)]
               if os.path.exists(os.path.join(CSRC, h))) if HEADERS else 0.0


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS + ["sample_launch.cu"]] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB) -> str:
    """`out` other than LIB (with EBC_NVCC_FLAGS) builds an experimental variant next to the product library;
    load it with EBC_LIB=<path>."""
    if not force and out == LIB and not is_stale():
        return LIB
    extra = os.environ.get("EBC_NVCC_FLAGS", "").split()
    nvcc = nvcc_path()
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(_newest_header(), os.path.getmtime(os.path.abspath(__file__)))
    units = _units(extra)

    def compile_one(u):
        obj, src, defs = u
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t):
            return
        cmd = [nvcc] + extra + FLAGS + defs + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with cf.ThreadPoolExecutor(max(1, min(os.cpu_count() or 1, len(units)))) as ex:
        list(ex.map(compile_one, units))
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + [u[0] for u in units] +
                   ["-lpthread", "-ldl"], check=True)
    return out


if __name__ == "__main__":
    outs = [a for a in sys.argv[1:] if a.endswith(".so")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=os.path.abspath(outs[0]) if outs else LIB))
