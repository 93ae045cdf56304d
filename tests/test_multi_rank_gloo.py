"""Multi-rank orchestration on CPU: the product's host epoch driver (epoch_driver.cpp) over an
oracle-backed test backend, 2 processes, gloo all-reduce through the same ebc_allreduce_fn hook the
GPU path uses with NCCL.  1-rank and 2-rank runs must produce identical counters, tau and stop epoch."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import largest_component, random_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "_build")
LIB = os.path.join(BUILD, "libebc_hostdriver_test.so")
CSRC = os.path.join(ROOT, "paper_1910_11039_b200", "csrc")
HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


def build_harness():
    srcs = [os.path.join(ROOT, "tests", "host_driver_harness.cpp")] + \
           [os.path.join(CSRC, f) for f in ("epoch_driver.cpp", "host_stopping.cpp", "host_diameter.cpp", "host_graph.cpp")]
    deps = srcs + [os.path.join(ROOT, "oracle", "ebc_oracle.c"), os.path.join(CSRC, "epoch_driver.hpp"),
                   os.path.join(CSRC, "host_common.hpp")]
    if os.path.exists(LIB) and all(os.path.getmtime(d) <= os.path.getmtime(LIB) for d in deps):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    obj = os.path.join(BUILD, "ebc_oracle.o")
    subprocess.run(["gcc", "-std=c11", "-O2", "-fPIC", "-c", os.path.join(ROOT, "oracle", "ebc_oracle.c"), "-o", obj], check=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-Wno-unknown-pragmas", "-o", LIB] + srcs + [obj, "-lm"],
                   check=True)
    return LIB


def run_harness(off, tg, rank, world, hook, **kw):
    L = C.CDLL(build_harness())
    L.harness_last_error.restype = C.c_char_p
    n = len(off) - 1
    counts = np.zeros(n, dtype=np.uint64)
    stats = np.zeros(8, dtype=np.uint64)
    L.harness_run.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.c_double, C.c_double,
                              C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, HOOK,
                              C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    rc = L.harness_run(n, off.ctypes.data_as(C.POINTER(C.c_uint64)), tg.ctypes.data_as(C.POINTER(C.c_uint32)),
                       kw.get("eps", 0.05), 0.1, 7, kw.get("bound", 0), kw.get("allocator", 0), kw.get("epoch", 512),
                       kw.get("calib", 300), int(kw.get("overlap", True)), rank, world, hook,
                       counts.ctypes.data_as(C.POINTER(C.c_uint64)), stats.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc != 0:
        raise RuntimeError(L.harness_last_error().decode())
    return counts, stats


def graph():
    (off, tg), _ = largest_component(*random_graph(500, 1400, 17))
    return np.ascontiguousarray(off, dtype=np.uint64), np.ascontiguousarray(tg, dtype=np.uint32)


def _worker(rank, world, port, kw, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    from paper_1910_11039_b200.distributed import make_allreduce_hook
    hook = make_allreduce_hook()  # the product's hook; gloo => it reduces the host frame buffer in place
    off, tg = graph()
    counts, stats = run_harness(off, tg, rank, world, C.cast(hook, HOOK), **kw)
    q.put((rank, counts, stats))
    dist.barrier()
    dist.destroy_process_group()


def run_world(world, kw):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    procs = [ctx.Process(target=_worker, args=(r, world, port, kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


@pytest.mark.parametrize("kw", [dict(eps=0.05, bound=0), dict(eps=0.03, bound=1, allocator=1, epoch=128),
                                dict(eps=0.03, bound=1, overlap=False, epoch=128)])
def test_two_ranks_equal_one_rank(kw):
    off, tg = graph()
    null_hook = C.cast(None, HOOK)
    c1, s1 = run_harness(off, tg, 0, 1, null_hook, **kw)
    res = run_world(2, kw)
    for rank, c2, s2 in res:
        assert np.array_equal(c1, c2), rank
        assert np.array_equal(s1, s2), rank
    epochs, samples, tau, omega, calib, discarded, n0, vd = (int(x) for x in s1)
    assert tau == samples - calib - discarded and n0 == kw.get("epoch", 512)
    if kw["bound"] == 1:
        assert tau < omega  # the adaptive rule fired before the static budget
        assert discarded == (n0 if kw.get("overlap", True) else 0)  # the epoch in flight is discarded
    else:
        assert discarded == 0 and tau >= omega


def test_harness_equals_oracle_replay():
    from oracle import Oracle
    off, tg = graph()
    o = Oracle(off, tg)
    n = len(off) - 1
    c1, s1 = run_harness(off, tg, 0, 1, C.cast(None, HOOK), eps=0.03, bound=1, allocator=1, epoch=128)
    calib = o.accumulate(7, 0, 300, tag=1)
    dl, du = Oracle.calibrate(calib, n, 0.1, 1)
    epochs, S = o.run_epochs(7, 128, 10 ** 6, 0.03, int(s1[3]), dl, du, 1)
    assert epochs == int(s1[0]) and np.array_equal(S[1:], c1) and int(S[0]) == int(s1[2])


def test_world_size_needs_hook():
    off, tg = graph()
    with pytest.raises(RuntimeError, match="allreduce"):
        run_harness(off, tg, 0, 2, C.cast(None, HOOK))
