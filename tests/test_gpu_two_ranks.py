"""Two ranks of the real GPU path (ebc_run with rank/world_size and the allreduce hook) sharing ONE
device, frames reduced with gloo through the host.  No kernel of one rank waits on the other rank (the
only coupling is the host-side collective), so time-slicing the GPU between the two processes is safe.
Checks what SURVEY.md section 8e promises: results do not depend on the number of ranks."""
import os

import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from helpers import largest_component, random_graph

pytestmark = pytest.mark.gpu


def _graph():
    (off, tg), _ = largest_component(*random_graph(3000, 11000, 41))
    return off, tg


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1910_11039_b200.distributed import make_allreduce_hook
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    errors = []
    hook = make_allreduce_hook(on_error=errors.append)
    off, tg = _graph()
    g = ebc.Graph.from_csr(off, tg)
    cfg = ebc.RunConfig(eps=0.03, delta=0.1, seed=7, bound=ebc.EMPIRICAL_BERNSTEIN, allocator=ebc.WEIGHTED,
                        epoch_samples=512, device=0, rank=rank, world_size=world, allreduce=hook, slots=64)
    res, st = ebc.run_pipeline(g, cfg)
    q.put((rank, res.counts, res.tau_total, st["epochs"], st["discarded_samples"], [str(e) for e in errors]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_device_equal_one_rank():
    import torch.multiprocessing as mp
    off, tg = _graph()
    g = ebc.Graph.from_csr(off, tg)
    ref, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.03, delta=0.1, seed=7, bound=ebc.EMPIRICAL_BERNSTEIN,
                                               allocator=ebc.WEIGHTED, epoch_samples=512, slots=64))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 150
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, counts, tau, epochs, discarded, errors in out:
        assert not errors, errors
        assert np.array_equal(counts, ref.counts), rank
        assert (tau, epochs, discarded) == (ref.tau_total, st["epochs"], st["discarded_samples"])
    assert st["tau"] < st["omega"]  # the adaptive (empirical Bernstein) rule stopped the run


def _worker_native(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1910_11039_b200.distributed import NativeNcclComm
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)  # moves the id only
    comm = NativeNcclComm.from_process_group(device=rank)
    off, tg = _graph()
    g = ebc.Graph.from_csr(off, tg)
    cfg = ebc.RunConfig(eps=0.03, delta=0.1, seed=7, bound=ebc.EMPIRICAL_BERNSTEIN, allocator=ebc.WEIGHTED,
                        epoch_samples=512, device=rank, rank=rank, world_size=world, slots=64, **comm.hook())
    res, st = ebc.run_pipeline(g, cfg)  # reserved_sms = auto: the all-reduce runs beside the next epoch's sampling
    q.put((rank, res.counts, res.tau_total, st["epochs"], st["discarded_samples"], []))
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def test_two_ranks_on_two_devices_native_nccl_equal_one_rank():
    """One process per GPU, frames all-reduced by the library's own NCCL transport (ncclAllReduce between peers on
    the aggregation stream, next to the sampling lanes): counters, tau, epochs as with one rank.  Needs two GPUs
    (NCCL refuses two ranks on one device); the one-GPU pool of this project skips it."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    off, tg = _graph()
    g = ebc.Graph.from_csr(off, tg)
    ref, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.03, delta=0.1, seed=7, bound=ebc.EMPIRICAL_BERNSTEIN,
                                               allocator=ebc.WEIGHTED, epoch_samples=512, slots=64))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29950 + os.getpid() % 40
    procs = [ctx.Process(target=_worker_native, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, counts, tau, epochs, discarded, _ in out:
        assert np.array_equal(counts, ref.counts), rank
        assert (tau, epochs, discarded) == (ref.tau_total, st["epochs"], st["discarded_samples"])
