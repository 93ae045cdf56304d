"""torch.distributed plumbing for multi-GPU runs (one process per GPU).

The C ABI takes a sum-allreduce hook (ebc_allreduce_fn, include/ebc_b200.h): it is handed the device
address of an epoch frame (u32 words) and the CUDA stream the reduction must be enqueued on.  Here the
hook wraps that memory as a torch tensor (zero copy, __cuda_array_interface__) and calls
torch.distributed.all_reduce (NCCL over NVLink/NVSwitch) under that stream.  For CPU tests the same hook
works on host memory with the gloo backend.

Replaces Communicator::ireduce_sum + ibroadcast (/root/reference/proj/include/epochbc/comm.hpp:38-51,
call sites engine.cpp:149,160,232-262): after the all-reduce every rank holds the same frame and
evaluates the same stop predicate, so no flag broadcast is needed.
"""
from __future__ import annotations

import ctypes as C

from . import _capi


class _DeviceWords:
    """Minimal __cuda_array_interface__ carrier for `count` 32-bit words at device address `ptr`."""

    def __init__(self, ptr: int, count: int):
        # int32 view: two's-complement addition makes the i32 sum bit-identical to the u32 sum
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False), "version": 2}


def make_allreduce_hook(group=None, on_error=None):
    """Returns a ctypes callback usable as RunConfig.allreduce (keep a reference to it alive)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def hook(user, buf, count, stream):
        try:
            if stream:  # the CUDA backend always passes its aggregation stream: `buf` is device memory
                t = torch.as_tensor(_DeviceWords(buf, count), device="cuda")
                with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)  # NCCL; gloo stages through the host
            else:  # host memory (the CPU test backend passes no stream)
                arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_int32)), shape=(count,))
                dist.all_reduce(torch.from_numpy(arr), op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception as e:  # never let an exception cross the C boundary
            if on_error is not None:
                on_error(e)
            return 1

    return _capi.ALLREDUCE_FN(hook)


class NativeNcclComm:
    """The library's own NCCL transport (ebc_nccl_*, include/ebc_b200.h): the epoch-frame all-reduce is a C
    function inside libebc_b200.so, so no Python runs per epoch.  torch.distributed (or anything else that
    can move 128 bytes) is only used once, to hand rank 0's NCCL unique id to the other ranks.

        comm = NativeNcclComm.from_process_group(device)          # inside torchrun
        cfg = RunConfig(..., rank=comm.rank, world_size=comm.world_size, **comm.hook())
    """

    ID_BYTES = 128

    def __init__(self, unique_id: bytes, rank: int, world_size: int, device: int = -1):
        L = _capi.load()
        if len(unique_id) != self.ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.rank, self.world_size = rank, world_size
        self._h = C.c_void_p()
        buf = C.create_string_buffer(unique_id, self.ID_BYTES)
        st = L.ebc_nccl_comm_create(buf, rank, world_size, device, C.byref(self._h))
        if st != 0:
            raise RuntimeError(f"ebc_nccl_comm_create failed ({st}): {L.ebc_last_error().decode()}")
        self._fn = C.cast(L.ebc_nccl_allreduce, _capi.ALLREDUCE_FN)

    @staticmethod
    def unique_id() -> bytes:
        L = _capi.load()
        buf = C.create_string_buffer(NativeNcclComm.ID_BYTES)
        st = L.ebc_nccl_unique_id(buf)
        if st != 0:
            raise RuntimeError(f"ebc_nccl_unique_id failed ({st}): {L.ebc_last_error().decode()}")
        return buf.raw

    @classmethod
    def from_process_group(cls, device: int = -1, group=None):
        """Rank 0 creates the id; it is broadcast through the (already initialised) torch process group."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return cls(box[0], rank, world, device)

    def hook(self) -> dict:
        """Keyword arguments for RunConfig: the C all-reduce function and this communicator as its user pointer."""
        return {"allreduce": self._fn, "allreduce_user": self._h.value}

    def close(self):
        if self._h:
            _capi.load().ebc_nccl_comm_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
