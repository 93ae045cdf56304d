"""Does the frame reduction of epoch e run BESIDE the sampling of epoch e+1?

One GPU stands in for a rank of a multi-GPU run: ebc_run is given an all-reduce hook (honoured for world_size 1)
that enqueues, on the aggregation stream it is handed, a stand-in for NCCL's kernel -- eight CTAs of 640 threads and
64 KB of shared memory each (tools/microbench/standin.cu: the footprint of eight NCCL channels), busy for 100 us --
between two CUDA events.  The hook is called while the
next epoch's sampling kernel is already running on its lane (overlap = 1), so the time between the two events is the
time the reduction needs to get SM resources plus its own run time:
  * reserved_sms = -1 (none): the sampling grid holds every register of every SM; the stand-in starts when sampling
    CTAs retire, i.e. in the tail of the next epoch;
  * reserved_sms = 8: the main pass leaves eight SMs empty and the stand-in runs at once.
usage: python tools/overlap_timeline.py [workload key] [epoch_samples]"""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, subprocess
import torch
import paper_1910_11039_b200 as ebc
from paper_1910_11039_b200 import _capi
from paper_1910_11039_b200.distributed import _DeviceWords
from bench import workload_of, build_graph

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "microbench", "standin.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                os.path.join(HERE, "microbench", "standin.cu")], check=True)
standin = ctypes.CDLL(so)
standin.standin_launch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
key = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
epoch = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
w = workload_of(key)
g = build_graph(w, on_device=w["kind"] == "rmat")
for reserved in (-1, 8):
    marks = []
    def hook(user, buf, count, stream):
        s = torch.cuda.ExternalStream(stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            standin.standin_launch(stream, 8, 190000, sink.data_ptr())  # 100 us at 1.9 GHz
            b.record(s)
        marks.append((a, b))
        return 0
    fn = _capi.ALLREDUCE_FN(hook)
    cfg = ebc.RunConfig(eps=1e-4, delta=w["delta"], seed=7, omega_override=8 * epoch, epoch_samples=epoch,
                        allreduce=fn, reserved_sms=reserved, overlap=1)
    for rep in range(2):  # the second run is the measured one (allocations, first-touch)
        marks.clear()
        res, st = ebc.run_pipeline(g, cfg)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in marks]
    per_epoch = st["adaptive_s"] / st["epochs"] * 1e3
    print(f"{w['workload']}: reserved_sms {reserved:2d}: {st['epochs']} epochs of {epoch} samples, {per_epoch:.2f} ms per epoch, "
          f"adaptive {st['adaptive_s']*1e3:.1f} ms; stand-in all-reduce, enqueue -> done per epoch (ms): "
          + " ".join(f"{x:.2f}" for x in ms))
