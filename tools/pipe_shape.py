"""End-to-end time of config 2 (ebc_graph_from_csr + ebc_run with host buffers) against the pipeline's launch shape and
epoch size.  usage: python tools/pipe_shape.py
One B200, round 2: default (two warps, 3 epochs of 35 840) 24.6 ms, one warp 27.1 ms, two warps with 2 epochs of
53 248 23.4 ms, one warp with 1 epoch of 107 520 24.9 ms (adaptive phase 10.4-12.5 ms of it: 23 samples per slot do
not amortise the ramp and the tail of a launch; the rest is CSR copy 3, upload 4.4, diameter 2.4, calibration 1.2 ms)."""
import sys, time; sys.path.insert(0, '.')
import numpy as np, paper_1910_11039_b200 as ebc
g = ebc.gen_rmat_device(20, 16, seed=2).largest_connected_component(device=-1)
off, tg = g.offsets, g.targets
for kw in (dict(), dict(block_threads=32), dict(block_threads=64, epoch_samples=53248), dict(block_threads=32, epoch_samples=53248), dict(block_threads=32, epoch_samples=107520)):
    ts = []
    for i in range(6):
        t0 = time.time()
        g2 = ebc.Graph.from_csr(off, tg, validate=False)
        res, st = ebc.run_pipeline(g2, ebc.RunConfig(eps=0.005, delta=0.1, seed=7, work_counters=False, **kw))
        _ = float(res.scores[0]); ts.append(time.time() - t0)
    print(kw, "median %.4f s" % sorted(ts[1:])[2], "adaptive %.4f" % st["adaptive_s"], "epochs", st["epochs"], "tau", st["tau"], "samples", st["samples"])
