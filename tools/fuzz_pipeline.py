"""Randomised full-pipeline parity on the GPU: ebc_run against the oracle replaying the same epoch schedule
(diameter bound, omega, calibration, per-epoch stop decisions under both bounds and allocators, counters, tau).
usage: python tools/fuzz_pipeline.py [cases] [seed]"""
import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1910_11039_b200 as ebc
from oracle import Oracle
from helpers import random_graph, grid_graph, largest_component

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time(); bad = 0
for c in range(cases):
    kind = rng.integers(0, 3)
    if kind == 0:
        n = int(rng.integers(200, 3000)); (off, tg), _ = largest_component(*random_graph(n, int(rng.integers(2 * n, 6 * n)), int(rng.integers(1 << 30))))
    elif kind == 1:
        (off, tg), _ = largest_component(*grid_graph(int(rng.integers(8, 40)), int(rng.integers(8, 40)), float(rng.uniform(0, 0.15)), int(rng.integers(1 << 30))))
    else:
        g0 = ebc.gen_rmat(int(rng.integers(8, 13)), int(rng.integers(4, 20)), seed=int(rng.integers(1 << 30))).largest_connected_component()
        off, tg = g0.offsets.copy(), g0.targets.copy()
    g = ebc.Graph.from_csr(off, tg); n = g.num_vertices
    if n < 3:
        continue
    o = Oracle(off, tg)
    bound = int(rng.integers(0, 2)); alloc = int(rng.integers(0, 2))
    eps = float(rng.choice([0.02, 0.03, 0.05, 0.08])); delta = float(rng.choice([0.05, 0.1, 0.2]))
    seed = int(rng.integers(1, 1 << 40)); calib_n = int(rng.choice([0, 100, 800])); ep = int(rng.choice([0, 256, 1024, 3000]))
    cfg = ebc.RunConfig(eps=eps, delta=delta, seed=seed, bound=bound, allocator=alloc, epoch_samples=ep, calib_samples=calib_n,
                        overlap=bool(rng.integers(0, 2)), block_threads=int(rng.choice([0, 32, 64, 128])), renumber=int(rng.choice([-1, 0, 1])))
    res, st = ebc.run_pipeline(g, cfg)
    vd = o.diameter(4, seed)[2]
    omega = Oracle.compute_omega(vd, eps, delta)
    calib = o.accumulate(seed, 0, calib_n, tag=1) if calib_n else np.zeros(n + 1, dtype=np.uint64)
    dl, du = Oracle.calibrate(calib, n, delta, alloc)
    epochs, S = o.run_epochs(seed, st["n0"], 10 ** 6, eps, omega, dl, du, bound)
    ok = (st["vertex_diameter_bound"] == vd and st["omega"] == omega and st["epochs"] == epochs and res.tau_total == int(S[0])
          and np.array_equal(res.counts, S[1:]) and st["tau"] == st["samples"] - st["calibration_samples"] - st["discarded_samples"])
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: kind {kind} n {n} {cfg} -> epochs {st['epochs']} vs {epochs}, tau {res.tau_total} vs {int(S[0])}, vd {st['vertex_diameter_bound']} vs {vd}", flush=True)
print(f"{cases} cases, {bad} mismatches, {time.time() - t0:.1f}s")
sys.exit(1 if bad else 0)
