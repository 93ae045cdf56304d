"""Runs BASELINE.json configs through ebc_run on one GPU and prints time-to-stop / throughput.
usage: python tools/run_configs.py 1 2 3 [4]"""
import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_1910_11039_b200 as ebc

def build(c):
    t = time.time()
    if c == 1: g = ebc.gen_erdos_renyi(10000, 50000, 1); eps = 0.01
    elif c == 2: g = ebc.gen_rmat_device(20, 16, seed=2); eps = 0.005
    elif c == 3: g = ebc.gen_grid(2000, 2000, 0.05, 0.001, 3); eps = 0.01
    elif c == 4: g = ebc.gen_rmat_device(24, 16, seed=4); eps = 0.001
    elif c == 5: g = ebc.gen_rmat_device(26, 16, seed=5); eps = 0.001
    t1 = time.time() - t
    g = g.largest_connected_component(device=-1 if c in (2, 4, 5) else None)  # same graphs as the host path, in seconds
    print(f"config {c}: n={g.num_vertices} m={g.num_edges} gen {t1:.1f}s lcc {time.time()-t-t1:.1f}s", flush=True)
    return g, eps

for c in [int(x) for x in sys.argv[1:]] or [1, 2, 3]:
    g, eps = build(c)
    for rep in range(2):
        t = time.time()
        res, st = ebc.run_pipeline(g, ebc.RunConfig(eps=eps, delta=0.1, seed=7))
        dt = time.time() - t
        w = st["work"]
        print(f"  run {rep}: {dt:.3f}s  tau={st['tau']} omega={st['omega']} vd={st['vertex_diameter_bound']} epochs={st['epochs']} n0={st['n0']} "
              f"upload {st['upload_s']:.3f} diam {st['diameter_s']:.3f} calib {st['calibration_s']:.3f} adaptive {st['adaptive_s']:.3f} "
              f"-> {st['tau']/st['adaptive_s']:.0f} samples/s adaptive; per sample: E_bfs {w['E_bfs']/w['samples']:.0f} levels {w['levels']/w['samples']:.1f} "
              f"E_walk {w['E_walk']/w['samples']:.0f} L {w['L']/w['samples']:.1f} overflow {st['overflow_samples']}", flush=True)
    # sustained throughput on a fixed budget
    s = ebc.Sampler(g, ebc.RunConfig()); inf = s.info()
    N = 200000 if c != 3 else 60000
    s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
    s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1); w = s.work()
    print(f"  sustained: {N/ms*1e3:.0f} samples/s, BFS GTEPS {w['E_bfs']/ms/1e6:.2f}, slots {inf['slots']} block {inf['block_threads']} items {inf['items_per_thread']} dev GB {inf['device_bytes']/1e9:.1f}", flush=True)
    s.close()
