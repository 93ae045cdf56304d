"""Default-shape sustained rate on config 4 / 5 (A/B of library builds): python tools/sweep_big2.py 4 5"""
import sys, time; sys.path.insert(0, '.')
import paper_1910_11039_b200 as ebc
for c in [int(x) for x in sys.argv[1:]] or [4]:
    scale, seed = {4: (24, 4), 5: (26, 5)}[c]
    g = ebc.gen_rmat_device(scale, 16, seed=seed).largest_connected_component(device=-1)
    N = {4: 200000, 5: 100000}[c]
    for rep in range(2):
        s = ebc.Sampler(g, ebc.RunConfig()); inf = s.info()
        s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
        s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1); w = s.work()
        print(f"config {c} block {inf['block_threads']} items {inf['items_per_thread']} slots {inf['slots']}: {N/ms*1e3:.0f} samples/s, BFS GTEPS {w['E_bfs']/ms/1e6:.2f}", flush=True)
        s.close()
