"""Launch-shape sweep on the large configs (4: R-MAT-24, 5: R-MAT-26) where device memory, not the SM
count, limits the number of slots: sustained samples/s for block_threads in 128 / 256 / 512.
usage: python tools/sweep_big.py 5 [4]"""
import sys, time; sys.path.insert(0, '.')
import paper_1910_11039_b200 as ebc

for c in [int(x) for x in sys.argv[1:]] or [5]:
    scale, seed = {4: (24, 4), 5: (26, 5), 2: (20, 2)}[c]
    t = time.time()
    g = ebc.gen_rmat_device(scale, 16, seed=seed).largest_connected_component(device=-1)
    print(f"config {c}: n={g.num_vertices} m={g.num_edges} built in {time.time()-t:.1f}s", flush=True)
    N = {2: 400000, 4: 200000, 5: 100000}[c]
    for block, items in ((128, 4), (256, 4), (512, 4), (512, 2), (256, 2)):
        try:
            t = time.time()
            s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items)); inf = s.info()
            t_setup = time.time() - t
            s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
            s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1); w = s.work()
            print(f"  block {block} items {items} slots {inf['slots']} dev GB {inf['device_bytes']/1e9:.1f} setup {t_setup:.1f}s: "
                  f"{N/ms*1e3:.0f} samples/s, BFS GTEPS {w['E_bfs']/ms/1e6:.2f}", flush=True)
            s.close()
        except Exception as e:
            print(f"  block {block} items {items}: {e}", flush=True)
