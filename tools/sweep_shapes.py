"""Sustained samples/s per launch shape on one graph class.
usage: python tools/sweep_shapes.py GRAPH "block,items[,renumber[,slot_capacity]];..."   (GRAPH: c1 rmat14 rmat17 c2 rmat22 er1m c3 c4 c5)"""
import sys, time; sys.path.insert(0, '.')
import paper_1910_11039_b200 as ebc
name = sys.argv[1]
shapes = [tuple(int(x) for x in s.split(',')) for s in sys.argv[2].split(';')]
N = 400000
if name == "c1": g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component()
elif name == "rmat14": g = ebc.gen_rmat(14, 16, seed=2).largest_connected_component()
elif name == "rmat17": g = ebc.gen_rmat(17, 16, seed=2).largest_connected_component()
elif name == "c2": g = ebc.gen_rmat_device(20, 16, seed=2).largest_connected_component(device=-1)
elif name == "rmat22": g = ebc.gen_rmat_device(22, 16, seed=2).largest_connected_component(device=-1)
elif name == "er1m": g = ebc.gen_erdos_renyi(1000000, 8000000, 1).largest_connected_component(); N = 200000
elif name == "c3": g = ebc.gen_grid(2000, 2000, 0.05, 0.001, 3).largest_connected_component(); N = 40000
elif name == "c4": g = ebc.gen_rmat_device(24, 16, seed=4).largest_connected_component(device=-1)
elif name == "c5": g = ebc.gen_rmat_device(26, 16, seed=5).largest_connected_component(device=-1); N = 200000
print(f"{name}: n={g.num_vertices} m={g.num_edges}", flush=True)
for shape in shapes:
    block, items = shape[:2]
    ren = shape[2] if len(shape) > 2 else 0
    capv = shape[3] if len(shape) > 3 else 0
    try:
        t = time.time()
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, renumber=ren, slot_capacity=capv)); inf = s.info()
        setup = time.time() - t
        s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
        s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1)
        print(f"  {block}x{items} renumber {ren}->{inf['renumbered']} cap {inf['slot_capacity']} slots {inf['slots']} dev GB {inf['device_bytes']/1e9:.1f} setup {setup*1e3:.0f} ms: {N/ms*1e3:.0f} samples/s", flush=True)
        s.close()
    except Exception as e:
        print(f"  {block}x{items}: {e}", flush=True)
