"""Randomised parity sweep on the GPU: random graphs x launch shapes x numbering x slot capacities, frames and
records against the CPU oracle.  usage: python tools/fuzz_parity.py [cases] [seed]"""
import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_1910_11039_b200 as ebc
from oracle import Oracle
from helpers import random_graph, grid_graph, complete_bipartite_chain, star_graph

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time(); bad = 0
for c in range(cases):
    kind = rng.integers(0, 8)
    if kind == 0:
        n = int(rng.integers(5, 400)); csr = random_graph(n, int(rng.integers(n // 2, 6 * n)), int(rng.integers(1 << 30)))
    elif kind == 1:
        csr = grid_graph(int(rng.integers(3, 30)), int(rng.integers(3, 30)), float(rng.uniform(0, 0.3)), int(rng.integers(1 << 30)))
    elif kind == 2:
        layers = [int(rng.integers(1, 5))] + [int(rng.integers(2, 80)) for _ in range(int(rng.integers(2, 14)))] + [int(rng.integers(1, 4))]
        csr = complete_bipartite_chain(layers)
    elif kind == 3:
        g0 = ebc.gen_rmat(int(rng.integers(6, 13)), int(rng.integers(2, 20)), seed=int(rng.integers(1 << 30))).largest_connected_component()
        csr = (g0.offsets.copy(), g0.targets.copy())
    elif kind == 4:
        csr = star_graph(int(rng.integers(3, 3000)))
    elif kind == 6:  # low maximum degree: the fixed-stride-row path (expand_level_ell)
        n = int(rng.integers(20, 3000)); csr = random_graph(n, int(rng.integers(n // 2, 3 * n // 2)), int(rng.integers(1 << 30)))
    elif kind == 7:
        csr = grid_graph(int(rng.integers(20, 90)), int(rng.integers(20, 90)), float(rng.uniform(0, 0.15)), int(rng.integers(1 << 30)))
    else:
        n = int(rng.integers(1200, 4000)); csr = random_graph(n, int(rng.integers(2 * n, 12 * n)), int(rng.integers(1 << 30)))
    off, tg = csr
    if len(off) - 1 < 2:
        continue
    g = ebc.Graph.from_csr(off, tg)
    n = g.num_vertices
    block = int(rng.choice([32, 64, 128, 256, 512])); items = int(rng.choice([1, 2, 4]))
    cfg = ebc.RunConfig(block_threads=block, items_per_thread=items, slots=int(rng.choice([1, 3, 16, 0])),
                        renumber=int(rng.choice([-1, 0, 1, 2])), materialize_final_level=bool(rng.integers(0, 2)),
                        slot_capacity=int(rng.choice([0, 0, max(2, n // 7), 8])))
    seed = int(rng.integers(1 << 40)); first = int(rng.integers(1 << 20)); count = int(rng.integers(50, 1500))
    o = Oracle(off, tg)
    s = ebc.Sampler(g, cfg)
    rec, paths = s.sample_debug(seed, first, count, path_stride=48)
    want = o.accumulate(seed, first, count)
    ok = np.array_equal(s.read_frame(0), want)
    for i in range(0, count, max(1, count // 25)):
        w = o.sample(seed, first + i)
        r = rec[i]
        ok = ok and (int(r["s"]), int(r["t"]), int(r["dist"]), int(r["meet"]), int(r["draws"]), int(r["path_len"])) == \
            (w["s"], w["t"], w["dist"], w["meet"], w["draws"], len(w["path"]))
        if len(w["path"]) <= 48:
            ok = ok and np.array_equal(paths[i, :len(w["path"])], w["path"])
    s.close()
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: kind {kind} n {n} block {block} items {items} cfg {cfg} seed {seed} first {first} count {count}", flush=True)
print(f"{cases} cases, {bad} mismatches, {time.time() - t0:.1f}s")
sys.exit(1 if bad else 0)
