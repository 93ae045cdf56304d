"""Randomised host-vs-device ingestion parity: from_edges (+ largest component) and R-MAT generation.
usage: python tools/fuzz_ingestion.py [cases] [seed]"""
import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_1910_11039_b200 as ebc
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
def same(a, b):
    return (a.num_vertices == b.num_vertices and np.array_equal(a.offsets, b.offsets) and np.array_equal(a.targets, b.targets)
            and np.array_equal(a.original_ids, b.original_ids))
bad = 0; t0 = time.time()
for c in range(cases):
    if rng.integers(0, 4) == 0:
        sc, ef, sd = int(rng.integers(2, 15)), int(rng.integers(1, 20)), int(rng.integers(1 << 40))
        h = ebc.gen_rmat(sc, ef, seed=sd)
        ok = same(ebc.gen_rmat_device(sc, ef, seed=sd), h) and same(ebc.gen_rmat_device(sc, ef, seed=sd, take_lcc=True), h.largest_connected_component())
        what = f"rmat {sc} {ef} {sd}"
    else:
        n = int(rng.integers(1, 5000)); m = int(rng.integers(0, 4 * n + 2))
        hi = n if rng.integers(0, 2) else max(1, n // int(rng.integers(1, 8)))   # sparse id ranges -> many components, isolated vertices
        src = rng.integers(0, hi, size=m, dtype=np.uint64); dst = rng.integers(0, hi, size=m, dtype=np.uint64)
        h = ebc.Graph.from_edges(n, src, dst)
        d = ebc.Graph.from_edges_device(n, src, dst)
        ok = same(d, h) and same(ebc.Graph.from_edges_device(n, src, dst, take_lcc=True), h.largest_connected_component()) \
            and same(h.largest_connected_component(device=-1), h.largest_connected_component())
        what = f"edges n {n} m {m} hi {hi}"
    if not ok:
        bad += 1; print("MISMATCH", c, what, flush=True)
print(f"{cases} cases, {bad} mismatches, {time.time() - t0:.1f}s")
sys.exit(1 if bad else 0)
