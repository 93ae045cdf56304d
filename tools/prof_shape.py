"""ncu driver: one warm-up launch, then one launch of N samples with an explicit launch shape.
usage: python tools/prof_shape.py <workload key> <samples> <block> <items> [renumber]"""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11039_b200 as ebc
from bench import workload_of, build_graph
key, N, block, items = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ren = int(sys.argv[5]) if len(sys.argv) > 5 else 0
w = workload_of(key)
g = build_graph(w, on_device=w["kind"] == "rmat" and w["scale"] >= 22)
s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, renumber=ren))
s.sample(7, 0, max(N // 4, 1), frame=0); s.sync()
s.mark(0); s.sample(7, 1 << 22, N, frame=1); s.mark(1)
print(f"{key}: {N} samples in {s.elapsed_ms(0, 1):.2f} ms; info {s.info()}")
