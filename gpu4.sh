timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -15
python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat(20,16,seed=2).largest_connected_component()
for block,items,slots in ((128,4,0),(128,2,0),(128,1,0),(64,4,0),(256,4,0),(256,2,0),(512,2,0)):
    s=ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, slots=slots)); inf=s.info()
    s.sample(7,0,20000); s.sync(); s.work(reset=True)
    s.mark(0); s.sample(7,20000,200000); s.mark(1); ms=s.elapsed_ms(0,1)
    w=s.work(); B=ebc.algorithmic_bytes(w)
    print(f"block {block} items {items} slots {inf['slots']}: {ms:.1f} ms, {200000/ms*1e3:.0f} samples/s, GTEPS {w['E_bfs']/ms/1e6:.2f}, alg GB/s {B/ms/1e6:.1f}", flush=True)
    s.close()
PY
