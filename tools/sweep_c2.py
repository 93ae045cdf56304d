# throughput sweep on config 2 over launch shapes: python tools/sweep_c2.py "128,4,0;64,4,0"
import sys; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat(20,16,seed=2).largest_connected_component()
shapes=[tuple(int(x) for x in s.split(',')) for s in (sys.argv[1] if len(sys.argv)>1 else "128,4,0").split(';')]
N=int(sys.argv[2]) if len(sys.argv)>2 else 200000
for block,items,slots in shapes:
    s=ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, slots=slots)); inf=s.info()
    s.sample(7,0,20000); s.sync(); s.work(reset=True)
    s.mark(0); s.sample(7,20000,N); s.mark(1); ms=s.elapsed_ms(0,1)
    w=s.work(); B=ebc.algorithmic_bytes(w)
    print(f"block {block} items {items} slots {inf['slots']}: {ms:.1f} ms, {N/ms*1e3:.0f} samples/s, GTEPS {w['E_bfs']/ms/1e6:.2f}, alg GB/s {B/ms/1e6:.1f}", flush=True)
    s.close()
