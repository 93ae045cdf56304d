# What would hub-clustered vertex ids buy?  Runs config 2 as generated and with the vertices renumbered
# by descending degree (a DIFFERENT labelled graph: indicative timing only, not a parity case).
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
SCALE=int(next((a for a in sys.argv[1:] if a.isdigit()),"20"))
g=ebc.gen_rmat(SCALE,16,seed=2).largest_connected_component()
off=g.offsets; tgt=g.targets; n=len(off)-1
deg=np.diff(off).astype(np.int64)
def run(graph,name,N=400000 if SCALE<=20 else 40000):
    if "--dry" in sys.argv: print(name, len(graph.offsets)-1, len(graph.targets)); return
    s=ebc.Sampler(graph, ebc.RunConfig()); inf=s.info()
    s.sample(7,0,N//10); s.sync(); s.work(reset=True)
    s.mark(0); s.sample(7,N//10,N); s.mark(1); ms=s.elapsed_ms(0,1)
    w=s.work()
    print(f"{name}: {ms:.1f} ms, {N/ms*1e3:.0f} samples/s, E_bfs/sample {w['E_bfs']/w['samples']:.0f}, V_set/sample {w['V_set']/w['samples']:.0f}", flush=True)
    s.close()
run(g,"as generated")
for mode in ("degree-desc","class-desc","random"):
    if mode=="degree-desc":
        order=np.argsort(-deg,kind='stable')
    elif mode=="class-desc":
        order=np.argsort(-np.floor(np.log2(np.maximum(deg,1))).astype(np.int64)-(deg>0),kind='stable')
    else:
        order=np.random.default_rng(1).permutation(n)
    perm=np.empty(n,dtype=np.int64); perm[order]=np.arange(n)
    src=np.repeat(np.arange(n,dtype=np.int64),deg)
    keep=src<tgt
    g2=ebc.Graph.from_edges(n, perm[src[keep]].astype(np.uint64), perm[tgt[keep].astype(np.int64)].astype(np.uint64))
    run(g2,mode)
