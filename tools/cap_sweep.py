import sys, time; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
c=int(sys.argv[1]); N=int(sys.argv[2])
g=(ebc.gen_rmat(20,16,seed=2) if c==2 else ebc.gen_rmat(24,16,seed=4)).largest_connected_component()
n=g.num_vertices
for div in (4, 6, 8, 12):
    s=ebc.Sampler(g, ebc.RunConfig(slot_capacity=n//div)); inf=s.info()
    rec,_=s.sample_debug(7,0,min(N,1<<20))
    import numpy as np
    s.mark(0); s.sample(7,N,N); s.mark(1); ms=s.elapsed_ms(0,1)
    print(f"config {c} cap n/{div}={n//div}: slots {inf['slots']} dev GB {inf['device_bytes']/1e9:.1f}: {N/ms*1e3:.0f} samples/s", flush=True)
    s.close()
