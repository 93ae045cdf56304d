# slot capacity vs slots in flight on a memory-limited input: python tools/cap_sweep_big.py 26 5 "4,8,16,32"
import sys, time; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
scale=int(sys.argv[1]); seed=int(sys.argv[2]); divs=[int(x) for x in sys.argv[3].split(',')]
t=time.time(); g=ebc.gen_rmat_device(scale,16,seed=seed,take_lcc=True); n=g.num_vertices
print(f"scale {scale}: n={n} m={g.num_edges} built in {time.time()-t:.1f}s", flush=True)
N=60000
for d in divs:
    s=ebc.Sampler(g, ebc.RunConfig(slot_capacity=max(n//d, 1<<17))); inf=s.info()
    s.sample(7,0,N//4); s.sync(); s.work(reset=True)
    s.mark(0); s.sample(7,N,N); s.mark(1); ms=s.elapsed_ms(0,1); w=s.work()
    print(f"cap n/{d}: slots {inf['slots']} dev GB {inf['device_bytes']/1e9:.1f}: {N/ms*1e3:.0f} samples/s, samples run {w['samples']} (re-runs {w['samples']-N})", flush=True)
    s.close(); ebc._capi.load().ebc_release_device_cache()
