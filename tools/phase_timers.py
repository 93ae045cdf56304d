import sys; sys.path.insert(0,'.')
import numpy as np, paper_1910_11039_b200 as ebc
c=int(sys.argv[1]) if len(sys.argv)>1 else 2
g=(ebc.gen_rmat_device(24,16,seed=4).largest_connected_component(device=-1) if c==4 else ebc.gen_rmat_device(26,16,seed=5).largest_connected_component(device=-1) if c==5 else ebc.gen_rmat(20,16,seed=2) if c==2 else ebc.gen_grid(2000,2000,0.05,0.001,3) if c==3 else ebc.gen_erdos_renyi(10000,50000,1)).largest_connected_component()
s=ebc.Sampler(g, ebc.RunConfig()); N=200000 if c!=3 else 40000
s.sample(7,0,N//4); s.sync(); s.work(reset=True)
s.mark(0); s.sample(7,N,N); s.mark(1); ms=s.elapsed_ms(0,1); w=s.work()
names=["init","expand","probe","degsum","meet rest","walk","finish","meet large","meet small","meet pick"]
vals=[w[k] for k in ebc.WORK_NAMES[:10]]; tot=sum(vals)
print(f"config {c}: {N/ms*1e3:.0f} samples/s; thread-0 cycles per phase:")
for n_,v in zip(names,vals): print(f"  {n_:8s} {100*v/tot:5.1f}%  {v/N:10.0f} cycles/sample")
nl=w[ebc.WORK_NAMES[10]]
print(f"  large meet sets: {nl/N:.3f} of the samples, {vals[7]/max(nl,1):.0f} cycles each; small ones {(vals[8]+vals[9])/max(N-nl,1):.0f} cycles each")
