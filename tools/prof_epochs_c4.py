# short single-GPU driver for ncu: config-4 (R-MAT-24) sampling with the default launch shape
import sys; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat_device(24,16,seed=4).largest_connected_component(device=-1)
s=ebc.Sampler(g, ebc.RunConfig()); print(s.info())
B=int(sys.argv[1]) if len(sys.argv)>1 else 8192
for k in range(3):
    s.sample(7,k*B,B,frame=k&1)
s.sync(); print("ok", s.work())
