# short single-GPU driver for ncu: a few epochs of config-2 sampling + fold
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat(20,16,seed=2).largest_connected_component()
s=ebc.Sampler(g, ebc.RunConfig())
n=g.num_vertices
dl,du=ebc.calibrate(np.zeros(n+1,dtype=np.uint64),n,0.1); s.set_stopping(0.005,1<<62,dl,du)
B=int(sys.argv[1]) if len(sys.argv)>1 else 16384
for k in range(3):
    s.sample(7,k*B,B,frame=k&1); s.fold_and_check(k&1)
s.sync(); print("ok", s.work())
