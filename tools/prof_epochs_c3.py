# short single-GPU driver for ncu: config-3 (grid) sampling
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
g=ebc.gen_grid(2000,2000,0.05,0.001,3).largest_connected_component()
s=ebc.Sampler(g, ebc.RunConfig())
B=int(sys.argv[1]) if len(sys.argv)>1 else 4096
for k in range(3):
    s.sample(7,k*B,B,frame=k&1)
s.sync(); print("ok", s.work())
