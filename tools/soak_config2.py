# config 2 at full size: N samples on the GPU vs the CPU oracle, frames compared word for word
import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
from oracle import Oracle
N=int(sys.argv[1]) if len(sys.argv)>1 else 500000
g=ebc.gen_rmat_device(20,16,seed=2,take_lcc=True)
s=ebc.Sampler(g, ebc.RunConfig())
t=time.time(); s.sample(7,0,N); got=s.read_frame(0); tg=time.time()-t
o=Oracle(g.offsets,g.targets)
t=time.time(); want=o.accumulate(7,0,N); tc=time.time()-t
print(f"config 2, {N} samples: GPU {tg:.2f}s, oracle {tc:.1f}s, frames identical: {np.array_equal(got,want)}; tau {int(got[0])}, counted vertices {int(got[1:].sum())}")
