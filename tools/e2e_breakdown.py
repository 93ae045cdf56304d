import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat(20,16,seed=2).largest_connected_component()
off,tg=g.offsets,g.targets
cfg=ebc.RunConfig(eps=0.005,delta=0.1,seed=7)
for i in range(int(sys.argv[1]) if len(sys.argv)>1 else 4):
    t0=time.time(); g2=ebc.Graph.from_csr(off,tg,validate=False); t1=time.time()
    res,st=ebc.run_pipeline(g2,cfg); t2=time.time()
    del g2; t3=time.time()
    print(f"run {i}: from_csr {t1-t0:.3f}  run_pipeline(py) {t2-t1:.3f}  [C wall_s {st['wall_s']:.3f}: upload {st['upload_s']:.3f} diam {st['diameter_s']:.3f} calib {st['calibration_s']:.3f} adapt {st['adaptive_s']:.3f}]  del {t3-t2:.3f}", flush=True)
