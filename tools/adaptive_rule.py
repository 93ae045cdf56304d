# Hoeffding/uniform vs empirical Bernstein/weighted on config 2: where does the run stop, how long does it take
import sys, time; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat_device(20,16,seed=2,take_lcc=True)
for name,kw in (("hoeffding/uniform",{}),("bernstein/uniform",dict(bound=ebc.EMPIRICAL_BERNSTEIN)),("bernstein/weighted",dict(bound=ebc.EMPIRICAL_BERNSTEIN,allocator=ebc.WEIGHTED)),("hoeffding/weighted",dict(allocator=ebc.WEIGHTED))):
    for rep in range(2):
        t=time.time(); res,st=ebc.run_pipeline(g, ebc.RunConfig(eps=0.005,delta=0.1,seed=7,**kw)); dt=time.time()-t
    print(f"{name:20s}: tau={st['tau']} of omega={st['omega']} epochs={st['epochs']} discarded={st['discarded_samples']} calib_s={st['calibration_s']:.3f} adaptive_s={st['adaptive_s']:.3f} check_s={st['check_s']:.3f} total {dt:.3f}s", flush=True)
