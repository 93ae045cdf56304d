# host vs device graph ingestion: python tools/ingest_timing.py 20 [24]
import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_1910_11039_b200 as ebc
for scale in [int(x) for x in sys.argv[1:]] or [20]:
    t=time.time(); g=ebc.gen_rmat_device(scale,16,seed=2,take_lcc=True); t_first=time.time()-t
    t=time.time(); g=ebc.gen_rmat_device(scale,16,seed=2,take_lcc=True); t_dev=time.time()-t
    print(f"scale {scale}: device gen+canonicalise+lcc {t_dev:.3f}s (first call {t_first:.3f}s)  n={g.num_vertices} m={g.num_edges}", flush=True)
    if scale<=24:
        t=time.time(); h=ebc.gen_rmat(scale,16,seed=2); t1=time.time()-t
        t=time.time(); h=h.largest_connected_component(); t2=time.time()-t
        same = np.array_equal(g.offsets,h.offsets) and np.array_equal(g.targets,h.targets) and np.array_equal(g.original_ids,h.original_ids)
        print(f"          host   gen+canonicalise {t1:.3f}s + lcc {t2:.3f}s   identical={same}", flush=True)
