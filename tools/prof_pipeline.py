# short single-GPU driver for ncu: one full config-2 pipeline run (diameter BFS, calibration, epochs, fold + check)
import sys; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
g=ebc.gen_rmat(20,16,seed=2).largest_connected_component()
res,st=ebc.run_pipeline(g, ebc.RunConfig(eps=0.005,delta=0.1,seed=7))
print("ok", st["tau"], st["epochs"], st["diameter_upper_bound"])
