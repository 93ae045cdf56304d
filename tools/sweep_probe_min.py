"""Sustained samples/s against the probe threshold (EBC_PROBE_MIN_SLOTS: levels with fewer adjacency slots are
expanded without trying the read-only final-level probe).  usage: python tools/sweep_probe_min.py [graphs] [values]
One process per point (the threshold is read when a sampler is created)."""
import os, subprocess, sys
graphs = (sys.argv[1] if len(sys.argv) > 1 else "c1,rmat14,rmat17,c2,er1m,c3,c4").split(",")
values = (sys.argv[2] if len(sys.argv) > 2 else "64,128,256,512,1024,2048").split(",")
CHILD = r'''
import sys; sys.path.insert(0, '.')
import paper_1910_11039_b200 as ebc
name = sys.argv[1]
if name == "c1": g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component(); N = 400000
elif name == "rmat14": g = ebc.gen_rmat(14, 16, seed=2).largest_connected_component(); N = 400000
elif name == "rmat17": g = ebc.gen_rmat(17, 16, seed=2).largest_connected_component(); N = 400000
elif name == "c2": g = ebc.gen_rmat_device(20, 16, seed=2).largest_connected_component(device=-1); N = 400000
elif name == "er1m": g = ebc.gen_erdos_renyi(1000000, 8000000, 1).largest_connected_component(); N = 200000
elif name == "c3": g = ebc.gen_grid(2000, 2000, 0.05, 0.001, 3).largest_connected_component(); N = 40000
elif name == "c4": g = ebc.gen_rmat_device(24, 16, seed=4).largest_connected_component(device=-1); N = 200000
s = ebc.Sampler(g, ebc.RunConfig())
s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1)
print(f"{N / ms * 1e3:.0f}")
'''
for gname in graphs:
    row = []
    for v in values:
        env = dict(os.environ, EBC_PROBE_MIN_SLOTS=v)
        out = subprocess.run([sys.executable, "-c", CHILD, gname], env=env, capture_output=True, text=True)
        row.append(f"{v}: {out.stdout.strip() or out.stderr.strip()[-200:]}")
    print(f"{gname:8s} " + "   ".join(row), flush=True)
