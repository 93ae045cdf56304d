"""Slot capacity (settled vertices per side per slot) on the large hub configs: sustained samples/s, slots that fit,
samples abandoned and re-run in a full-capacity slot.  usage: python tools/cap_sweep_c5.py 5 [4]"""
import sys; sys.path.insert(0, '.')
import paper_1910_11039_b200 as ebc
for c in [int(x) for x in sys.argv[1:]] or [5]:
    scale, seed = {2: (20, 2), 4: (24, 4), 5: (26, 5)}[c]
    g = ebc.gen_rmat_device(scale, 16, seed=seed).largest_connected_component(device=-1)
    n = g.num_vertices; N = 200000
    for div in (4, 6, 8, 12, 16):
        s = ebc.Sampler(g, ebc.RunConfig(slot_capacity=n // div)); inf = s.info()
        s.sample(7, 0, N // 4); s.sync(); s.work(reset=True)
        s.mark(0); s.sample(7, N, N); s.mark(1); ms = s.elapsed_ms(0, 1)
        rec = None
        print(f"config {c} cap n/{div}={n//div}: slots {inf['slots']} dev GB {inf['device_bytes']/1e9:.1f}: {N/ms*1e3:.0f} samples/s", flush=True)
        s.close()
