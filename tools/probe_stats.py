"""How the final-level probe fares per sample: probed (flags & 2), contact-edge buffer overflow (flags & 4).
usage: python tools/probe_stats.py 2|4 [samples] [block threads]"""
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1910_11039_b200 as ebc
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
scale, seed = {2: (20, 2), 4: (24, 4), 5: (26, 5), 22: (22, 2)}[c]
g = ebc.gen_rmat_device(scale, 16, seed=seed).largest_connected_component(device=-1)
s = ebc.Sampler(g, ebc.RunConfig(block_threads=int(sys.argv[3]) if len(sys.argv) > 3 else 0))
rec, _ = s.sample_debug(7, 0, N, path_stride=1)
f = rec["flags"]
print(f"config {c}: {N} samples: probed {np.mean((f & 2) != 0):.3f}, probe overflowed {np.mean((f & 4) != 0):.3f}, "
      f"overflowed and then probed a later level {np.mean(((f & 4) != 0) & ((f & 2) != 0)):.3f}, re-run in a large slot {np.mean((f & 1) != 0):.4f}, "
      f"meet set resolved in global memory (more contact edges than the shared-memory path holds) {np.mean((f & 8) != 0):.3f} at {s.info()['block_threads']} threads")
mc = rec["meet_count"]
print("meet set size: mean %.1f, p50 %d, p90 %d, p99 %d, max %d" % (mc.mean(), *np.percentile(mc, [50, 90, 99]), mc.max()))
print("meet set size of overflowed samples: mean %.1f" % mc[(f & 4) != 0].mean() if ((f & 4) != 0).any() else "no overflow")
