"""Single-GPU driver for ncu: warm-up launches, then ONE sampling launch of N samples of a bench workload.
usage: python tools/prof_launch.py <workload key> <samples> [warm-up samples]
Profile the last sample_kernel launch (ncu -k regex:sample_kernel --launch-skip <warm-up launches>)."""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11039_b200 as ebc
from bench import workload_of, build_graph
key = sys.argv[1]; N = int(sys.argv[2]); W = int(sys.argv[3]) if len(sys.argv) > 3 else max(N // 4, 1)
w = workload_of(key)
g = build_graph(w, on_device=w["kind"] == "rmat" and w["scale"] >= 22)
s = ebc.Sampler(g, ebc.RunConfig(work_counters=os.environ.get("EBC_PROF_STATS", "0") != "0"))  # the kernels bench.py times
s.sample(7, 0, W, frame=0); s.sync()
s.mark(0); s.sample(7, 1 << 22, N, frame=1); s.mark(1)
ms = s.elapsed_ms(0, 1)
print(f"{key}: {N} samples in {ms:.2f} ms = {N / ms * 1e3:.0f} samples/s; info {s.info()}")
