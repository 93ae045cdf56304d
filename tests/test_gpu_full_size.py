"""BASELINE.json configs at their FULL sizes: the oracle cannot replay them in seconds, so parity is
checked through size-independent properties plus oracle spot checks on randomly chosen sample indices.

 * conservation: tau == number of samples; sum of all counters == sum of the sampled paths' lengths
   == sum over samples of (d(s,t) - 1) for reachable pairs  (SPEC.md sampler invariants);
 * launch-shape independence: different (block, items, slots) give identical frames;
 * oracle spot check: (s, t, d, meet vertex, draws, path) of random indices equal the CPU oracle's.
"""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from oracle import Oracle

pytestmark = pytest.mark.gpu
SEED = 7


def _check(g, samples, spot, stride, shapes):
    n = g.num_vertices
    frames = []
    for block, items, slots in shapes:
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, slots=slots))
        rec, paths = s.sample_debug(SEED, 0, samples, path_stride=stride)
        f = s.read_frame(0)
        frames.append(f)
        assert int(f[0]) == samples
        reach = rec["dist"] != 0xFFFFFFFF
        assert int(f[1:].sum()) == int(rec["path_len"].sum())
        assert np.array_equal(rec["path_len"][reach], rec["dist"][reach] - 1) and not rec["path_len"][~reach].any()
        assert (rec["s"] != rec["t"]).all() and rec["s"].max() < n and rec["t"].max() < n
        assert int(f[1:].max()) <= samples
        s.close()
    for f in frames[1:]:
        assert np.array_equal(frames[0], f)
    o = Oracle(g.offsets, g.targets)
    rng = np.random.default_rng(1)
    for i in rng.choice(samples, spot, replace=False):
        w = o.sample(SEED, int(i))
        r = rec[int(i)]
        assert (int(r["s"]), int(r["t"]), int(r["dist"]), int(r["meet"]), int(r["draws"])) == \
               (w["s"], w["t"], w["dist"], w["meet"], w["draws"]), i
        k = min(stride, len(w["path"]))
        assert np.array_equal(paths[int(i), :k], w["path"][:k])
    return frames[0]


def test_config2_rmat20_full_size():
    g = ebc.gen_rmat(20, 16, seed=2).largest_connected_component()
    assert (g.num_vertices, g.num_edges) == (645739, 15700555)
    _check(g, 107520, 150, 8, [(128, 4, 0), (64, 2, 256), (256, 4, 0)])


def test_config2_pipeline_full_size():
    """The whole config-2 run: vertex-diameter bound and omega as the CPU oracle computes them, the stop
    at the first epoch with tau >= omega, counters equal to the frame of the same sample indices."""
    g = ebc.gen_rmat(20, 16, seed=2).largest_connected_component()
    res, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.005, delta=0.1, seed=SEED))
    o = Oracle(g.offsets, g.targets)
    assert st["vertex_diameter_bound"] == o.diameter(4, SEED)[2]
    assert st["omega"] == Oracle.compute_omega(st["vertex_diameter_bound"], 0.005, 0.1) == 106052
    assert st["tau"] == st["epochs"] * st["n0"] >= st["omega"] > (st["epochs"] - 1) * st["n0"]
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=64, items_per_thread=4))
    s.sample(SEED, 0, st["tau"])
    assert np.array_equal(s.read_frame(0)[1:], res.counts)
    assert np.array_equal(res.scores, res.counts.astype(np.float64) / float(st["tau"]))


def test_config3_grid_full_size():
    g = ebc.gen_grid(2000, 2000, 0.05, 0.001, 3).largest_connected_component()
    assert g.num_vertices > 3_990_000
    f = _check(g, 6144, 25, 160, [(128, 4, 0), (256, 2, 64)])
    assert int(f[1:].sum()) > 6144 * 40  # paths are long on the grid (mean ~85 internal vertices)


def test_config1_er_full_run_twice_identical():
    g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component()
    a, sa = ebc.run_pipeline(g, ebc.RunConfig(eps=0.01, delta=0.1, seed=SEED))
    b, sb = ebc.run_pipeline(g, ebc.RunConfig(eps=0.01, delta=0.1, seed=SEED, block_threads=32, items_per_thread=2, slots=37))
    assert np.array_equal(a.counts, b.counts) and sa["tau"] == sb["tau"] == 32768 and sa["epochs"] == sb["epochs"]
