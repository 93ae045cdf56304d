"""BASELINE.json configs at their FULL sizes.  The oracle cannot replay whole runs of the large configs in
seconds, so parity is checked through

 * conservation: tau == number of samples; sum of all counters == sum of the sampled paths' lengths
   == sum over samples of (d(s,t) - 1) for reachable pairs  (SPEC.md sampler invariants);
 * launch-shape independence: different (block, items, slots) give identical frames;
 * oracle spot checks: (s, t, d, meet vertex, meet-set size, draws, full path) of >= 200-300 randomly chosen
   sample indices equal the CPU oracle's (reference: sampler.cpp:54-164);
 * word-for-word frames: the epoch frame of a contiguous block of sample indices equals the oracle's
   (config 2: the whole run of 107 520 samples; configs 3-5: a 2 000 / 1 000-sample block);
 * the full config-2 pipeline against an oracle replay of the same epochs (counters, tau, stop epoch).
Configs 4 and 5 run with their DEFAULT launch shape (256x4) and slot counts.
"""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from helpers import oracle_frame
from oracle import Oracle

pytestmark = pytest.mark.gpu
SEED = 7


def _check(g, samples, spot, stride, shapes, block_first=None, block_count=0, expect_default=None):
    n = g.num_vertices
    frames = []
    rec = paths = None
    for k, (block, items, slots) in enumerate(shapes):
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, slots=slots))
        if k == 0 and expect_default is not None:
            inf = s.info()
            assert (inf["block_threads"], inf["items_per_thread"]) == expect_default, inf
        r, p = s.sample_debug(SEED, 0, samples, path_stride=stride)
        f = s.read_frame(0)
        frames.append(f)
        assert int(f[0]) == samples
        reach = r["dist"] != 0xFFFFFFFF
        assert int(f[1:].sum()) == int(r["path_len"].sum())
        assert np.array_equal(r["path_len"][reach], r["dist"][reach] - 1) and not r["path_len"][~reach].any()
        assert (r["s"] != r["t"]).all() and r["s"].max() < n and r["t"].max() < n
        assert int(f[1:].max()) <= samples
        if k == 0:
            rec, paths = r, p
            if block_count:  # a contiguous block of other indices into the second frame, word for word
                s.sample(SEED, block_first, block_count, frame=1)
                got = s.read_frame(1)
                want = oracle_frame(g.offsets, g.targets, SEED, block_first, block_count)
                assert np.array_equal(got, want), "epoch frame differs from the oracle's"
        else:
            assert np.array_equal(r["dist"], rec["dist"]) and np.array_equal(r["meet"], rec["meet"])
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
        if w["dist"] != 0xFFFFFFFF:
            assert int(r["meet_count"]) == len(o.last_meet_set()), i
        k = min(stride, len(w["path"]))
        assert np.array_equal(paths[int(i), :k], w["path"][:k])
    return frames[0]


def test_config2_rmat20_full_size():
    g = ebc.gen_rmat(20, 16, seed=2).largest_connected_component()
    assert (g.num_vertices, g.num_edges) == (645739, 15700555)
    f = _check(g, 107520, 300, 8, [(0, 0, 0), (64, 2, 0), (256, 4, 256)], expect_default=(32, 2))
    # the whole run's frame, word for word (was tools/soak_config2.py)
    assert np.array_equal(f, oracle_frame(g.offsets, g.targets, SEED, 0, 107520))


def test_config2_pipeline_full_size():
    """The whole config-2 run against an oracle replay: vertex-diameter bound and omega as the CPU oracle computes
    them, every epoch's frame from the oracle, check_stop (stopping.cpp:125-142) on the accumulated state after each
    epoch -- the stop epoch, tau and every counter must agree."""
    g = ebc.gen_rmat(20, 16, seed=2).largest_connected_component()
    res, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.005, delta=0.1, seed=SEED))
    o = Oracle(g.offsets, g.targets)
    n = g.num_vertices
    assert st["vertex_diameter_bound"] == o.diameter(4, SEED)[2]
    assert st["omega"] == Oracle.compute_omega(st["vertex_diameter_bound"], 0.005, 0.1) == 106052
    assert st["tau"] == st["epochs"] * st["n0"] >= st["omega"] > (st["epochs"] - 1) * st["n0"]
    dl, du = Oracle.calibrate(np.zeros(n + 1, dtype=np.uint64), n, 0.1, 0)
    S = np.zeros(n + 1, dtype=np.uint64)
    stop_epoch = None
    for e in range(st["epochs"] + 1):
        S += oracle_frame(g.offsets, g.targets, SEED, e * st["n0"], st["n0"])
        if Oracle.check_stop(S, 0.005, st["omega"], dl, du, 0):
            stop_epoch = e + 1
            break
    assert stop_epoch == st["epochs"] and int(S[0]) == st["tau"]
    assert np.array_equal(S[1:], res.counts)
    assert np.array_equal(res.scores, res.counts.astype(np.float64) / float(st["tau"]))


def test_config3_grid_full_size():
    g = ebc.gen_grid(2000, 2000, 0.05, 0.001, 3).largest_connected_component()
    assert g.num_vertices > 3_990_000
    f = _check(g, 6144, 200, 160, [(0, 0, 0), (256, 2, 64)], block_first=1 << 20, block_count=2000)
    assert int(f[1:].sum()) > 6144 * 40  # paths are long on the grid (mean ~85 internal vertices)


def test_config4_rmat24_full_size():
    """BASELINE configs[3]: R-MAT scale 24 (graph seed 4), default launch shape 256x4."""
    g = ebc.gen_rmat_device(24, 16, seed=4, take_lcc=True)
    assert g.num_vertices > 8_000_000 and g.num_edges > 250_000_000
    _check(g, 20480, 300, 8, [(0, 0, 0), (128, 4, 96)], block_first=3_000_000, block_count=2000,
           expect_default=(256, 4))


def test_config5_rmat26_full_size():
    """BASELINE configs[4]: Kronecker/R-MAT scale 26 (graph seed 5, 2.1 * 10^9 arcs), default launch shape 256x4."""
    g = ebc.gen_rmat_device(26, 16, seed=5, take_lcc=True)
    assert g.num_vertices > 30_000_000 and 2 * g.num_edges > 2_000_000_000
    _check(g, 20480, 300, 8, [(0, 0, 0), (512, 4, 64)], block_first=3_000_000, block_count=1000,
           expect_default=(256, 4))


def test_config1_er_full_run_twice_identical():
    g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component()
    a, sa = ebc.run_pipeline(g, ebc.RunConfig(eps=0.01, delta=0.1, seed=SEED))
    b, sb = ebc.run_pipeline(g, ebc.RunConfig(eps=0.01, delta=0.1, seed=SEED, block_threads=32, items_per_thread=2, slots=37))
    assert np.array_equal(a.counts, b.counts) and sa["tau"] == sb["tau"] == 32768 and sa["epochs"] == sb["epochs"]
