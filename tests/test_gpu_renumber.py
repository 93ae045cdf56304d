"""Device-side numberings (ebc_run_config.renumber: 1 = degree classes, 2 = neighbourhood clusters) must be
invisible: samples, paths, frames, search state, work counters and the full pipeline are those of the caller's
graph, bit for bit.

The numbering is automatic on hub graphs (max degree >= 1024: degree classes) and on large hub-free graphs
(>= 2^18 vertices: clusters), so the small graphs force it with renumber=1 / 2 and the hub graphs are also run
with renumber=-1."""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from oracle import Oracle
from test_gpu_parity import SEED, check_samples, small_graphs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", list(small_graphs().keys()))
def test_small_graph_samples_renumbered(name, mode):
    check_samples(small_graphs()[name], 600, ebc.RunConfig(block_threads=64, slots=8, renumber=mode))


def test_explicit_pairs_renumbered():
    off, tg = small_graphs()["layers70"]
    n = len(off) - 1
    pairs = np.array([[0, n - 1], [1, n - 2], [n - 1, 0], [5, 6], [0, 3]], dtype=np.uint32)
    check_samples((off, tg), len(pairs), ebc.RunConfig(block_threads=64, slots=2, renumber=1), pairs=pairs)


def test_search_state_renumbered():
    for name in ("er300dense", "layers70", "grid12"):
        off, tg = small_graphs()[name]
        g = ebc.Graph.from_csr(off, tg)
        o = Oracle(off, tg)
        for mode in (1, 2):
            s = ebc.Sampler(g, ebc.RunConfig(block_threads=64, slots=1, materialize_final_level=True, renumber=mode))
            assert s.info()["renumbered"] == mode
            for i in range(25):
                rec, _ = s.sample_debug(SEED, i, 1)
                want = o.sample(SEED, i)
                assert int(rec[0]["dist"]) == want["dist"]
                for side in (0, 1):
                    d, sg = s.last_state(side)
                    od, osg = o.last_state(side)
                    assert np.array_equal(d, od), (name, i, side)
                    assert np.array_equal(sg, osg), (name, i, side)


@pytest.mark.parametrize("materialize", [False, True])
def test_hub_graph_both_numberings_agree(materialize):
    g = ebc.gen_rmat(15, 16, seed=5).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    want = o.accumulate(SEED, 0, 3000)
    ow = dict(zip(ebc.WORK_NAMES[:11], (int(x) for x in o.work())))
    out = []
    for mode in (1, -1, 2):
        s = ebc.Sampler(g, ebc.RunConfig(renumber=mode, materialize_final_level=materialize))
        rec, paths = s.sample_debug(SEED, 0, 3000, path_stride=12)
        assert np.array_equal(s.read_frame(0), want)
        w = s.work()
        for k in (ebc.WORK_NAMES[:11] if materialize else
                  ("E_bfs", "E_lvl", "V_exp", "M", "S_walk", "E_walk", "P_walk", "L", "levels")):
            assert w[k] == ow[k], (mode, k)
        out.append((rec, paths))
    for other in out[1:]:
        for k in ("s", "t", "dist", "meet", "meet_count", "draws", "path_len", "weight_lo", "weight_hi", "flags"):
            assert np.array_equal(out[0][0][k], other[0][k]), k
        assert np.array_equal(out[0][1], other[1])
    for i in range(0, 3000, 41):
        w = o.sample(SEED, i)
        assert (int(out[0][0][i]["dist"]), int(out[0][0][i]["meet"])) == (w["dist"], w["meet"])
        assert np.array_equal(out[0][1][i, :len(w["path"])], w["path"])


def test_randomly_labelled_hub_graph():
    """Arbitrary input ids (the case the numbering helps most): shuffle an R-MAT graph's labels."""
    g0 = ebc.gen_rmat(13, 16, seed=3).largest_connected_component()
    off, tg = g0.offsets, g0.targets
    n = len(off) - 1
    perm = np.random.default_rng(5).permutation(n)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off).astype(np.int64))
    keep = src < tg
    g = ebc.Graph.from_edges(n, perm[src[keep]].astype(np.uint64), perm[tg[keep].astype(np.int64)].astype(np.uint64))
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig())
    assert s.info()["renumbered"] == 1
    s.sample(SEED, 0, 4000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 4000))


def test_pipeline_identical_with_and_without_numbering():
    g = ebc.gen_rmat(14, 16, seed=2).largest_connected_component()
    res = []
    for mode in (1, -1):
        cfg = ebc.RunConfig(eps=0.02, delta=0.1, seed=3, renumber=mode)
        res.append(ebc.run_pipeline(g, cfg))
    (a, sa), (b, sb) = res
    assert np.array_equal(a.scores, b.scores) and np.array_equal(a.counts, b.counts)
    assert a.tau_total == b.tau_total
    for k in ("tau", "epochs", "omega", "diameter_upper_bound", "vertex_diameter_bound"):
        assert sa[k] == sb[k], k


def test_large_hub_free_graph_is_clustered_automatically():
    """A grid above 2^18 vertices gets the neighbourhood-cluster numbering by default; frames equal the oracle's
    and those of the unnumbered run."""
    g = ebc.gen_grid(600, 600, 0.05, 0.001, 3).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    want = o.accumulate(SEED, 0, 1500)
    for mode, expect in ((0, 2), (-1, 0)):
        s = ebc.Sampler(g, ebc.RunConfig(renumber=mode))
        assert s.info()["renumbered"] == expect
        rec, paths = s.sample_debug(SEED, 0, 1500, path_stride=200)
        assert np.array_equal(s.read_frame(0), want)
        for i in range(0, 1500, 97):
            w = o.sample(SEED, i)
            assert (int(rec[i]["dist"]), int(rec[i]["meet"]), int(rec[i]["draws"])) == (w["dist"], w["meet"], w["draws"])
            assert np.array_equal(paths[i, :len(w["path"])], w["path"][:200])
        s.close()
