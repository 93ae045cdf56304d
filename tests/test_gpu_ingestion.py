"""Graph ingestion on the GPU: from_edges canonicalisation, largest connected
component and the R-MAT generator must return exactly the graphs the host implementations return
(which in turn are checked against the reference's Graph::from_edges / largest_connected_component in
the CPU suite)."""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
gen_rmat_device = ebc.gen_rmat_device

pytestmark = pytest.mark.gpu


def same_graph(a, b):
    assert a.num_vertices == b.num_vertices and a.num_edges == b.num_edges
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.targets, b.targets)
    assert np.array_equal(a.original_ids, b.original_ids)


@pytest.mark.parametrize("scale,ef,seed", [(4, 2, 1), (10, 16, 2), (14, 16, 3), (16, 8, 4)])
def test_rmat_generator_matches_host(scale, ef, seed):
    same_graph(gen_rmat_device(scale, ef, seed=seed), ebc.gen_rmat(scale, ef, seed=seed))
    same_graph(gen_rmat_device(scale, ef, seed=seed, take_lcc=True),
               ebc.gen_rmat(scale, ef, seed=seed).largest_connected_component())


def test_rmat_generator_quadrant_corner_cases():
    # a = 1: every sample is the loop (0, 0) -> nothing survives; b = 1: the single edge (0, 2^scale - 1)
    assert gen_rmat_device(6, 4, 1.0, 0.0, 0.0, 0.0, seed=1).num_edges == 0
    same_graph(gen_rmat_device(6, 4, 0.0, 1.0, 0.0, 0.0, seed=1), ebc.gen_rmat(6, 4, 0.0, 1.0, 0.0, 0.0, seed=1))
    with pytest.raises(ebc.ConfigError):
        gen_rmat_device(10, 16, 0.5, 0.5, 0.5, 0.5)


def test_from_edges_matches_host():
    rng = np.random.default_rng(3)
    for n, m in ((1, 0), (2, 1), (50, 30), (1000, 5000), (20000, 300000)):
        src = rng.integers(0, n, size=m, dtype=np.uint64)
        dst = rng.integers(0, n, size=m, dtype=np.uint64)   # loops and duplicates (both directions) included
        if m > 10:
            src[:5], dst[:5] = dst[5:10].copy(), src[5:10].copy()
        host = ebc.Graph.from_edges(n, src, dst)
        same_graph(ebc.Graph.from_edges_device(n, src, dst), host)
        same_graph(ebc.Graph.from_edges_device(n, src, dst, take_lcc=True), host.largest_connected_component())
    with pytest.raises(ebc.ConfigError):
        ebc.Graph.from_edges_device(4, np.array([0, 9], dtype=np.uint64), np.array([1, 2], dtype=np.uint64))


def test_largest_component_tie_break_and_renumbering():
    # three components of equal size (paths 3-4-5, 0-1-2 split as 0-2 / isolated...), plus isolated vertices:
    # the tie goes to the component holding the smallest original id (graph.cpp:262-267)
    src = np.array([6, 7, 3, 4, 0, 1], dtype=np.uint64)
    dst = np.array([7, 8, 4, 5, 1, 2], dtype=np.uint64)
    g = ebc.Graph.from_edges(11, src, dst)
    same_graph(g.largest_connected_component(device=-1), g.largest_connected_component())
    assert list(g.largest_connected_component(device=-1).original_ids) == [0, 1, 2]
    # components of a component: original ids must be carried through a second pass
    big = ebc.gen_rmat(12, 2, seed=7)                      # sparse: many components
    lcc = big.largest_connected_component()
    same_graph(big.largest_connected_component(device=-1), lcc)
    same_graph(lcc.largest_connected_component(device=-1), lcc)
    # low-degree, high-diameter input (many hooking conflicts along long paths)
    grid = ebc.gen_grid(300, 200, 0.45, 0.0, 5)
    same_graph(grid.largest_connected_component(device=-1), grid.largest_connected_component())


def test_device_generated_graph_feeds_the_sampler():
    from oracle import Oracle
    g = gen_rmat_device(13, 16, seed=9, take_lcc=True)
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig())
    s.sample(7, 0, 1500)
    assert np.array_equal(s.read_frame(0), o.accumulate(7, 0, 1500))
