"""Pins the plain-C oracle to the UNMODIFIED reference compiled with the Philox stream shim
(oracle/_ref/libebc_ref_shim.so) on >= 10^4 random (graph, s, t, stream) cases, and to the plain
reference build for exact betweenness / diameter / ingestion.  Skipped where oracle/_ref is absent."""
import numpy as np
import pytest

import oracle
from helpers import complete_bipartite_chain, grid_graph, largest_component, random_graph
from oracle import Oracle, RefPlain, RefShim

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built (needs /root/reference)")


def test_ten_thousand_random_cases():
    cases = 0
    rng = np.random.default_rng(2024)
    for gi in range(14):
        n = int(rng.integers(20, 400))
        m = int(n * rng.uniform(0.8, 6.0))
        off, tg = random_graph(n, m, 100 + gi)
        o, r = Oracle(off, tg), RefShim(off, tg)
        for i in range(600):
            seed = int(rng.integers(0, 2 ** 63))
            a, b = o.sample(seed, i), r.sample(seed, i)
            assert (a["s"], a["t"], a["draws"]) == (b["s"], b["t"], b["draws"])
            assert np.array_equal(a["path"], b["path"])
            cases += 1
        # explicit pairs
        for i in range(150):
            s, t = (int(x) for x in rng.choice(n, 2, replace=False))
            a, b = o.sample(5, i, pair=(s, t)), r.sample(5, i, pair=(s, t))
            assert a["draws"] == b["draws"] and np.array_equal(a["path"], b["path"])
            for side in (0, 1):
                d1, s1 = o.last_state(side)
                d2, s2 = r.last_state(side)
                assert np.array_equal(d1, d2) and np.array_equal(s1, s2)
            cases += 1
    assert cases >= 10000


def test_wide_arithmetic_paths():
    """sigma saturation at 2^64-1 and 128-bit meet weights (sampler.cpp:11-30,121-133)."""
    for widths in ([1] + [40] * 13 + [1], [2] + [90] * 11 + [3], [1] + [17] * 33 + [1]):
        off, tg = complete_bipartite_chain(widths)
        o, r = Oracle(off, tg), RefShim(off, tg)
        n = len(off) - 1
        for i in range(200):
            a, b = o.sample(11, i), r.sample(11, i)
            assert a["draws"] == b["draws"] and np.array_equal(a["path"], b["path"])
        a, b = o.sample(11, 0, pair=(0, n - 1)), r.sample(11, 0, pair=(0, n - 1))
        assert a["draws"] == b["draws"] and np.array_equal(a["path"], b["path"])
        for side in (0, 1):
            assert np.array_equal(o.last_state(side)[1], r.last_state(side)[1])
        assert np.array_equal(o.last_meet_set(), r.last_meet_set())
    assert int(o.last_state(0)[1].max()) > 2 ** 63


def test_frames_stopping_and_brandes():
    (off, tg), _ = largest_component(*random_graph(600, 1500, 9))
    n = len(off) - 1
    o, r, p = Oracle(off, tg), RefShim(off, tg), RefPlain.from_csr(off, tg)
    assert np.array_equal(o.accumulate(3, 50, 3000), r.accumulate(3, 50, 3000))
    calib = r.accumulate(3, 0, 500, tag=1)
    for alloc in (0, 1):
        dl, du = Oracle.calibrate(calib, n, 0.1, alloc)
        rl, ru = RefShim.calibrate(calib, n, 0.1, alloc)
        assert np.array_equal(dl, rl) and np.array_equal(du, ru)
        S = np.zeros(n + 1, dtype=np.uint64)
        for e in range(10):
            r.accumulate(3, e * 400, 400, frame=S)
            for bound in (0, 1):
                for eps in (0.02, 0.05, 0.1, 0.2):
                    assert Oracle.check_stop(S, eps, 10 ** 9, dl, du, bound) == RefShim.check_stop(S, eps, 10 ** 9, rl, ru, bound)
    assert np.max(np.abs(o.brandes() - p.brandes(0))) <= 1e-12
    for seed in range(6):
        assert o.diameter(4, seed) == p.diameter(4, seed)
    off, tg = grid_graph(30, 20, 0.0, 0)
    assert Oracle(off, tg).diameter(4, 1) == RefPlain.from_csr(off, tg).diameter(4, 1)


def test_mt19937_restatement_matches_libstdcxx():
    rng = np.random.default_rng(1)
    bounds = np.concatenate([[0, 1, 2, 3], rng.integers(1, 2 ** 62, 500).astype(np.uint64)]).astype(np.uint64)
    for master, rank, thread in ((0, 0, 0), (7, 0, 0xd1a0), (2 ** 63 + 1, 5, 9)):
        assert np.array_equal(Oracle.mt_draws(master, rank, thread, bounds), RefPlain.rng_draws(master, rank, thread, bounds))
