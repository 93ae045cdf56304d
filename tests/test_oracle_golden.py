"""The CPU oracle (oracle/ebc_oracle.c) against golden vectors generated from the UNMODIFIED reference
(tests/golden/reference_golden.json, made by tests/golden/make_golden.py) and against the worked
examples of the reference's SPEC.md.  No GPU needed."""
import json
import os

import numpy as np
import pytest

from helpers import csr_from_edges, cycle_graph, path_graph, star_graph
from oracle import Oracle

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "reference_golden.json")) as f:
    GOLD = json.load(f)
SEED = GOLD["seed"]


def graph_of(entry):
    e = np.array(entry["edges"], dtype=np.int64).reshape(-1, 2)
    return csr_from_edges(entry["n"], e[:, 0], e[:, 1])


def test_philox_known_answers():
    """Random123 known-answer vectors for philox4x32-10."""
    kat = [([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
           ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
           ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1])]
    for ctr, key, want in kat:
        assert [int(x) for x in Oracle.philox_block(ctr, key)] == want


def test_stream_next_below_is_lemire():
    bounds = np.array([1, 2, 3, 10, 1000, 2 ** 32 + 1, 2 ** 63 + 5], dtype=np.uint64)
    raw = Oracle.stream_draws(9, 3, 12345, np.zeros(len(bounds), dtype=np.uint64))
    got = Oracle.stream_draws(9, 3, 12345, bounds)
    for b, x, g in zip(bounds, raw, got):
        m = int(x) * int(b)
        if (m & (2 ** 64 - 1)) >= ((2 ** 64 - int(b)) % int(b)):  # no rejection on this draw
            assert int(g) == m >> 64


@pytest.mark.parametrize("name", list(GOLD["graphs"].keys()))
def test_samples_match_reference(name):
    entry = GOLD["graphs"][name]
    off, tg = graph_of(entry)
    o = Oracle(off, tg)
    for want in entry["samples"]:
        got = o.sample(SEED, want["i"])
        assert (got["s"], got["t"], got["draws"]) == (want["s"], want["t"], want["draws"])
        assert [int(x) for x in got["path"]] == want["path"]
        for st in entry["states"]:
            if st["i"] == want["i"]:
                for side in (0, 1):
                    d, sg = o.last_state(side)
                    assert [int(x) for x in d] == st[f"dist{side}"]
                    assert [str(int(x)) for x in sg] == st[f"sigma{side}"]
                if got["dist"] != 0xFFFFFFFF:
                    assert [int(x) for x in o.last_meet_set()] == st["meet"]
    for want in entry["explicit"]:
        got = o.sample(SEED, 1000, pair=(want["s"], want["t"]))
        assert got["draws"] == want["draws"] and [int(x) for x in got["path"]] == want["path"]
    assert [int(x) for x in o.accumulate(SEED, 0, 500)] == entry["frame500"]
    assert [int(x) for x in o.accumulate(SEED, 0, 200, tag=1)] == entry["calib200"]


@pytest.mark.parametrize("name", list(GOLD["graphs"].keys()))
def test_stopping_matches_reference(name):
    entry = GOLD["graphs"][name]
    off, tg = graph_of(entry)
    o = Oracle(off, tg)
    n = entry["n"]
    calib = np.array(entry["calib200"], dtype=np.uint64)
    for case in entry["stopping"]:
        dl, du = Oracle.calibrate(calib, n, 0.1, case["allocator"])
        assert [float.hex(float(x)) for x in dl] == case["delta_lower"]
        assert [float.hex(float(x)) for x in du] == case["delta_upper"]
        S = np.zeros(n + 1, dtype=np.uint64)
        dec = []
        for e in range(12):
            o.accumulate(SEED, e * 250, 250, frame=S)
            dec.append(int(Oracle.check_stop(S, case["eps"], 10 ** 9, dl, du, case["bound"])))
        assert dec == case["decisions"]
        assert [int(x) for x in S] == case["final_S"]
        # run_epochs replays the same schedule and stops at the first positive decision
        if 1 in dec:
            epochs, S2 = o.run_epochs(SEED, 250, 12, case["eps"], 10 ** 9, dl, du, case["bound"])
            assert epochs == dec.index(1) + 1


@pytest.mark.parametrize("name", list(GOLD["graphs"].keys()))
def test_brandes_and_diameter_match_reference(name):
    entry = GOLD["graphs"][name]
    off, tg = graph_of(entry)
    o = Oracle(off, tg)
    want = np.array([float.fromhex(x) for x in entry["brandes"]])
    assert np.max(np.abs(o.brandes(2) - want)) <= 1e-12
    if entry["diameter"] == "disconnected":
        with pytest.raises(ValueError):
            o.diameter(4, 0)
    else:
        for seed, w in entry["diameter"].items():
            assert list(o.diameter(4, int(seed))) == w
        d, far, ecc, reached = o.bfs(0)
        assert [int(x) for x in d] == entry["bfs0"]["dist"]
        assert (far, ecc, reached) == (entry["bfs0"]["farthest"], entry["bfs0"]["ecc"], entry["bfs0"]["reached"])


def test_scalar_functions_match_reference():
    for vd, eps, delta, want in GOLD["compute_omega"]:
        assert Oracle.compute_omega(vd, eps, delta) == want
    for p, t, want in GOLD["epoch_length"]:
        assert Oracle.epoch_length(p, t) == want
    for b, dv, tau, kind, want in GOLD["bound_width"]:
        assert float.hex(Oracle.bound_width(b, dv, tau, kind)) == want
    m = GOLD["mt_stream"]
    got = Oracle.mt_draws(*m["args"], np.array([int(x) for x in m["bounds"]], dtype=np.uint64))
    assert [str(int(x)) for x in got] == m["draws"]


# ---- worked examples of the reference's SPEC.md ----
def test_spec_examples_stopping():
    assert Oracle.compute_omega(2, 0.1, 0.1) == 166
    assert Oracle.compute_omega(6, 0.05, 0.1) == 1061
    assert Oracle.epoch_length(1, 1) == 1000 and Oracle.epoch_length(2, 2) == 158 and Oracle.epoch_length(16, 24) == 1
    assert abs(Oracle.bound_width(0.3, 1e-5, 5000, 0) - 0.033931) < 1e-6
    dl, du = Oracle.calibrate(np.zeros(5, dtype=np.uint64), 4, 0.1, 0)
    assert np.all(dl == 0.0125) and np.all(du == 0.0125)      # SPEC.md: n=4, delta=.1 uniform
    S = np.zeros(5, dtype=np.uint64)
    for tau, want in ((876, False), (877, True)):
        S[0] = tau
        assert Oracle.check_stop(S, 0.05, 10 ** 9, dl, du, 0) == want
    S[0] = 10
    assert Oracle.check_stop(S, 0.05, 10, dl, du, 0)          # tau = omega -> true
    # weighted allocator: budget invariant and more mass on the sampled vertex
    calib = np.array([100, 50, 0, 0, 0], dtype=np.uint64)
    wl, wu = Oracle.calibrate(calib, 4, 0.1, 1)
    assert wl[0] > 0.0125 / 2 and float(np.sum(wl) + np.sum(wu)) <= 0.1


def test_spec_examples_sampler_and_exact():
    o = Oracle(*path_graph(4))
    assert [int(x) for x in o.sample(SEED, 0, pair=(0, 3))["path"]] == [1, 2]   # unique path
    assert np.allclose(o.brandes(1), [0, 1 / 3, 1 / 3, 0])
    assert abs(Oracle(*star_graph(5)).brandes(1)[0] - 0.6) < 1e-12
    tri = Oracle(*cycle_graph(3))
    assert all(len(tri.sample(SEED, i)["path"]) == 0 for i in range(50))         # adjacent endpoints
    c4 = Oracle(*cycle_graph(4))
    hits = sum(int(c4.sample(SEED, i, pair=(0, 2))["path"][0] == 1) for i in range(20000))
    assert abs(hits - 10000) < 3 * 71                                            # each middle vertex ~1/2
    two = Oracle(*csr_from_edges(6, [0, 1, 2, 0, 4, 5], [1, 2, 3, 4, 5, 3]))
    first = [tuple(int(x) for x in two.sample(SEED, i, pair=(0, 3))["path"]) for i in range(20000)]
    assert set(first) == {(1, 2), (4, 5)} and abs(first.count((1, 2)) - 10000) < 3 * 71


def test_sample_pair_uniform():
    o = Oracle(*cycle_graph(3))
    counts = {}
    for i in range(60000):
        s = o.sample(SEED, i)
        counts[(s["s"], s["t"])] = counts.get((s["s"], s["t"]), 0) + 1
    assert len(counts) == 6 and all(abs(c - 10000) < 4 * 92 for c in counts.values())


def test_unbiased_against_exact_on_small_graph():
    """SPEC.md sampler invariant: |c/tau - b| <= 4 sqrt(b(1-b)/tau) + 1e-4 at tau = 200000, n <= 30."""
    rng = np.random.default_rng(3)
    off, tg = csr_from_edges(24, rng.integers(0, 24, 60), rng.integers(0, 24, 60))
    o = Oracle(off, tg)
    tau = 200000
    f = o.accumulate(SEED, 0, tau)
    b = o.brandes(1)
    est = f[1:].astype(np.float64) / tau
    assert np.all(np.abs(est - b) <= 4 * np.sqrt(b * (1 - b) / tau) + 1e-4)
