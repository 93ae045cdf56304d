#!/usr/bin/env python
"""Generates tests/golden/*.json from the UNMODIFIED reference (oracle/_ref, built from /root/reference).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (and through it the CUDA path) to outputs of the reference's
own compiled code: sample_pair / sample_shortest_path / apply_sample / check_stop / calibrate /
compute_omega under the Philox stream shim, and brandes_exact / diameter_upper_bound / epoch_length /
Rng (mt19937_64) from the plain build.  Graphs are stored as explicit edge lists, so the fixtures do
not depend on any random generator.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import (complete_bipartite_chain, csr_from_edges, cycle_graph, grid_graph, largest_component,  # noqa: E402
                     path_graph, random_graph, star_graph)
from oracle import RefPlain, RefShim  # noqa: E402

SEED = 7


def edges_of(off, tg):
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off.astype(np.int64)))
    keep = rows < tg
    return [[int(a), int(b)] for a, b in zip(rows[keep], tg[keep])]


def graphs():
    two_paths = csr_from_edges(6, [0, 1, 2, 0, 4, 5], [1, 2, 3, 4, 5, 3])  # two parallel length-3 paths 0..3
    triangle = cycle_graph(3)
    return {
        "path4": path_graph(4), "cycle4": cycle_graph(4), "triangle": triangle, "star5": star_graph(5),
        "two_parallel_paths": two_paths,
        "er120": largest_component(*random_graph(120, 260, 1))[0],
        "er_disconnected": random_graph(40, 25, 5),
        "grid9x7": grid_graph(9, 7, 0.08, 3),
        "layers30": complete_bipartite_chain([1] + [30] * 14 + [1]),  # 30^13 paths: u128 weights + saturation
    }


def main():
    oracle.build(ref=True)
    out = {"seed": SEED, "graphs": {}}
    for name, (off, tg) in graphs().items():
        n = len(off) - 1
        r = RefShim(off, tg)
        entry = {"n": n, "edges": edges_of(off, tg), "samples": [], "states": []}
        for i in range(60):
            s = r.sample(SEED, i)
            entry["samples"].append({"i": i, "s": s["s"], "t": s["t"], "draws": s["draws"],
                                     "path": [int(x) for x in s["path"]]})
            if i < 4:
                st = {"i": i}
                for side in (0, 1):
                    d, sg = r.last_state(side)
                    st[f"dist{side}"] = [int(x) for x in d]
                    st[f"sigma{side}"] = [str(int(x)) for x in sg]
                st["meet"] = [int(x) for x in r.last_meet_set()] if len(s["path"]) or True else []
                entry["states"].append(st)
        # explicit pairs (test hook: no pair draws)
        entry["explicit"] = []
        for (a, b) in [(0, n - 1), (n - 1, 0), (0, 1)]:
            s = r.sample(SEED, 1000, pair=(a, b))
            entry["explicit"].append({"s": a, "t": b, "draws": s["draws"], "path": [int(x) for x in s["path"]]})
        frame = r.accumulate(SEED, 0, 500)
        entry["frame500"] = [int(x) for x in frame]
        calib = r.accumulate(SEED, 0, 200, tag=1)
        entry["calib200"] = [int(x) for x in calib]
        # stopping: calibrate (uniform / weighted) and check_stop replay per epoch of 250 samples
        entry["stopping"] = []
        for bound in (0, 1):
            for alloc in (0, 1):
                dl, du = RefShim.calibrate(calib, n, 0.1, alloc)
                S = np.zeros(n + 1, dtype=np.uint64)
                decisions = []
                eps = 0.12 if bound == 0 else 0.2
                for e in range(12):
                    r.accumulate(SEED, e * 250, 250, frame=S)
                    decisions.append(int(RefShim.check_stop(S, eps, 10 ** 9, dl, du, bound)))
                entry["stopping"].append({"bound": bound, "allocator": alloc, "eps": eps,
                                          "delta_lower": [float.hex(float(x)) for x in dl],
                                          "delta_upper": [float.hex(float(x)) for x in du],
                                          "decisions": decisions, "final_S": [int(x) for x in S]})
        # plain build: exact betweenness, diameter phase
        p = RefPlain.from_csr(off, tg)
        entry["brandes"] = [float.hex(float(x)) for x in p.brandes(2)]
        try:
            entry["diameter"] = {str(seed): list(p.diameter(4, seed)) for seed in (0, 7, 99)}
            d, far, ecc, reached = p.bfs(0)
            entry["bfs0"] = {"dist": [int(x) for x in d], "farthest": far, "ecc": ecc, "reached": reached}
        except ValueError:
            entry["diameter"] = "disconnected"
        out["graphs"][name] = entry
    out["compute_omega"] = [[vd, eps, delta, RefShim.compute_omega(vd, eps, delta)]
                            for vd in (2, 3, 6, 9, 11, 257, 1000) for eps in (0.1, 0.05, 0.01, 0.005, 0.001)
                            for delta in (0.1, 0.01)]
    out["epoch_length"] = [[p_, t_, RefPlain.epoch_length(p_, t_)] for p_, t_ in
                           [(1, 1), (2, 2), (16, 24), (1, 8), (4, 1), (8, 8)]]
    bounds = [0, 10, 1000, 2 ** 40 + 7, 3, 0, 17, 2 ** 63 + 5, 1] * 4
    out["mt_stream"] = {"args": [7, 0, 0xd1a0], "bounds": [str(b) for b in bounds],
                        "draws": [str(int(x)) for x in RefPlain.rng_draws(7, 0, 0xd1a0, bounds)]}
    out["bound_width"] = [[b, dv, tau, kind, float.hex(RefShim.bound(b, dv, tau, kind))]
                          for b in (0.0, 0.013, 0.5, 1.0) for dv in (1e-5, 0.0125) for tau in (2, 877, 5000)
                          for kind in (0, 1)]
    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
