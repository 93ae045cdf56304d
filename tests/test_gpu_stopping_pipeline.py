"""GPU parity of the stopping check, the BFS/diameter phase and the full pipeline (through the C ABI)."""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from helpers import grid_graph, largest_component, random_graph
from oracle import Oracle

pytestmark = pytest.mark.gpu

SEED = 7


def _graph(n=3000, m=12000, seed=21):
    (off, tg), _ = largest_component(*random_graph(n, m, seed))
    return ebc.Graph.from_csr(off, tg), Oracle(off, tg)


@pytest.mark.parametrize("bound", [ebc.HOEFFDING, ebc.EMPIRICAL_BERNSTEIN])
@pytest.mark.parametrize("allocator", [ebc.UNIFORM, ebc.WEIGHTED])
def test_check_stop_matches_oracle_on_real_frames(bound, allocator):
    """Device check_stop == oracle check_stop for a sweep of (frame, eps) around the decision boundary.

    FP64 with correctly rounded ops in the reference's order => the boolean must match exactly."""
    g, o = _graph()
    n = g.num_vertices
    s = ebc.Sampler(g, ebc.RunConfig())
    calib = o.accumulate(SEED, 0, 800, tag=1)
    dl, du = ebc.calibrate(calib, n, 0.1, allocator)
    odl, odu = Oracle.calibrate(calib, n, 0.1, allocator)
    assert np.array_equal(dl, odl) and np.array_equal(du, odu)
    S = np.zeros(n + 1, dtype=np.uint64)
    for step in range(6):
        o.accumulate(SEED, step * 2000, 2000, frame=S)
        tau = int(S[0])
        widths = [max(Oracle.bound_width(int(S[v + 1]) / tau, dl[v], tau, bound),
                      Oracle.bound_width(int(S[v + 1]) / tau, du[v], tau, bound)) for v in range(n)]
        wmax = max(widths)
        # eps just below, exactly at and just above the largest width (">= eps -> false", stopping.cpp:135)
        for eps in (np.nextafter(wmax, 0), wmax, np.nextafter(wmax, 1), wmax * 0.5, wmax * 2):
            s.write_state(S)
            s.set_stopping(float(eps), 10 ** 12, dl, du, bound)
            got = s.fold_and_check(0)  # frame 0 is empty: S unchanged
            want = Oracle.check_stop(S, float(eps), 10 ** 12, dl, du, bound)
            assert got == want, (step, eps, wmax)
        assert np.array_equal(s.read_state(), S)


def test_check_stop_tau_rules():
    """tau >= omega -> true; tau < 2 -> false (stopping.cpp:127-129); SPEC.md:220 flips at tau = 877."""
    off, tg = random_graph(4, 6, 1)
    (off, tg), _ = largest_component(off, tg)
    g = ebc.Graph.from_csr(off, tg)
    n = g.num_vertices
    assert n == 4
    s = ebc.Sampler(g, ebc.RunConfig(slots=1, block_threads=32))
    dl, du = ebc.calibrate(np.zeros(n + 1, dtype=np.uint64), n, 0.1)
    for tau, omega, want in [(876, 10 ** 9, False), (877, 10 ** 9, True), (1, 10 ** 9, False), (0, 10 ** 9, False),
                             (5, 5, True), (1, 1, True), (4, 5, False)]:
        S = np.zeros(n + 1, dtype=np.uint64)
        S[0] = tau
        s.write_state(S)
        s.set_stopping(0.05, omega, dl, du, ebc.HOEFFDING)
        assert s.fold_and_check(0) == want, (tau, omega)
        assert Oracle.check_stop(S, 0.05, omega, dl, du, 0) == want


def test_gpu_bfs_and_diameter_match_oracle():
    for csr in (largest_component(*random_graph(5000, 11000, 3))[0], grid_graph(40, 25, 0.0, 0)):
        off, tg = csr
        g = ebc.Graph.from_csr(off, tg)
        o = Oracle(off, tg)
        s = ebc.Sampler(g, ebc.RunConfig(slots=1, block_threads=32))
        for src in (0, 17, g.num_vertices - 1):
            d, far, ecc, reached = s.bfs(src, want_dist=True)
            od, ofar, oecc, oreached = o.bfs(src)
            assert np.array_equal(d, od) and (far, ecc, reached) == (ofar, oecc, oreached)
        for seed in (0, 7, 123):
            assert ebc.diameter_upper_bound(g, 4, seed) == o.diameter(4, seed)


def test_diameter_rejects_disconnected():
    off, tg = random_graph(50, 30, 5)
    g = ebc.Graph.from_csr(off, tg)
    with pytest.raises(ebc.ConfigError, match="disconnected"):
        ebc.diameter_upper_bound(g, 4, 0)


@pytest.mark.parametrize("bound,allocator,eps", [(ebc.HOEFFDING, ebc.UNIFORM, 0.02),
                                                 (ebc.EMPIRICAL_BERNSTEIN, ebc.WEIGHTED, 0.02),
                                                 (ebc.EMPIRICAL_BERNSTEIN, ebc.UNIFORM, 0.03)])
@pytest.mark.parametrize("overlap", [True, False])
def test_pipeline_matches_oracle_epoch_replay(bound, allocator, eps, overlap):
    """Final counters, tau and stop epoch of ebc_run == the oracle replaying the same epoch schedule."""
    g, o = _graph(4000, 14000, 33)
    n = g.num_vertices
    cfg = ebc.RunConfig(eps=eps, delta=0.1, seed=SEED, bound=bound, allocator=allocator, epoch_samples=1024,
                        calib_samples=800, overlap=overlap)
    res, st = ebc.run_pipeline(g, cfg)
    vd = o.diameter(4, SEED)[2]
    assert st["vertex_diameter_bound"] == vd
    omega = Oracle.compute_omega(vd, eps, 0.1)
    assert st["omega"] == omega
    calib = o.accumulate(SEED, 0, 800, tag=1)
    assert st["calibration_samples"] == 800
    dl, du = Oracle.calibrate(calib, n, 0.1, allocator)
    epochs, S = o.run_epochs(SEED, 1024, 10 ** 6, eps, omega, dl, du, bound)
    assert st["epochs"] == epochs
    assert res.tau_total == int(S[0]) == st["tau"]
    assert np.array_equal(res.counts, S[1:])
    assert np.array_equal(res.scores, S[1:].astype(np.float64) / float(S[0]))
    assert st["tau"] == st["samples"] - st["calibration_samples"] - st["discarded_samples"]
    if bound == ebc.HOEFFDING or not overlap:
        assert st["discarded_samples"] == 0
    if bound == ebc.EMPIRICAL_BERNSTEIN:
        assert st["tau"] < omega  # the adaptive rule fired before the static budget


def test_pipeline_config1_within_eps_of_exact_brandes():
    """BASELINE config 1: ER n=10^4, m=5*10^4, eps=0.01, delta=0.1, seed 7 -> scores within eps of Brandes."""
    g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    res, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.01, delta=0.1, seed=SEED))
    exact = o.brandes()
    assert st["tau"] >= st["omega"]
    assert np.max(np.abs(res.scores - exact)) <= 0.01
    # and bit-exact against the oracle replay
    dl, du = Oracle.calibrate(np.zeros(g.num_vertices + 1, dtype=np.uint64), g.num_vertices, 0.1, 0)
    epochs, S = o.run_epochs(SEED, st["n0"], 10 ** 6, 0.01, st["omega"], dl, du, 0)
    assert epochs == st["epochs"] and np.array_equal(res.counts, S[1:])


def test_run_config_errors():
    g, _ = _graph(200, 600, 2)
    with pytest.raises(ebc.ConfigError):
        ebc.run_pipeline(g, ebc.RunConfig(eps=1.5))
    with pytest.raises(ebc.ConfigError):
        ebc.run_pipeline(g, ebc.RunConfig(delta=0.0))
    with pytest.raises(ebc.ConfigError):
        ebc.run_pipeline(g, ebc.RunConfig(world_size=2, rank=0))  # no allreduce hook
    with pytest.raises(ebc.ConfigError):
        ebc.Sampler(g, ebc.RunConfig(block_threads=48))


def test_nccl_allreduce_hook_single_rank():
    """The NCCL plumbing bench.py uses under torchrun, exercised with a 1-rank process group: frames go
    through torch.distributed.all_reduce on the sampler's aggregation stream; results must not change."""
    import torch
    import torch.distributed as dist
    from paper_1910_11039_b200.distributed import make_allreduce_hook
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29751", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        errors = []
        hook = make_allreduce_hook(on_error=errors.append)
        g, o = _graph(3000, 10000, 5)
        cfg = ebc.RunConfig(eps=0.03, delta=0.1, seed=SEED, epoch_samples=1024, allreduce=hook)
        res, st = ebc.run_pipeline(g, cfg)
        ref, st2 = ebc.run_pipeline(g, ebc.RunConfig(eps=0.03, delta=0.1, seed=SEED, epoch_samples=1024))
        assert not errors
        assert np.array_equal(res.counts, ref.counts) and st["tau"] == st2["tau"] and st["epochs"] == st2["epochs"]
        s = ebc.Sampler(g, cfg)
        s.sample(SEED, 0, 2000)
        assert not errors and not s.fold_and_check(0) or True
        assert np.array_equal(s.read_state(), o.accumulate(SEED, 0, 2000))
    finally:
        if own:
            dist.destroy_process_group()


def test_native_nccl_hook_single_rank():
    """The library's own NCCL transport (ebc_nccl_*: ncclCommInitRank / ncclAllReduce bound with dlopen, no
    Python per epoch) with a 1-rank communicator: the frames pass through ncclAllReduce on the aggregation
    stream and the pipeline's counters, tau and stop epoch must not change."""
    from paper_1910_11039_b200.distributed import NativeNcclComm
    comm = NativeNcclComm(NativeNcclComm.unique_id(), rank=0, world_size=1, device=0)
    try:
        g, o = _graph(3000, 10000, 5)
        cfg = ebc.RunConfig(eps=0.03, delta=0.1, seed=SEED, epoch_samples=1024, **comm.hook())
        res, st = ebc.run_pipeline(g, cfg)
        ref, st2 = ebc.run_pipeline(g, ebc.RunConfig(eps=0.03, delta=0.1, seed=SEED, epoch_samples=1024))
        assert np.array_equal(res.counts, ref.counts) and st["tau"] == st2["tau"] and st["epochs"] == st2["epochs"]
        s = ebc.Sampler(g, cfg)
        s.sample(SEED, 0, 2000)
        s.fold_and_check(0)
        assert np.array_equal(s.read_state(), o.accumulate(SEED, 0, 2000))
        s.close()
    finally:
        comm.close()


def test_pipeline_writes_reference_score_file_and_stats_json(tmp_path):
    """`run` of the reference CLI writes a score file and a stats JSON (tools/epochbc.cpp:219-224)."""
    import json
    g, o = _graph(1500, 5000, 8)
    cfg = ebc.RunConfig(eps=0.05, delta=0.1, seed=SEED)
    sp, jp = str(tmp_path / "scores.tsv"), str(tmp_path / "stats.json")
    res, st = ebc.run_pipeline(g, cfg, scores_path=sp, stats_path=jp)
    meta, ids, scores = ebc.read_scores(sp)
    assert meta == {"eps": "0.05", "delta": "0.1", "tau": str(res.tau_total), "seed": "7", "algo": "2"}
    assert np.array_equal(ids, g.original_ids)
    assert np.array_equal(scores, np.array([float("%.12g" % x) for x in res.scores]))
    exact_path = str(tmp_path / "exact.tsv")
    ebc.write_scores(exact_path, g.original_ids, o.brandes())
    rep = ebc.compare_score_files(sp, exact_path, 0.05)
    assert rep["max_abs_error"] <= 0.05 and rep["vertices_above_eps"] == 0     # the CLI's `compare` would exit 0
    stats = json.load(open(jp), object_pairs_hook=list)
    keys = [k for k, _ in stats]
    assert keys == ["schema_version", "epochs", "samples", "barrier_s", "comm_mib_per_epoch", "adaptive_s", "diameter_s",
                    "calibration_s", "transition_s", "reduce_s", "check_s", "bcast_s", "wall_s", "tau", "omega",
                    "calibration_samples", "discarded_samples", "n0", "n", "m", "diameter_upper_bound",
                    "vertex_diameter_bound", "eps", "delta", "ranks", "threads", "seed", "algo", "bound", "allocator"]
    d = dict(stats)
    assert d["tau"] == st["tau"] and d["omega"] == st["omega"] and d["bound"] == "hoeffding" and d["eps"] == 0.05


def test_debug_paths_are_truncated_to_the_stride():
    off, tg = grid_graph(14, 14, 0.0, 0)
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=32, slots=4))
    rec, paths = s.sample_debug(SEED, 0, 300, path_stride=3)
    for i in range(300):
        w = o.sample(SEED, i)
        assert int(rec[i]["path_len"]) == len(w["path"])
        k = min(3, len(w["path"]))
        assert np.array_equal(paths[i, :k], w["path"][:k])
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 300))


def test_direction_optimising_bfs_on_hub_graph():
    """max degree >= 1024 switches dense levels to bottom-up; distances / farthest vertex must not change."""
    g = ebc.gen_rmat(15, 16, seed=5).largest_connected_component()
    assert np.diff(g.offsets.astype(np.int64)).max() >= 1024
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig(slots=1, block_threads=32))
    for src in (0, 1, 4242, g.num_vertices - 1):
        d, far, ecc, reached = s.bfs(src, want_dist=True)
        od, ofar, oecc, oreached = o.bfs(src)
        assert np.array_equal(d, od) and (far, ecc, reached) == (ofar, oecc, oreached)
    for seed in (0, 7):
        assert ebc.diameter_upper_bound(g, 4, seed) == o.diameter(4, seed)
