"""GPU parity: the CUDA sampling path (through the C ABI) against the CPU oracle, bit-exact.

Integer/index work => every comparison is exact equality.
"""
import numpy as np
import pytest

import paper_1910_11039_b200 as ebc
from helpers import (complete_bipartite_chain, cycle_graph, grid_graph, largest_component, path_graph,
                     random_graph, star_graph)
from oracle import Oracle

pytestmark = pytest.mark.gpu

SEED = 7


def small_graphs():
    return {
        "er200": random_graph(200, 400, 1),
        "er300dense": random_graph(300, 2000, 2),
        "grid12": grid_graph(12, 12, 0.05, 3),
        "layers40": complete_bipartite_chain([1] + [40] * 13 + [1]),   # sigma ~ 40^12: 128-bit weights
        "layers70": complete_bipartite_chain([3] + [70] * 12 + [2]),   # sigma saturates at 2^64-1
        "path4": path_graph(4),
        "cycle4": cycle_graph(4),
        "star5": star_graph(5),
        "disconnected": random_graph(50, 30, 5),
        "two_vertices": path_graph(2),
    }


def check_samples(g_csr, count, cfg, seed=SEED, first=0, pairs=None, stride=64):
    off, tg = g_csr
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s = ebc.Sampler(g, cfg)
    rec, paths = s.sample_debug(seed, first, count, pairs=pairs, path_stride=stride)
    frame = np.zeros(g.num_vertices + 1, dtype=np.uint64)
    for i in range(count):
        want = o.sample(seed, first + i, pair=None if pairs is None else tuple(int(x) for x in pairs[i]))
        got = rec[i]
        assert (int(got["s"]), int(got["t"])) == (want["s"], want["t"]), i
        assert int(got["dist"]) == want["dist"], (i, got, want)
        assert int(got["meet"]) == want["meet"], (i, got, want)
        assert int(got["draws"]) == want["draws"], (i, got, want)
        assert int(got["path_len"]) == len(want["path"]), (i, got, want)
        if want["dist"] != 0xFFFFFFFF:
            assert int(got["meet_count"]) == len(o.last_meet_set()), i
        if len(want["path"]) <= stride:
            assert np.array_equal(paths[i, :len(want["path"])], want["path"]), (i, paths[i], want["path"])
        frame[0] += 1
        np.add.at(frame, want["path"].astype(np.int64) + 1, 1)
    assert np.array_equal(s.read_frame(0), frame)
    return s, o


@pytest.mark.parametrize("name", list(small_graphs().keys()))
@pytest.mark.parametrize("block", [32, 128])
def test_small_graph_samples(name, block):
    csr = small_graphs()[name]
    cfg = ebc.RunConfig(block_threads=block, slots=8)
    check_samples(csr, 600, cfg)


@pytest.mark.parametrize("block", [32, 64, 256])
def test_search_state_matches_oracle(block):
    """dist / sigma of both sides after single samples (slots == 1 so the state stays inspectable)."""
    for name in ("er300dense", "layers40", "layers70", "grid12"):
        off, tg = small_graphs()[name]
        g = ebc.Graph.from_csr(off, tg)
        o = Oracle(off, tg)
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, slots=1, materialize_final_level=True))
        for i in range(25):
            rec, _ = s.sample_debug(SEED, i, 1)
            want = o.sample(SEED, i)
            assert int(rec[0]["dist"]) == want["dist"]
            for side in (0, 1):
                d, sg = s.last_state(side)
                od, osg = o.last_state(side)
                assert np.array_equal(d, od), (name, i, side)
                assert np.array_equal(sg, osg), (name, i, side)


def test_explicit_pairs_and_weights():
    off, tg = small_graphs()["layers70"]
    n = len(off) - 1
    pairs = np.array([[0, n - 1], [1, n - 2], [n - 1, 0], [5, 6], [0, 3]], dtype=np.uint32)
    s, o = check_samples((off, tg), len(pairs), ebc.RunConfig(block_threads=64, slots=2), pairs=pairs)
    rec, _ = s.sample_debug(SEED, 0, 1, pairs=pairs[:1])
    # 3 * 70^12 * 2 shortest paths: the saturating 128-bit total must agree with Python integers
    o.sample(SEED, 0, pair=(0, n - 1))
    fs = o.last_state(0)[1]
    bs = o.last_state(1)[1]
    total = sum(int(fs[v]) * int(bs[v]) for v in o.last_meet_set())
    total = min(total, 2 ** 128 - 1)
    assert (int(rec[0]["weight_hi"]) << 64) | int(rec[0]["weight_lo"]) == total


def test_capacity_overflow_reruns_in_large_slots():
    """A slot capacity far below what samples settle forces the re-run path; results must not change."""
    off, tg = small_graphs()["er300dense"]
    cfg = ebc.RunConfig(block_threads=32, slots=4, slot_capacity=8)
    s, _ = check_samples((off, tg), 400, cfg)
    rec, _ = s.sample_debug(SEED, 0, 400)
    assert (rec["flags"] & 1).sum() == 0  # records come from the completed (re-run) sample
    assert s.work()["samples"] == 800


def test_label_space_wraparound(monkeypatch):
    """Labels are base + 2 idx + side with base growing monotonically; when the u32 space runs out the slot's
    labels are zeroed and base restarts.  EBC_TEST_LABEL_BASE starts the slots just below the reset
    threshold so the slots cross it within a few samples."""
    off, tg = small_graphs()["grid12"]
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    n = g.num_vertices
    # reset happens when base + 2 cap + 2 >= 0xffffffff - 4096 - 4 (cap == n here)
    monkeypatch.setenv("EBC_TEST_LABEL_BASE", str(0xFFFFFFFF - 4096 - 4 - 2 * n - 2 - 4000))
    for block, slots in ((32, 1), (128, 3)):
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, slots=slots, materialize_final_level=True))
        s.sample(SEED, 0, 3000)
        assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 3000))
        rec, paths = s.sample_debug(SEED, 3000, 50, frame=1, path_stride=24)
        for i in range(50):
            w = o.sample(SEED, 3000 + i)
            assert int(rec[i]["dist"]) == w["dist"] and np.array_equal(paths[i, :len(w["path"])], w["path"])
    monkeypatch.delenv("EBC_TEST_LABEL_BASE")
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=32, slots=1))
    s.sample(SEED, 0, 20000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 20000))


def test_frames_accumulate_and_epochs_fold():
    off, tg = random_graph(2000, 9000, 11)
    (off, tg), _ = largest_component(off, tg)
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s = ebc.Sampler(g, ebc.RunConfig(materialize_final_level=True))
    n = g.num_vertices
    dl, du = ebc.calibrate(np.zeros(n + 1, dtype=np.uint64), n, 0.1)
    s.set_stopping(0.005, 10 ** 9, dl, du)  # Hoeffding width at tau=12000 is ~0.021: never stops here
    S = np.zeros(n + 1, dtype=np.uint64)
    for e in range(4):
        s.sample(SEED, e * 3000, 3000, frame=e & 1)
        assert not s.fold_and_check(e & 1)
        o.accumulate(SEED, e * 3000, 3000, frame=S)
        assert np.array_equal(s.read_state(), S)
        assert s.read_frame(e & 1).sum() == 0
    w = s.work()
    ow = o.work()
    for i, k in enumerate(ebc.WORK_NAMES[:11]):
        assert w[k] == int(ow[i]), k
    assert w["samples"] == 12000


def test_config1_er_counters_bit_exact():
    g = ebc.gen_erdos_renyi(10000, 50000, 1).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig())
    s.sample(SEED, 0, 8000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 8000))


def test_rmat14_counters_bit_exact():
    g = ebc.gen_rmat(14, 16, seed=2).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig())
    s.sample(SEED, 100, 4000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 100, 4000))
    rec, paths = s.sample_debug(SEED, 0, 200, frame=1, path_stride=16)
    for i in range(200):
        want = o.sample(SEED, i)
        assert int(rec[i]["meet"]) == want["meet"] and int(rec[i]["dist"]) == want["dist"]
        assert np.array_equal(paths[i, :len(want["path"])], want["path"])


@pytest.mark.parametrize("block,items", [(32, 1), (64, 2), (128, 4), (256, 4), (512, 2)])
def test_final_level_probe_is_result_identical(block, items):
    """Large last levels are only scanned (contact edges -> meet set); paths, counters and the work the
    reference algorithm defines must not change.  R-MAT-15 has levels far above the probe threshold."""
    g = ebc.gen_rmat(15, 16, seed=5).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    fast = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items))
    full = ebc.Sampler(g, ebc.RunConfig(block_threads=block, items_per_thread=items, materialize_final_level=True))
    rec, paths = fast.sample_debug(SEED, 0, 3000, path_stride=12)
    rec2, paths2 = full.sample_debug(SEED, 0, 3000, path_stride=12)
    assert (rec["flags"] & 2).sum() > 1000          # the probe path really ran
    assert (rec2["flags"] & 2).sum() == 0
    for k in ("s", "t", "dist", "meet", "meet_count", "draws", "path_len", "weight_lo", "weight_hi"):
        assert np.array_equal(rec[k], rec2[k]), k
    assert np.array_equal(paths, paths2)
    want = o.accumulate(SEED, 0, 3000)
    assert np.array_equal(fast.read_frame(0), want) and np.array_equal(full.read_frame(0), want)
    for i in range(0, 3000, 37):
        w = o.sample(SEED, i)
        assert (int(rec[i]["dist"]), int(rec[i]["meet"]), int(rec[i]["draws"])) == (w["dist"], w["meet"], w["draws"])
        assert int(rec[i]["meet_count"]) == len(o.last_meet_set())
        assert np.array_equal(paths[i, :len(w["path"])], w["path"])
    ow = dict(zip(ebc.WORK_NAMES[:11], (int(x) for x in o.work())))   # 3000 + 82 samples
    o2 = Oracle(g.offsets, g.targets)
    o2.accumulate(SEED, 0, 3000)
    ow = dict(zip(ebc.WORK_NAMES[:11], (int(x) for x in o2.work())))
    wf, wm = fast.work(), full.work()
    for k in ebc.WORK_NAMES[:11]:
        assert wm[k] == ow[k], k                      # materialised: every counter equals the reference algorithm's
    for k in ("E_bfs", "E_lvl", "V_exp", "M", "S_walk", "E_walk", "P_walk", "L", "levels"):
        assert wf[k] == ow[k], k                      # scanned edges, levels, walks: unchanged
    assert wf["V_set"] < ow["V_set"] and wf["F_chk"] < ow["F_chk"]   # last-level vertices are not settled


@pytest.mark.parametrize("block,bitmap", [(32, "0"), (32, "1"), (128, "0"), (128, "1")])
def test_large_contact_sets_are_resolved_without_settling(block, bitmap, monkeypatch):
    """A probed final level with far more contact edges than the shared-memory resolver holds (7800 here)
    goes through pick_meet_large: sigma sums per member by atomics in global scratch (they saturate at
    2^64-1 here), the meet vertex by a weighted quickselect over the 130 members' discovery keys whose weights
    (2^128 each, the total saturates) leave 128 bits in every prefix.  Layers 40^12 -> 60 -> 130 <- 60 <- 40^12:
    the frontier more than doubles into the middle, sigma reaches 40^12 * 60 > 2^64 there."""
    monkeypatch.setenv("EBC_BITMAP", bitmap)
    widths = [2] + [40] * 12 + [60, 130, 60] + [40] * 12 + [2]
    off, tg = complete_bipartite_chain(widths)
    core = len(off) - 1
    n = 60000                                     # isolated padding: the contact-edge buffer scales with n
    off = np.concatenate([off, np.full(n - core, off[-1], dtype=np.uint64)])
    pairs = np.array([[0, core - 1], [1, core - 2], [core - 1, 0], [0, core - 2], [core - 2, 1]], dtype=np.uint32)
    s, o = check_samples((off, tg), len(pairs), ebc.RunConfig(block_threads=block, slots=2), pairs=pairs)
    rec, _ = s.sample_debug(SEED, 0, len(pairs), pairs=pairs)
    assert np.all((rec["flags"] & 2) != 0) and np.all((rec["flags"] & 5) == 0)   # probed, nothing fell back
    assert np.all(rec["meet_count"] == 130)
    o.sample(SEED, 0, pair=(0, core - 1))
    fs, bs = o.last_state(0)[1], o.last_state(1)[1]
    assert max(int(fs[v]) for v in o.last_meet_set()) == 2 ** 64 - 1 or max(int(bs[v]) for v in o.last_meet_set()) == 2 ** 64 - 1
    total = min(sum(int(fs[v]) * int(bs[v]) for v in o.last_meet_set()), 2 ** 128 - 1)
    assert (int(rec[0]["weight_hi"]) << 64) | int(rec[0]["weight_lo"]) == total


@pytest.mark.parametrize("block", [32, 64, 256])
def test_meet_vertex_by_all_three_paths(block):
    """The meet vertex of a probed level is chosen in registers (at most 32 contact edges: flag 16), from shared
    memory (up to 128 ... 512 edges), or by the weighted quickselect in the slot's global arrays (more: flag 8).  An
    R-MAT graph takes all three; every sample's (s, t, d, meet, |meet set|, draws, path) and the total meet
    weight equal the oracle's."""
    g0 = ebc.gen_rmat(14, 24, seed=11).largest_connected_component()
    off, tg = g0.offsets.copy(), g0.targets.copy()
    s, o = check_samples((off, tg), 1200, ebc.RunConfig(block_threads=block, items_per_thread=2, slots=64), first=500)
    rec, _ = s.sample_debug(SEED, 500, 1200, frame=1)
    f = rec["flags"]
    probed = (f & 2) != 0
    assert ((f & 16) != 0).sum() > 100 and ((f & 8) != 0).sum() > (5 if block <= 64 else 0)
    assert (probed & ((f & 24) == 0)).sum() > 20          # the shared-memory path
    assert not ((f & 16) != 0)[~probed].any() and not ((f & 8) != 0)[~probed].any()
    for i in range(0, 1200, 7):
        o.sample(SEED, 500 + i)
        fs, bs = o.last_state(0)[1], o.last_state(1)[1]
        total = min(sum(int(fs[v]) * int(bs[v]) for v in o.last_meet_set()), 2 ** 128 - 1)
        assert (int(rec[i]["weight_hi"]) << 64) | int(rec[i]["weight_lo"]) == total, i
    s.close()


@pytest.mark.parametrize("block,bitmap", [(32, "1"), (32, "0"), (128, "1")])
def test_meet_paths_with_saturated_sigma_and_weights(block, bitmap, monkeypatch):
    """Every level is probed here (EBC_PROBE_MIN_SLOTS / EBC_PROBE_GROWTH_X4), so small contact sets reach the register
    path and the shared-memory path, too.  Seventy diamonds on either side double sigma seventy times: both sides'
    sigma are 2^64 - 1 where the searches meet, every weight is (2^64 - 1)^2 and the total saturates at 2^128 - 1 --
    carries of the butterfly total, prefixes that leave 128 bits, the quickselect's 'exceeds' rule.  The two layers in
    the middle decide the number of contact edges: 16 / 25 (registers), 64 / 120 (shared memory), 256 / 576 (global
    memory).  Records (meet vertex, |meet set|, draws, full paths) and total weights equal the oracle's."""
    monkeypatch.setenv("EBC_BITMAP", bitmap)
    monkeypatch.setenv("EBC_PROBE_MIN_SLOTS", "1")
    monkeypatch.setenv("EBC_PROBE_GROWTH_X4", "0")
    monkeypatch.setenv("EBC_ELL", "0")             # (the thin chains would otherwise take the fixed-stride-row kernel)
    seen = {"registers": 0, "shared": 0, "global": 0}
    for mid in ((4, 4), (5, 5), (8, 8), (3, 40, 3), (16, 16), (24, 24)):
        widths = [1] + [2, 1] * 70 + list(mid) + [1, 2] * 70 + [1]
        off, tg = complete_bipartite_chain(widths)
        core = len(off) - 1
        n = 30000                                  # isolated padding: the contact-edge buffer scales with n
        off = np.concatenate([off, np.full(n - core, off[-1], dtype=np.uint64)])
        pairs = np.array([[0, core - 1], [core - 1, 0], [1, core - 2], [core - 3, 2]], dtype=np.uint32)
        s, o = check_samples((off, tg), len(pairs), ebc.RunConfig(block_threads=block, slots=2), pairs=pairs, stride=320)
        rec, _ = s.sample_debug(SEED, 0, len(pairs), pairs=pairs, frame=1)
        for i in range(len(pairs)):
            o.sample(SEED, i, pair=tuple(int(x) for x in pairs[i]))
            fs, bs = o.last_state(0)[1], o.last_state(1)[1]
            total = min(sum(int(fs[v]) * int(bs[v]) for v in o.last_meet_set()), 2 ** 128 - 1)
            assert (int(rec[i]["weight_hi"]) << 64) | int(rec[i]["weight_lo"]) == total, (mid, i)
            f = int(rec[i]["flags"])
            if (f & 2) and total == 2 ** 128 - 1:
                seen["registers" if f & 16 else "global" if f & 8 else "shared"] += 1
        s.close()
    assert seen["registers"] > 0 and seen["shared"] > 0 and seen["global"] > 0, seen


def test_final_level_probe_with_tiny_edge_buffer_falls_back():
    """slot_capacity so small that the contact-edge buffer overflows: expand_level / large-slot fallbacks."""
    g = ebc.gen_rmat(13, 16, seed=9).largest_connected_component()
    o = Oracle(g.offsets, g.targets)
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=64, items_per_thread=2, slots=16, slot_capacity=64))
    s.sample(SEED, 0, 1500)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 0, 1500))


@pytest.mark.parametrize("reserved", [8, 140])
def test_reserved_sms_do_not_change_results(monkeypatch, reserved):
    """ebc_run_config.reserved_sms: CTAs of the main pass that land on the reserved SMs only hold the place until the
    rest of the grid runs elsewhere, then leave (room for the frame all-reduce of the previous epoch).  Frames are
    those of the oracle wherever the CTAs were placed, also with two launches in flight (both epoch lanes)."""
    monkeypatch.setenv("EBC_RESERVED_SMS", str(reserved))
    g0 = ebc.gen_rmat(12, 16, seed=5).largest_connected_component()
    off, tg = g0.offsets.copy(), g0.targets.copy()
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s = ebc.Sampler(g, ebc.RunConfig())
    s.sample(SEED, 100, 20000, frame=0)
    s.sample(SEED, 30000, 20000, frame=1)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 100, 20000))
    assert np.array_equal(s.read_frame(1), o.accumulate(SEED, 30000, 20000))
    s.close()


def _ring_lattice(n, chords=True):
    """Every vertex tied to i+1, i+2, i+5 (degree 6) plus a few chords: rows of five to eight entries, no hubs."""
    src = np.concatenate([np.arange(n)] * 3)
    dst = np.concatenate([(np.arange(n) + k) % n for k in (1, 2, 5)])
    if chords:
        c = np.arange(0, n, 37)
        src, dst = np.concatenate([src, c]), np.concatenate([dst, (c * 7 + n // 3) % n])
    from helpers import csr_from_edges
    return csr_from_edges(n, src, dst)


@pytest.mark.parametrize("block", [32, 64, 128])
def test_fixed_stride_rows_samples_state_and_work_counters(block, monkeypatch):
    """Graphs of maximum degree <= 8 take the fixed-stride-row kernel (expand_level_ell: both entry groups, hash-set
    dedup, parent masks, degrees carried in the entries).  Samples, paths, dist / sigma arrays and ALL work counters
    equal the oracle's -- that kernel settles every level, so V_set / F_chk / E_lvl need no materialize flag -- and
    the general kernel (EBC_ELL=0) gives the same records."""
    off, tg = _ring_lattice(3000)
    deg = np.diff(off)
    assert deg.max() <= 8 and deg.max() >= 7 and deg.min() >= 6
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s, _ = check_samples((off, tg), 500, ebc.RunConfig(block_threads=block, slots=8))
    assert s.info()["fixed_rows"]
    s.close()
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=block))
    s.sample(SEED, 1000, 6000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 1000, 6000))
    w, ow = s.work(), o.work()
    for i, k in enumerate(ebc.WORK_NAMES[:11]):
        assert w[k] == int(ow[i]), k
    rec_a, paths_a = s.sample_debug(SEED, 0, 300, frame=1, path_stride=32)
    s.close()
    s1 = ebc.Sampler(g, ebc.RunConfig(block_threads=block, slots=1))
    for i in range(10):
        s1.sample_debug(SEED, i, 1)
        o.sample(SEED, i)
        for side in (0, 1):
            d, sg = s1.last_state(side)
            od, osg = o.last_state(side)
            assert np.array_equal(d, od) and np.array_equal(sg, osg), (i, side)
    s1.close()
    monkeypatch.setenv("EBC_ELL", "0")
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=block))
    assert not s.info()["fixed_rows"]
    rec_b, paths_b = s.sample_debug(SEED, 0, 300, frame=1, path_stride=32)
    for f in ("s", "t", "dist", "meet", "meet_count", "draws", "path_len", "weight_lo", "weight_hi"):
        assert np.array_equal(rec_a[f], rec_b[f]), f
    assert np.array_equal(paths_a, paths_b)
    s.close()


@pytest.mark.parametrize("block,width", [(32, 4), (64, 4), (128, 4), (64, 8)])
def test_fixed_stride_rows_of_four_entries(block, width, monkeypatch):
    """Maximum degree <= 4 (a 2-D lattice with holes, here disconnected as well): rows are stored as 16 bytes
    (SamplerParams::ell_width = 4, kernel variant FIXED = 4: one entry group, half the dedup tables); EBC_ELL_WIDTH=8
    keeps the 32-byte rows.  Samples, paths, frames, all work counters and the dist / sigma arrays equal the oracle's."""
    if width == 8:
        monkeypatch.setenv("EBC_ELL_WIDTH", "8")
    off, tg = grid_graph(61, 47, drop=0.12, seed=5)
    assert np.diff(off).max() == 4
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s, _ = check_samples((off, tg), 500, ebc.RunConfig(block_threads=block, slots=8))
    assert s.info()["fixed_rows"] and s.info()["fixed_row_width"] == width
    s.close()
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=block))
    s.sample(SEED, 1000, 6000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 1000, 6000))
    w, ow = s.work(), o.work()
    for i, k in enumerate(ebc.WORK_NAMES[:11]):
        assert w[k] == int(ow[i]), k
    s.close()
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, work_counters=0))  # the kernels without statistics
    s.sample(SEED, 1000, 6000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 1000, 6000))
    s.close()
    s1 = ebc.Sampler(g, ebc.RunConfig(block_threads=block, slots=1))
    for i in range(10):
        s1.sample_debug(SEED, i, 1)
        o.sample(SEED, i)
        for side in (0, 1):
            d, sg = s1.last_state(side)
            od, osg = o.last_state(side)
            assert np.array_equal(d, od) and np.array_equal(sg, osg), (i, side)
    s1.close()
    for off2, tg2 in (path_graph(900), cycle_graph(901), grid_graph(40, 40)):  # degree 2 throughout; a full lattice
        s = ebc.Sampler(ebc.Graph.from_csr(off2, tg2), ebc.RunConfig(block_threads=block))
        assert s.info()["fixed_row_width"] == width
        s.sample(SEED, 0, 3000)
        assert np.array_equal(s.read_frame(0), Oracle(off2, tg2).accumulate(SEED, 0, 3000))
        s.close()


@pytest.mark.parametrize("block,copy16", [(32, "1"), (64, "1"), (128, "1"), (64, "0")])
def test_fixed_stride_rows_with_16_byte_copy(block, copy16, monkeypatch):
    """A lattice with a few shortcuts (config 3): rows of up to eight entries, but few have more than four.  The
    expansion then reads a 16-byte copy of every row (SamplerParams::ell4) and follows an escape word to the 32-byte
    row where it must; EBC_ELL4 forces the copy on (here also on a graph where EVERY row escapes) or off.  Samples,
    paths, frames, work counters and dist / sigma arrays equal the oracle's."""
    monkeypatch.setenv("EBC_ELL4", copy16)
    off, tg = grid_graph(53, 49, drop=0.05, seed=8)
    n = len(off) - 1
    rng = np.random.default_rng(3)
    src, dst = [], []
    for u in range(n):
        src += [u] * int(off[u + 1] - off[u]); dst += [int(x) for x in tg[off[u]:off[u + 1]]]
    extra = rng.integers(0, n, size=(60, 2))
    from helpers import csr_from_edges
    off, tg = csr_from_edges(n, np.concatenate([np.array(src), extra[:, 0]]), np.concatenate([np.array(dst), extra[:, 1]]))
    deg = np.diff(off)
    assert 4 < deg.max() <= 8 and (deg > 4).sum() * 8 < n
    for graph in ((off, tg), _ring_lattice(2000)):
        o_, t_ = graph
        g = ebc.Graph.from_csr(o_, t_)
        o = Oracle(o_, t_)
        s, _ = check_samples((o_, t_), 400, ebc.RunConfig(block_threads=block, slots=8))
        info = s.info()
        assert info["fixed_rows"] and info["fixed_row_width"] == 8 and info["fixed_row_copy16"] == (copy16 == "1")
        s.close()
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block))
        s.sample(SEED, 1000, 5000)
        assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 1000, 5000))
        w, ow = s.work(), o.work()
        for i, k in enumerate(ebc.WORK_NAMES[:11]):
            assert w[k] == int(ow[i]), k
        s.close()
        s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, work_counters=0))
        s.sample(SEED, 1000, 5000)
        assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 1000, 5000))
        s.close()


def test_fixed_stride_rows_need_a_symmetric_graph():
    """An arc without its reverse has no reverse position to record: the sampler notices while it builds the rows and
    runs the general kernel instead (validate=0 adopts the CSR as it is)."""
    off = np.array([0, 1, 3, 4], dtype=np.uint64)  # 0 -> 1, 1 -> {0, 2}, 2 -> 0 (2 -> 1 is missing)
    tg = np.array([1, 0, 2, 0], dtype=np.uint32)
    g = ebc.Graph.from_csr(off, tg, validate=False)
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=32, slots=2))
    assert not s.info()["fixed_rows"]
    s.close()


@pytest.mark.parametrize("name,block", [("er300dense", 32), ("grid12", 64), ("layers70", 128), ("rmat12", 64), ("rmat12", 256)])
def test_kernels_without_statistics_give_the_same_frames(name, block):
    """ebc_run_config.work_counters = 0 launches the production kernels (namespace ebc::lean: no work counters, records or
    state-dump bookkeeping).  Frames are the oracle's; the counters read zero; a launch that asks for records falls
    back to the kernels with statistics."""
    if name == "rmat12":
        g0 = ebc.gen_rmat(12, 16, seed=3).largest_connected_component()
        off, tg = g0.offsets.copy(), g0.targets.copy()
    else:
        off, tg = small_graphs()[name]
    g = ebc.Graph.from_csr(off, tg)
    o = Oracle(off, tg)
    s = ebc.Sampler(g, ebc.RunConfig(block_threads=block, work_counters=False))
    s.sample(SEED, 50, 3000)
    assert np.array_equal(s.read_frame(0), o.accumulate(SEED, 50, 3000))
    assert s.work()["samples"] == 0 and s.work()["E_bfs"] == 0
    rec, _ = s.sample_debug(SEED, 0, 40, frame=1)
    for i in range(40):
        want = o.sample(SEED, i)
        assert (int(rec[i]["s"]), int(rec[i]["t"]), int(rec[i]["dist"]), int(rec[i]["meet"])) == \
               (want["s"], want["t"], want["dist"], want["meet"])
    assert s.work()["samples"] == 40
    s.close()
    res_a, st_a = ebc.run_pipeline(g, ebc.RunConfig(eps=0.05, delta=0.1, seed=SEED, block_threads=block, work_counters=False))
    res_b, st_b = ebc.run_pipeline(g, ebc.RunConfig(eps=0.05, delta=0.1, seed=SEED, block_threads=block))
    assert np.array_equal(res_a.counts, res_b.counts) and st_a["tau"] == st_b["tau"] and st_a["epochs"] == st_b["epochs"]
    assert st_a["work"]["samples"] == 0 and st_b["work"]["samples"] > 0
