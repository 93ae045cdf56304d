"""Host-side logic and the C-ABI surface (no GPU needed): every symbol include/ebc_b200.h declares is
exported, graph ingestion / generators / host-side stopping parameters behave like the reference, and
the GPU-only entry points fail loudly (EBC_ERR_CUDA) when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_1910_11039_b200 as ebc
from helpers import csr_from_edges, largest_component, random_graph
from oracle import Oracle
from paper_1910_11039_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "ebc_b200.h")).read()
    declared = set(re.findall(r"EBC_API[^;]*?\b(ebc_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 45
    L = _capi.load()
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/ebc_b200.h but not exported"
    assert declared == set(_capi.SIGNATURES.keys())
    assert b"sm_100a" in L.ebc_version()


def test_struct_layouts_match_header():
    """ctypes mirrors of ebc_run_config / ebc_run_stats / ebc_sample_record: default-init round trip."""
    c = _capi.RunConfig()
    _capi.load().ebc_run_config_default(C.byref(c))
    assert (c.eps, c.delta, c.seed, c.calib_samples, c.diameter_sweeps, c.device, c.world_size, c.overlap) == \
           (0.001, 0.1, 1, 800, 4, -1, 1, 1)
    assert C.sizeof(_capi.SampleRecord) == 48 and C.sizeof(_capi.RunStats) == 8 * 19 + 8 * 12


def test_from_edges_canonicalises_like_reference_contract():
    rng = np.random.default_rng(0)
    n = 300
    src, dst = rng.integers(0, n, 2500), rng.integers(0, n, 2500)
    src[:20] = dst[:20]  # self-loops
    g = ebc.Graph.from_edges(n, np.concatenate([src, src]), np.concatenate([dst, dst]))  # duplicates
    off, tg = csr_from_edges(n, src, dst)
    assert np.array_equal(g.offsets, off) and np.array_equal(g.targets, tg)
    assert g.num_edges == len(tg) // 2 and np.array_equal(g.original_ids, np.arange(n))
    g2 = ebc.Graph.from_csr(off, tg)
    assert np.array_equal(g2.targets, tg)
    with pytest.raises(ebc.ConfigError, match="out of range"):
        ebc.Graph.from_edges(10, [1], [10])


def test_from_csr_validation():
    off, tg = csr_from_edges(5, [0, 1, 2], [1, 2, 3])
    bad = tg.copy()
    bad[0], bad[1] = bad[1], bad[0] if len(bad) > 1 else bad[0]
    with pytest.raises(ebc.ConfigError):
        ebc.Graph.from_csr(np.array([0, 2, 2], dtype=np.uint64), np.array([1, 1], dtype=np.uint32))  # duplicate + asymmetric
    with pytest.raises(ebc.ConfigError):
        ebc.Graph.from_csr(np.array([0, 1, 2], dtype=np.uint64), np.array([0, 1], dtype=np.uint32))  # self-loops
    with pytest.raises(ebc.ConfigError):
        ebc.Graph.from_csr(np.array([0, 1, 2], dtype=np.uint64), np.array([1, 7], dtype=np.uint32))  # out of range


def test_lcc_matches_scipy_and_tie_break():
    off, tg = random_graph(400, 230, 7)
    g = ebc.Graph.from_csr(off, tg).largest_connected_component()
    (loff, ltg), keep = largest_component(off, tg)
    assert np.array_equal(g.offsets, loff) and np.array_equal(g.targets, ltg)
    assert np.array_equal(g.original_ids, keep.astype(np.uint64))
    # two components of equal size: the one holding the smallest original id wins (graph.cpp:262-267)
    g = ebc.Graph.from_edges(6, [3, 4, 0, 1], [4, 5, 1, 2]).largest_connected_component()
    assert list(g.original_ids) == [0, 1, 2]


def test_file_formats_round_trip(tmp_path):
    off, tg = random_graph(120, 300, 4)
    g = ebc.Graph.from_csr(off, tg).largest_connected_component()
    for binary in (True, False):
        p = str(tmp_path / ("g.ebcg" if binary else "g.txt"))
        g.save(p, binary)
        h = ebc.Graph.load(p)
        assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.targets, g.targets)
        assert np.array_equal(h.original_ids, g.original_ids)
    raw = open(str(tmp_path / "g.ebcg"), "rb").read()
    assert raw[:4] == b"EBCG" and int.from_bytes(raw[4:8], "little") == 1          # graph.cpp:138-174
    assert int.from_bytes(raw[8:16], "little") == g.num_vertices and int.from_bytes(raw[16:24], "little") == g.num_edges
    # text format details (graph.cpp:71-126)
    p = tmp_path / "t.txt"
    p.write_text("# comment\n% other comment\n\n10 20\n20 30 0.5\n30 10\n 40\t10 \n")
    h = ebc.Graph.load(str(p))
    assert list(h.original_ids) == [10, 20, 30, 40] and h.num_edges == 4
    h2 = ebc.Graph.load(str(p), take_lcc=True)
    assert h2.num_vertices == 4
    for bad, msg in (("1 2 3 4\n", "too many fields"), ("1 x\n", "malformed line"), ("# only\n", "no edges"),
                     ("5 5\n", "no edges after removing self-loops"), ("1 2 abc\n", "malformed token")):
        p.write_text(bad)
        with pytest.raises(ebc.ParseError, match=msg):
            ebc.Graph.load(str(p))
    with pytest.raises(ebc.ParseError, match="cannot open"):
        ebc.Graph.load(str(tmp_path / "missing.txt"))
    (tmp_path / "trunc.ebcg").write_bytes(raw[:40])
    with pytest.raises(ebc.ParseError, match="truncated"):
        ebc.Graph.load(str(tmp_path / "trunc.ebcg"))
    (tmp_path / "ver.ebcg").write_bytes(b"EBCG" + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ebc.ParseError, match="unsupported version"):
        ebc.Graph.load(str(tmp_path / "ver.ebcg"))


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
def test_ingestion_matches_unmodified_reference(tmp_path):
    from oracle import RefPlain
    rng = np.random.default_rng(5)
    n = 700
    src, dst = rng.integers(0, n, 900), rng.integers(0, n, 900)
    g = ebc.Graph.from_edges(n, src, dst)
    r = RefPlain.from_edges(n, src, dst)
    ro, rt, ri = r.csr()
    assert np.array_equal(g.offsets, ro) and np.array_equal(g.targets, rt.astype(np.uint32))
    gl, rl = g.largest_connected_component(), r.lcc()
    ro, rt, ri = rl.csr()
    assert np.array_equal(gl.offsets, ro) and np.array_equal(gl.targets, rt.astype(np.uint32)) and np.array_equal(gl.original_ids, ri)
    rl.save(str(tmp_path / "r.ebcg"), True)   # written by the reference, read by us
    h = ebc.Graph.load(str(tmp_path / "r.ebcg"))
    assert np.array_equal(h.offsets, ro) and np.array_equal(h.original_ids, ri)
    gl.save(str(tmp_path / "g.ebcg"), True)   # written by us, read by the reference
    ro2, rt2, ri2 = RefPlain.load(str(tmp_path / "g.ebcg")).csr()
    assert np.array_equal(ro2, ro) and np.array_equal(rt2, rt) and np.array_equal(ri2, ri)
    gl.save(str(tmp_path / "g.txt"), False)
    ro3, rt3, ri3 = RefPlain.load(str(tmp_path / "g.txt")).csr()
    assert np.array_equal(ro3, ro) and np.array_equal(ri3, ri)


def test_generators_are_seeded_and_shaped():
    a = ebc.gen_erdos_renyi(2000, 9000, 1)
    b = ebc.gen_erdos_renyi(2000, 9000, 1)
    c = ebc.gen_erdos_renyi(2000, 9000, 2)
    assert a.num_edges == 9000 and np.array_equal(a.targets, b.targets) and not np.array_equal(a.targets, c.targets)
    r1, r2 = ebc.gen_rmat(12, 16, seed=2), ebc.gen_rmat(12, 16, seed=2)
    assert r1.num_vertices == 4096 and np.array_equal(r1.targets, r2.targets)
    deg = np.diff(r1.offsets.astype(np.int64))
    assert deg.max() > 20 * max(deg.mean(), 1)            # heavy-tailed
    assert 0.5 * 16 * 4096 < r1.num_edges <= 16 * 4096    # dedup / loops remove some of the 16 * 2^12 samples
    # quadrant convention (rmat.cpp:26-40): a=1 -> every sample is (0,0), a self-loop, nothing survives
    assert ebc.gen_rmat(6, 4, 1.0, 0.0, 0.0, 0.0, seed=1).num_edges == 0
    only_b = ebc.gen_rmat(6, 4, 0.0, 1.0, 0.0, 0.0, seed=1)   # b: target bit only -> single edge (0, 63)
    assert only_b.num_edges == 1 and only_b.degree(0) == 1 and only_b.degree(63) == 1
    gr = ebc.gen_grid(50, 40, 0.05, 0.001, 3)
    full = 49 * 40 + 50 * 39
    assert gr.num_vertices == 2000 and 0.9 * full < gr.num_edges < full + 10
    assert ebc.gen_grid(5, 4, 0.0, 0.0, 1).num_edges == 4 * 4 + 5 * 3
    with pytest.raises(ebc.ConfigError):
        ebc.gen_rmat(31, 16)
    with pytest.raises(ebc.ConfigError):
        ebc.gen_rmat(10, 16, 0.5, 0.5, 0.5, 0.5)
    with pytest.raises(ebc.ConfigError):
        ebc.gen_erdos_renyi(4, 100, 1)


def test_host_side_stopping_parameters_match_oracle():
    for vd in (2, 3, 9, 257):
        for eps in (0.1, 0.01, 0.005, 0.001):
            assert ebc.compute_omega(vd, eps, 0.1) == Oracle.compute_omega(vd, eps, 0.1)
    assert ebc.compute_omega(2, 0.1, 0.1) == 166 and ebc.compute_omega(6, 0.05, 0.1) == 1061
    assert (ebc.epoch_length(1, 1), ebc.epoch_length(2, 2), ebc.epoch_length(16, 24)) == (1000, 158, 1)
    with pytest.raises(ebc.ConfigError):
        ebc.compute_omega(1, 0.1, 0.1)
    with pytest.raises(ebc.ConfigError):
        ebc.epoch_length(0, 1)
    rng = np.random.default_rng(1)
    n = 500
    calib = np.concatenate([[1000], rng.integers(0, 50, n)]).astype(np.uint64)
    for alloc in (ebc.UNIFORM, ebc.WEIGHTED):
        dl, du = ebc.calibrate(calib, n, 0.1, alloc)
        ol, ou = Oracle.calibrate(calib, n, 0.1, alloc)
        assert np.array_equal(dl, ol) and np.array_equal(du, ou)
        assert float(np.sum(dl) + np.sum(du)) <= 0.1 * (1 + 1e-12)  # budget up to summation rounding
    assert ebc.parse_bound_kind("eb") == ebc.EMPIRICAL_BERNSTEIN and ebc.parse_allocator_kind("weighted") == ebc.WEIGHTED
    with pytest.raises(ebc.ConfigError, match="unknown bound kind"):
        ebc.parse_bound_kind("chernoff")


def test_shard_range_partitions_every_epoch():
    for first, count, world in ((0, 10, 3), (1024, 7168, 8), (5, 1, 4), (0, 0, 2), (99, 1000, 1)):
        got = [ebc.shard_range(first, count, r, world) for r in range(world)]
        pos = first
        for lo, cnt in got:
            assert lo == pos
            pos += cnt
        assert pos == first + count
        sizes = [c for _, c in got]
        assert max(sizes) - min(sizes) <= 1


def test_gpu_entry_points_fail_loudly_without_a_device(have_gpu):
    if have_gpu:
        pytest.skip("a CUDA device is present")
    g = ebc.gen_erdos_renyi(100, 300, 1).largest_connected_component()
    with pytest.raises(ebc.CudaError, match="no CPU fallback"):
        ebc.Sampler(g)
    with pytest.raises(ebc.CudaError, match="no CPU fallback"):
        ebc.run_pipeline(g, ebc.RunConfig(eps=0.1))
    with pytest.raises(ebc.CudaError):
        ebc.diameter_upper_bound(g)


def test_product_does_not_link_or_import_the_oracle():
    """The shipped library and package must not reference anything under oracle/."""
    import subprocess
    syms = subprocess.run(["nm", "-D", _capi.lib_path()], capture_output=True, text=True).stdout
    assert "ebc_oracle" not in syms and "refshim" not in syms and "refplain" not in syms
    pkg = os.path.join(ROOT, "paper_1910_11039_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "oracle/" not in text.replace("reference/proj/src/oracle", ""), f


def test_score_files_round_trip_and_compare(tmp_path):
    """write_scores / read_scores / compare_scores (score_io.cpp) behave like the reference's."""
    rng = np.random.default_rng(3)
    n = 400
    ids = rng.permutation(np.arange(1000, 1000 + n)).astype(np.uint64)
    exact = rng.random(n) ** 6
    approx = exact + rng.normal(0, 0.003, n)
    approx[5] += 0.05
    pa, pe = str(tmp_path / "approx.tsv"), str(tmp_path / "exact.tsv")
    ebc.write_scores(pa, ids, approx, {"tau": 12345, "eps": 0.01, "delta": 0.1, "seed": 7, "algo": 2})
    ebc.write_scores(pe, ids[::-1].copy(), exact[::-1].copy())
    text = open(pa).read().splitlines()
    assert text[:5] == ["# algo=2", "# delta=0.1", "# eps=0.01", "# seed=7", "# tau=12345"]      # std::map key order
    assert text[5] == "%d\t%.12g" % (int(ids[0]), approx[0])
    meta, rid, rsc = ebc.read_scores(pa)
    assert meta["tau"] == "12345" and np.array_equal(rid, ids)
    assert np.array_equal(rsc, np.array([float("%.12g" % x) for x in approx]))
    rep = ebc.compare_score_files(pa, pe, 0.01)
    assert rep["vertices"] == n and rep["vertices_above_eps"] >= 1 and rep["max_abs_error"] > 0.04
    assert 0.0 <= rep["top10_overlap"] <= 1.0 and 0.0 <= rep["top100_overlap"] <= 1.0
    with pytest.raises(ebc.ConfigError, match="vertex sets differ"):
        ebc.write_scores(str(tmp_path / "other.tsv"), ids + 1, exact)
        ebc.compare_score_files(pa, str(tmp_path / "other.tsv"), 0.01)
    (tmp_path / "bad.tsv").write_text("# a=b\n12 x\n")
    with pytest.raises(ebc.ParseError, match="malformed line 2"):
        ebc.read_scores(str(tmp_path / "bad.tsv"))
    if oracle.have_ref():
        from oracle import RefPlain
        pr = str(tmp_path / "ref.tsv")
        RefPlain.write_scores(pr, ids, approx, {"tau": 12345, "eps": 0.01, "delta": 0.1, "seed": 7, "algo": 2})
        assert open(pr, "rb").read() == open(pa, "rb").read()                                       # byte-identical files
        want = RefPlain.compare_files(pa, pe, 0.01)
        for k, v in want.items():
            assert rep[k] == v, k


def test_native_nccl_transport_without_gpu():
    """ebc_nccl_*: the unique id needs no device; creating a communicator without one fails loudly with the
    CUDA status (no CPU fallback), and argument errors map to the config class."""
    import ctypes as C
    from paper_1910_11039_b200 import _capi
    L = _capi.load()
    a, b = C.create_string_buffer(128), C.create_string_buffer(128)
    assert L.ebc_nccl_unique_id(a) == 0 and L.ebc_nccl_unique_id(b) == 0
    assert a.raw != b.raw and a.raw != bytes(128)
    h = C.c_void_p()
    assert L.ebc_nccl_comm_create(a, 2, 2, -1, C.byref(h)) == 2      # rank out of range: EBC_ERR_CONFIG
    assert b"rank" in L.ebc_last_error()
    import torch
    if not torch.cuda.is_available():
        assert L.ebc_nccl_comm_create(a, 0, 1, -1, C.byref(h)) == 5  # EBC_ERR_CUDA
        assert b"no CUDA device" in L.ebc_last_error()
    assert L.ebc_nccl_allreduce(None, None, 0, None) == 1            # null communicator: hook reports failure
    L.ebc_nccl_comm_free(None)
