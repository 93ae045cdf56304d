"""Host-side mirror of the reference interface for the KADABRA sampling path, over the C ABI.

Names and argument meaning follow /root/reference/proj/include/epochbc/*.hpp
(Graph, RunConfig, ApproxResult, RunStats, compute_omega, calibrate,
epoch_length, check_stop, run_pipeline); errors map to the reference's exception
classes (types.hpp:15-36).  All sampling work runs in libebc_b200.so's CUDA
kernels; there is no CPU implementation in this package.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional

import numpy as np

from . import _capi
from ._capi import RunConfig as _CRunConfig
from ._capi import RunStats as _CRunStats
from ._capi import SampleRecord as _CSampleRecord

TAG_ADAPTIVE = 0
TAG_CALIBRATION = 1
HOEFFDING, EMPIRICAL_BERNSTEIN = 0, 1
UNIFORM, WEIGHTED = 0, 1
WORK_NAMES = ["E_bfs", "E_lvl", "V_exp", "V_set", "F_chk", "M", "S_walk", "E_walk", "P_walk", "L",
              "levels", "samples"]


class ParseError(RuntimeError):
    """Malformed input data (types.hpp:15-19); also I/O failures (CLI exit 3)."""


class ConfigError(RuntimeError):
    """Invalid parameters / violated caller contract (types.hpp:22-36; CLI exit 2)."""


class BackendFault(RuntimeError):
    """Communication backend failure (types.hpp:27-30; CLI exit 4)."""


class CudaError(RuntimeError):
    """CUDA failure or no device: this package has no CPU fallback."""


_ERRORS = {_capi.EBC_ERR_CONFIG: ConfigError, _capi.EBC_ERR_PARSE: ParseError,
           _capi.EBC_ERR_BACKEND: BackendFault, _capi.EBC_ERR_CUDA: CudaError}


def _check(status: int) -> None:
    if status != _capi.EBC_OK:
        msg = _capi.load().ebc_last_error().decode(errors="replace")
        raise _ERRORS.get(status, RuntimeError)(msg)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def parse_bound_kind(name: str) -> int:
    """stopping.cpp:7-13"""
    if name == "hoeffding":
        return HOEFFDING
    if name in ("eb", "empirical-bernstein"):
        return EMPIRICAL_BERNSTEIN
    raise ConfigError("unknown bound kind: " + name)


def parse_allocator_kind(name: str) -> int:
    """stopping.cpp:15-21"""
    if name == "uniform":
        return UNIFORM
    if name == "weighted":
        return WEIGHTED
    raise ConfigError("unknown allocator kind: " + name)


# ------------------------------------------------------------------------------ graph
class Graph:
    """Immutable undirected CSR graph (epochbc::Graph, graph.hpp:21-52): u64 offsets, u32 targets."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        L = _capi.load()
        self.num_vertices = int(L.ebc_graph_num_vertices(self._h))
        self.num_edges = int(L.ebc_graph_num_edges(self._h))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _capi.load().ebc_graph_free(self._h)
                self._h = None
        except Exception:
            pass

    @staticmethod
    def _new(fn, *args) -> "Graph":
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return Graph(out)

    @classmethod
    def from_edges(cls, n: int, src, dst) -> "Graph":
        """Graph::from_edges (graph.cpp:14-46)."""
        s = np.ascontiguousarray(src, dtype=np.uint64)
        d = np.ascontiguousarray(dst, dtype=np.uint64)
        if s.shape != d.shape:
            raise ConfigError("from_edges: src and dst differ in length")
        return cls._new(_capi.load().ebc_graph_from_edges, n, _p(s, _capi.u64p), _p(d, _capi.u64p), len(s))

    @classmethod
    def from_edges_device(cls, n: int, src, dst, take_lcc: bool = False, device: int = -1) -> "Graph":
        """from_edges (and optionally the largest component) computed on the GPU; same result."""
        s = np.ascontiguousarray(src, dtype=np.uint64)
        d = np.ascontiguousarray(dst, dtype=np.uint64)
        if s.shape != d.shape:
            raise ConfigError("from_edges: src and dst differ in length")
        return cls._new(_capi.load().ebc_graph_from_edges_device, n, _p(s, _capi.u64p), _p(d, _capi.u64p), len(s),
                        int(take_lcc), device)

    @classmethod
    def from_csr(cls, offsets, targets, original_ids=None, validate=True) -> "Graph":
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        t = np.ascontiguousarray(targets, dtype=np.uint32)
        ids = None if original_ids is None else np.ascontiguousarray(original_ids, dtype=np.uint64)
        # the native side copies offsets[0..n], targets[0..offsets[n]) and ids[0..n): the buffers must hold them
        if o.ndim != 1 or t.ndim != 1 or len(o) < 1:
            raise ConfigError("from_csr: offsets must be a non-empty 1-d array (n + 1 entries)")
        if int(o[-1]) != len(t):
            raise ConfigError("from_csr: offsets[n] must equal len(targets)")
        if ids is not None and (ids.ndim != 1 or len(ids) != len(o) - 1):
            raise ConfigError("from_csr: original_ids must hold n entries")
        return cls._new(_capi.load().ebc_graph_from_csr, len(o) - 1, _p(o, _capi.u64p), _p(t, _capi.u32p),
                        None if ids is None else _p(ids, _capi.u64p), int(validate))

    @classmethod
    def load(cls, path: str, take_lcc: bool = False) -> "Graph":
        """load_graph_file (graph.cpp:204-215); take_lcc as tools/epochbc.cpp:87."""
        return cls._new(_capi.load().ebc_graph_load, str(path).encode(), int(take_lcc))

    def save(self, path: str, binary: bool = False) -> None:
        _check(_capi.load().ebc_graph_save(self._h, str(path).encode(), int(binary)))

    def largest_connected_component(self, device: Optional[int] = None) -> "Graph":
        """largest_connected_component (graph.cpp:229-290); device=ordinal (or -1) computes it on the GPU."""
        if device is not None:
            return self._new(_capi.load().ebc_graph_lcc_device, self._h, device)
        return self._new(_capi.load().ebc_graph_lcc, self._h)

    @property
    def offsets(self) -> np.ndarray:
        p = _capi.load().ebc_graph_offsets(self._h)
        return np.ctypeslib.as_array(p, shape=(self.num_vertices + 1,)).copy()

    @property
    def targets(self) -> np.ndarray:
        if self.num_edges == 0:
            return np.zeros(0, dtype=np.uint32)
        p = _capi.load().ebc_graph_targets(self._h)
        return np.ctypeslib.as_array(p, shape=(2 * self.num_edges,)).copy()

    @property
    def original_ids(self) -> np.ndarray:
        if self.num_vertices == 0:
            return np.zeros(0, dtype=np.uint64)
        p = _capi.load().ebc_graph_original_ids(self._h)
        return np.ctypeslib.as_array(p, shape=(self.num_vertices,)).copy()

    def degree(self, v: int) -> int:
        o = self.offsets
        return int(o[v + 1] - o[v])


def gen_erdos_renyi(n: int, m: int, seed: int) -> Graph:
    return Graph._new(_capi.load().ebc_gen_erdos_renyi, n, m, seed)


def gen_rmat(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05, seed: int = 1) -> Graph:
    """R-MAT with gen_rmat's quadrant convention (rmat.cpp:24-42)."""
    return Graph._new(_capi.load().ebc_gen_rmat, scale, edge_factor, a, b, c, d, seed)


def gen_rmat_device(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05, seed: int = 1,
                    take_lcc: bool = False, device: int = -1) -> Graph:
    """gen_rmat (and optionally the largest component) generated and canonicalised on the GPU; same graph."""
    return Graph._new(_capi.load().ebc_gen_rmat_device, scale, edge_factor, a, b, c, d, seed, int(take_lcc), device)


def gen_grid(width: int, height: int, delete_prob: float, shortcut_fraction: float, seed: int) -> Graph:
    return Graph._new(_capi.load().ebc_gen_grid, width, height, delete_prob, shortcut_fraction, seed)


# ---------------------------------------------------------------- host-side parameters
def compute_omega(vertex_diameter_bound: int, eps: float, delta: float) -> int:
    """compute_omega (stopping.cpp:31-41)."""
    out = C.c_uint64()
    _check(_capi.load().ebc_compute_omega(vertex_diameter_bound, eps, delta, C.byref(out)))
    return int(out.value)


def epoch_length(ranks: int, threads: int, base: float = 1000.0, exponent: float = 1.33) -> int:
    """epoch_length (engine.cpp:26-31)."""
    out = C.c_uint64()
    _check(_capi.load().ebc_epoch_length(ranks, threads, base, exponent, C.byref(out)))
    return int(out.value)


def calibrate(calib_words, n: int, delta: float, allocator: int = UNIFORM):
    """calibrate (stopping.cpp:43-92) -> (delta_lower, delta_upper)."""
    w = np.ascontiguousarray(calib_words, dtype=np.uint64)
    if len(w) != n + 1:
        raise ConfigError("calibrate: frame must have n+1 words")
    dl = np.zeros(n, dtype=np.float64)
    du = np.zeros(n, dtype=np.float64)
    _check(_capi.load().ebc_calibrate(_p(w, _capi.u64p), n, delta, allocator, _p(dl, _capi.f64p),
                                      _p(du, _capi.f64p)))
    return dl, du


def shard_range(first: int, count: int, rank: int, world: int):
    a, b = C.c_uint64(), C.c_uint64()
    _capi.load().ebc_shard_range(first, count, rank, world, C.byref(a), C.byref(b))
    return int(a.value), int(b.value)


def diameter_upper_bound(g: Graph, sweeps: int = 4, seed: int = 0):
    """diameter_upper_bound (bfs.cpp:36-76) with GPU BFS sweeps -> (upper, lower, vertex_diameter_bound)."""
    out = np.zeros(3, dtype=np.uint64)
    _check(_capi.load().ebc_diameter_upper_bound(g._h, sweeps, seed, _p(out, _capi.u64p)))
    return int(out[0]), int(out[1]), int(out[2])


# ------------------------------------------------------------------------------- run
@dataclasses.dataclass
class RunConfig:
    """RunConfig (engine.hpp:59-81) for the GPU path."""
    eps: float = 0.001
    delta: float = 0.1
    seed: int = 1
    bound: int = HOEFFDING
    allocator: int = UNIFORM
    omega_override: int = 0
    calib_samples: int = 800
    diameter_sweeps: int = 4
    vertex_diameter_override: int = 0
    epoch_samples: int = 0
    max_epochs: int = 0
    device: int = -1
    rank: int = 0
    world_size: int = 1
    allreduce: Optional[object] = None  # ctypes callback (see distributed.py)
    allreduce_user: int = 0  # void* handed back to the callback (the ebc_nccl_comm of NativeNcclComm)
    block_threads: int = 0
    slots: int = 0
    slot_capacity: int = 0
    overlap: bool = True
    items_per_thread: int = 0
    materialize_final_level: bool = False
    renumber: int = 0  # device-side numbering: 0 auto, -1 never, 1 degree classes (hubs), 2 neighbourhood clusters
    reserved_sms: int = 0  # SMs left to the frame all-reduce: 0 auto (4 when world_size > 1), -1 none, k > 0
    work_counters: bool = True  # False: production kernels without work counters / state-dump bookkeeping (3-10 % faster)

    def to_c(self) -> _CRunConfig:
        c = _CRunConfig()
        _capi.load().ebc_run_config_default(C.byref(c))
        for f in ("eps", "delta", "seed", "bound", "allocator", "omega_override", "calib_samples",
                  "diameter_sweeps", "vertex_diameter_override", "epoch_samples", "max_epochs", "device",
                  "rank", "world_size", "block_threads", "slots", "slot_capacity", "items_per_thread", "renumber",
                  "reserved_sms"):
            setattr(c, f, getattr(self, f))
        c.overlap = int(self.overlap)
        c.materialize_final_level = int(self.materialize_final_level)
        c.work_counters = int(self.work_counters)
        if self.allreduce is not None:
            c.allreduce = self.allreduce
            c.allreduce_user = self.allreduce_user
        return c


@dataclasses.dataclass
class ApproxResult:
    """ApproxResult (engine.hpp:83-87) plus the raw counters."""
    scores: np.ndarray
    tau_total: int
    original_ids: np.ndarray
    counts: np.ndarray


def _stats_dict(st: _CRunStats) -> dict:
    d = {k: getattr(st, k) for k, _ in _CRunStats._fields_ if k != "work"}
    d["work"] = dict(zip(WORK_NAMES, [int(x) for x in st.work]))
    return d


def run_pipeline(g: Graph, cfg: RunConfig, scores_path: Optional[str] = None, stats_path: Optional[str] = None):
    """Full pipeline on this process' GPU (run_pipeline / run_simulated, engine.cpp:281-434).

    Returns (ApproxResult, stats dict).  scores_path / stats_path write the score file and the stats
    JSON exactly as the reference CLI's `run` does (tools/epochbc.cpp:219-224)."""
    L = _capi.load()
    c = cfg.to_c()
    out = C.c_void_p()
    _check(L.ebc_run(g._h, C.byref(c), C.byref(out)))
    owner = _ResultOwner(out)
    if scores_path is not None:
        _check(L.ebc_result_write_scores(out, C.byref(c), str(scores_path).encode()))
    if stats_path is not None:
        need = C.c_uint64()
        _check(L.ebc_result_stats_json(out, C.byref(c), None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(L.ebc_result_stats_json(out, C.byref(c), buf, need.value, None))
        with open(stats_path, "wb") as f:
            f.write(buf.value)
    n = C.c_uint64()
    sp = _capi.f64p()
    _check(L.ebc_result_scores(out, C.byref(sp), C.byref(n)))
    scores = owner.view(sp, C.c_double, n.value)
    cp = _capi.u64p()
    _check(L.ebc_result_counts(out, C.byref(cp), C.byref(n)))
    counts = owner.view(cp, C.c_uint64, n.value)
    ip = _capi.u64p()
    _check(L.ebc_result_original_ids(out, C.byref(ip), C.byref(n)))
    ids = owner.view(ip, C.c_uint64, n.value)
    st = _CRunStats()
    _check(L.ebc_result_stats(out, C.byref(st)))
    res = ApproxResult(scores, int(L.ebc_result_tau(out)), ids, counts)
    return res, _stats_dict(st)


class _ResultOwner:
    """Keeps an ebc_result alive for as long as any array that views its buffers (the arrays are the
    pointers the C ABI returns -- "borrowed from the result handle" -- not copies)."""

    def __init__(self, handle):
        self._h = handle

    def view(self, ptr, ctype, n: int) -> np.ndarray:
        if n == 0:
            return np.zeros(0, dtype=np.dtype(ctype))
        ca = (ctype * n).from_address(C.addressof(ptr.contents))
        ca._owner = self  # numpy keeps `ca` as the array's base, `ca` keeps the handle
        a = np.ctypeslib.as_array(ca)
        a.flags.writeable = False
        return a

    def __del__(self):
        try:
            if self._h:
                _capi.load().ebc_result_free(self._h)
                self._h = None
        except Exception:
            pass


# --------------------------------------------------------------------------- sampler
class Sampler:
    """Device-resident sampler (SearchScratch / WorkerState / epoch frames on the GPU)."""

    def __init__(self, g: Graph, cfg: Optional[RunConfig] = None):
        self._g = g
        self.n = g.num_vertices
        self._cfg = cfg or RunConfig()
        c = self._cfg.to_c()
        self._keep = c  # keeps the allreduce callback alive
        out = C.c_void_p()
        _check(_capi.load().ebc_sampler_create(g._h, C.byref(c), C.byref(out)))
        self._h = out

    def close(self):
        if getattr(self, "_h", None):
            _capi.load().ebc_sampler_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sample(self, seed: int, first: int, count: int, frame: int = 0, tag: int = TAG_ADAPTIVE):
        _check(_capi.load().ebc_sampler_sample(self._h, seed, tag, first, count, frame))

    def sample_debug(self, seed: int, first: int, count: int, pairs=None, frame: int = 0,
                     tag: int = TAG_ADAPTIVE, path_stride: int = 0):
        """-> (records structured array, paths [count, path_stride] or None)."""
        rec = (_CSampleRecord * max(count, 1))()
        pr = None
        if pairs is not None:
            pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
            if len(pr) != 2 * count:
                raise ConfigError("sample_debug: pairs must hold 2*count vertices")
        paths = np.full((count, path_stride), 0xFFFFFFFF, dtype=np.uint32) if path_stride else None
        _check(_capi.load().ebc_sampler_sample_debug(
            self._h, seed, tag, first, count, None if pr is None else _p(pr, _capi.u32p), frame, rec,
            None if paths is None else _p(paths, _capi.u32p), path_stride))
        dt = np.dtype([(k, np.uint32) for k in ("s", "t", "dist", "meet", "meet_count", "draws", "path_len",
                                                 "flags")] + [("weight_lo", np.uint64), ("weight_hi", np.uint64)])
        arr = np.frombuffer(rec, dtype=dt, count=count).copy()
        return arr, paths

    def last_state(self, side: int):
        d = np.zeros(self.n, dtype=np.uint32)
        s = np.zeros(self.n, dtype=np.uint64)
        _check(_capi.load().ebc_sampler_last_state(self._h, side, _p(d, _capi.u32p), _p(s, _capi.u64p)))
        return d, s

    def set_stopping(self, eps: float, omega: int, delta_lower, delta_upper, bound: int = HOEFFDING):
        dl = np.ascontiguousarray(delta_lower, dtype=np.float64)
        du = np.ascontiguousarray(delta_upper, dtype=np.float64)
        if len(dl) != self.n or len(du) != self.n:
            raise ConfigError("check_stop: calibration missing")
        _check(_capi.load().ebc_sampler_set_stopping(self._h, eps, omega, _p(dl, _capi.f64p),
                                                     _p(du, _capi.f64p), bound))

    def fold_and_check(self, frame: int = 0) -> bool:
        stop = C.c_int()
        _check(_capi.load().ebc_sampler_fold_and_check(self._h, frame, C.byref(stop)))
        return bool(stop.value)

    def read_frame(self, which: int) -> np.ndarray:
        w = np.zeros(self.n + 1, dtype=np.uint64)
        _check(_capi.load().ebc_sampler_read_frame(self._h, which, _p(w, _capi.u64p)))
        return w

    def read_state(self) -> np.ndarray:
        return self.read_frame(2)

    def write_state(self, words):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        if len(w) != self.n + 1:
            raise ConfigError("write_state: need n+1 words")
        _check(_capi.load().ebc_sampler_write_state(self._h, _p(w, _capi.u64p)))

    def clear(self):
        _check(_capi.load().ebc_sampler_clear(self._h))

    def work(self, reset: bool = False) -> dict:
        w = np.zeros(12, dtype=np.uint64)
        _check(_capi.load().ebc_sampler_work(self._h, _p(w, _capi.u64p), int(reset)))
        return dict(zip(WORK_NAMES, [int(x) for x in w]))

    def mark(self, event: int):
        _check(_capi.load().ebc_sampler_mark(self._h, event))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(_capi.load().ebc_sampler_elapsed_ms(self._h, a, b, C.byref(ms)))
        return float(ms.value)

    def sync(self):
        _check(_capi.load().ebc_sampler_sync(self._h))

    def info(self) -> dict:
        w = np.zeros(6, dtype=np.uint64)
        _check(_capi.load().ebc_sampler_info(self._h, _p(w, _capi.u64p)))
        return dict(slots=int(w[0]), block_threads=int(w[1]), slot_capacity=int(w[2]),
                    device_bytes=int(w[3]), sm_count=int(w[4]), launches=int(w[5]) & ((1 << 48) - 1),
                    renumbered=(int(w[5]) >> 48) & 0xF, fixed_rows=bool((int(w[5]) >> 52) & 1),
                    fixed_row_width=(4 if (int(w[5]) >> 53) & 1 else 8) if (int(w[5]) >> 52) & 1 else 0,
                    fixed_row_copy16=bool((int(w[5]) >> 54) & 1),
                    items_per_thread=int(w[5]) >> 56)

    def stream(self) -> int:
        p = C.c_void_p()
        _check(_capi.load().ebc_sampler_stream(self._h, C.byref(p)))
        return int(p.value or 0)

    def frame_ptr(self, frame: int):
        p = C.c_void_p()
        w = C.c_uint64()
        _check(_capi.load().ebc_sampler_frame_ptr(self._h, frame, C.byref(p), C.byref(w)))
        return int(p.value), int(w.value)

    def bfs(self, source: int, want_dist: bool = False):
        """GPU BFS (bfs.cpp:9-34) -> (dist or None, farthest, eccentricity, reached)."""
        d = np.zeros(self.n, dtype=np.uint32) if want_dist else None
        out = np.zeros(3, dtype=np.uint64)
        _check(_capi.load().ebc_sampler_bfs(self._h, source, None if d is None else _p(d, _capi.u32p),
                                            _p(out, _capi.u64p)))
        return d, int(out[0]), int(out[1]), int(out[2])

    def flush_l2(self):
        _check(_capi.load().ebc_sampler_flush_l2(self._h))


# --------------------------------------------------------------------- score files (N2)
def write_scores(path: str, vertex_ids, scores, meta: Optional[dict] = None) -> None:
    """write_scores (score_io.cpp:12-21)."""
    ids = np.ascontiguousarray(vertex_ids, dtype=np.uint64)
    sc = np.ascontiguousarray(scores, dtype=np.float64)
    if ids.shape != sc.shape:
        raise ConfigError("write_scores: ids and scores differ in length")
    meta = meta or {}
    keys = (C.c_char_p * max(len(meta), 1))(*[str(k).encode() for k in meta])
    vals = (C.c_char_p * max(len(meta), 1))(*[str(v).encode() for v in meta.values()])
    _check(_capi.load().ebc_scores_write(str(path).encode(), _p(ids, _capi.u64p), _p(sc, _capi.f64p), len(ids), keys,
                                         vals, len(meta)))


def read_scores(path: str):
    """read_scores (score_io.cpp:23-52) -> (meta dict for the given keys is fetched lazily, ids, scores)."""
    L = _capi.load()
    h = C.c_void_p()
    _check(L.ebc_scores_read(str(path).encode(), C.byref(h)))
    try:
        ip, sp, n = _capi.u64p(), _capi.f64p(), C.c_uint64()
        _check(L.ebc_scores_data(h, C.byref(ip), C.byref(sp), C.byref(n)))
        ids = np.ctypeslib.as_array(ip, shape=(n.value,)).copy() if n.value else np.zeros(0, dtype=np.uint64)
        sc = np.ctypeslib.as_array(sp, shape=(n.value,)).copy() if n.value else np.zeros(0, dtype=np.float64)
        meta = {}
        for k in ("eps", "delta", "tau", "seed", "algo"):
            v = L.ebc_scores_meta(h, k.encode())
            if v is not None:
                meta[k] = v.decode()
        return meta, ids, sc
    finally:
        L.ebc_scores_free(h)


def compare_score_files(approx_path: str, exact_path: str, eps: float) -> dict:
    """compare_scores (score_io.cpp:98-122) on two score files."""
    L = _capi.load()
    a, b = C.c_void_p(), C.c_void_p()
    _check(L.ebc_scores_read(str(approx_path).encode(), C.byref(a)))
    try:
        _check(L.ebc_scores_read(str(exact_path).encode(), C.byref(b)))
        try:
            rep = _capi.CompareReport()
            _check(L.ebc_scores_compare(a, b, eps, C.byref(rep)))
            return {k: getattr(rep, k) for k, _ in _capi.CompareReport._fields_}
        finally:
            L.ebc_scores_free(b)
    finally:
        L.ebc_scores_free(a)


def release_device_cache() -> None:
    """Frees the device buffers, streams and events the library keeps cached between runs."""
    _capi.load().ebc_release_device_cache()


def algorithmic_bytes(work: dict) -> int:
    """bytes the reference algorithm must move for the counted work."""
    w = work
    return (8 * (w["E_bfs"] + w["E_walk"]) + 16 * w["E_lvl"] + 24 * w["V_exp"] + 28 * w["V_set"]
            + 4 * w["F_chk"] + 16 * w["M"] + 16 * w["S_walk"] + 8 * w["P_walk"] + 8 * w["L"])
