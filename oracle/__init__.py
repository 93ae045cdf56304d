"""TEST INFRASTRUCTURE -- ctypes loaders for the CPU checkers under oracle/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package; the shipped product
(paper_1910_11039_b200) never does.

Three checkers:
  Oracle    oracle/libebc_oracle.so           plain-C restatement (ebc_oracle.c)
  RefShim   oracle/_ref/libebc_ref_shim.so    UNMODIFIED reference sampler/stopping + Philox shim
  RefPlain  oracle/_ref/libebc_ref_plain.so   UNMODIFIED reference library (mt19937_64)
The two _ref libraries are compiled from /root/reference by oracle/Makefile in
the build container and travel prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)

WORK_NAMES = ["E_bfs", "E_lvl", "V_exp", "V_set", "F_chk", "M", "S_walk", "E_walk", "P_walk", "L",
              "levels"]


def algorithmic_bytes(work) -> int:
    """B = 8(E_bfs+E_walk) + 16 E_lvl + 24 V_exp + 28 V_set + 4 F_chk
    + 16 M + 16 S_walk + 8 P_walk + 8 L, from the implementation-independent work counters."""
    w = dict(zip(WORK_NAMES, [int(x) for x in work]))
    return (8 * (w["E_bfs"] + w["E_walk"]) + 16 * w["E_lvl"] + 24 * w["V_exp"] + 28 * w["V_set"]
            + 4 * w["F_chk"] + 16 * w["M"] + 16 * w["S_walk"] + 8 * w["P_walk"] + 8 * w["L"])


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and, when /root/reference is present, the _ref libraries."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _as(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def have_ref() -> bool:
    return (os.path.exists(os.path.join(HERE, "_ref", "libebc_ref_shim.so"))
            and os.path.exists(os.path.join(HERE, "_ref", "libebc_ref_plain.so")))


# --------------------------------------------------------------------------------------
class Oracle:
    """Plain-C restatement (oracle/ebc_oracle.c) on a CSR with u64 offsets / u32 targets."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            path = os.path.join(HERE, "libebc_oracle.so")
            if not os.path.exists(path):
                build(ref=False)
            L = C.CDLL(path)
            L.ebc_oracle_create.restype = C.c_void_p
            L.ebc_oracle_create.argtypes = [C.c_uint64, _u64p, _u32p]
            L.ebc_oracle_destroy.argtypes = [C.c_void_p]
            L.ebc_oracle_sample.restype = C.c_uint64
            L.ebc_oracle_sample.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                            C.c_uint32, C.c_uint32, _u32p, _u64p]
            L.ebc_oracle_last_state.argtypes = [C.c_void_p, C.c_int, _u32p, _u64p]
            L.ebc_oracle_last_meet_set.restype = C.c_uint64
            L.ebc_oracle_last_meet_set.argtypes = [C.c_void_p, _u32p, C.c_uint64]
            L.ebc_oracle_accumulate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                                C.c_uint64, _u64p]
            L.ebc_oracle_work.argtypes = [C.c_void_p, _u64p]
            L.ebc_oracle_work_reset.argtypes = [C.c_void_p]
            L.ebc_oracle_compute_omega.restype = C.c_uint64
            L.ebc_oracle_compute_omega.argtypes = [C.c_uint64, C.c_double, C.c_double]
            L.ebc_oracle_epoch_length.restype = C.c_uint64
            L.ebc_oracle_epoch_length.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
            L.ebc_oracle_calibrate.argtypes = [_u64p, C.c_uint64, C.c_double, C.c_int, _f64p, _f64p]
            L.ebc_oracle_bound_width.restype = C.c_double
            L.ebc_oracle_bound_width.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int]
            L.ebc_oracle_check_stop.restype = C.c_int
            L.ebc_oracle_check_stop.argtypes = [_u64p, C.c_uint64, C.c_double, C.c_uint64, _f64p,
                                                _f64p, C.c_int]
            L.ebc_oracle_run_epochs.restype = C.c_uint64
            L.ebc_oracle_run_epochs.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                                C.c_uint64, C.c_double, C.c_uint64, _f64p, _f64p,
                                                C.c_int, _u64p]
            L.ebc_oracle_bfs.argtypes = [C.c_void_p, C.c_uint32, _u32p, _u32p, _u64p]
            L.ebc_oracle_diameter.restype = C.c_int
            L.ebc_oracle_diameter.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _u64p]
            L.ebc_oracle_mt_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p, C.c_uint64,
                                              _u64p]
            L.ebc_oracle_philox_block.argtypes = [_u32p, _u32p, _u32p]
            L.ebc_oracle_stream_draws.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, _u64p,
                                                  C.c_uint64, _u64p]
            L.ebc_oracle_brandes_block.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, _f64p]
            L.ebc_oracle_brandes_finish.argtypes = [C.c_uint64, _f64p]
            cls._lib = L
        return cls._lib

    def __init__(self, offsets, targets):
        self.offsets = _as(offsets, np.uint64)
        self.targets = _as(targets, np.uint32)
        self.n = len(self.offsets) - 1
        L = self.lib()
        self.h = L.ebc_oracle_create(self.n, _ptr(self.offsets, _u64p), _ptr(self.targets, _u32p))
        self._path = np.zeros(max(self.n, 1), dtype=np.uint32)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib().ebc_oracle_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def sample(self, seed, index, tag=0, pair=None):
        """-> dict(s, t, dist, meet, draws, path) for stream (seed, tag, index)."""
        info = np.zeros(5, dtype=np.uint64)
        s, t = (0, 0) if pair is None else pair
        ln = self.lib().ebc_oracle_sample(self.h, seed, tag, index, 0 if pair is None else 1, s, t,
                                          _ptr(self._path, _u32p), _ptr(info, _u64p))
        return dict(s=int(info[0]), t=int(info[1]), dist=int(info[2]), meet=int(info[3]),
                    draws=int(info[4]), path=self._path[:ln].copy())

    def last_state(self, side):
        d = np.zeros(self.n, dtype=np.uint32)
        s = np.zeros(self.n, dtype=np.uint64)
        self.lib().ebc_oracle_last_state(self.h, side, _ptr(d, _u32p), _ptr(s, _u64p))
        return d, s

    def last_meet_set(self):
        buf = np.zeros(self.n, dtype=np.uint32)
        k = self.lib().ebc_oracle_last_meet_set(self.h, _ptr(buf, _u32p), self.n)
        return buf[:k].copy()

    def accumulate(self, seed, first, count, tag=0, frame=None):
        if frame is None:
            frame = np.zeros(self.n + 1, dtype=np.uint64)
        self.lib().ebc_oracle_accumulate(self.h, seed, tag, first, count, _ptr(frame, _u64p))
        return frame

    def work(self, reset=False):
        w = np.zeros(len(WORK_NAMES), dtype=np.uint64)
        self.lib().ebc_oracle_work(self.h, _ptr(w, _u64p))
        if reset:
            self.lib().ebc_oracle_work_reset(self.h)
        return w

    def run_epochs(self, seed, epoch_samples, max_epochs, eps, omega, dl, du, bound=0, tag=0):
        S = np.zeros(self.n + 1, dtype=np.uint64)
        dl = _as(dl, np.float64)
        du = _as(du, np.float64)
        e = self.lib().ebc_oracle_run_epochs(self.h, seed, tag, epoch_samples, max_epochs, eps,
                                             omega, _ptr(dl, _f64p), _ptr(du, _f64p), bound,
                                             _ptr(S, _u64p))
        return int(e), S

    def bfs(self, source):
        d = np.zeros(self.n, dtype=np.uint32)
        q = np.zeros(self.n, dtype=np.uint32)
        out = np.zeros(3, dtype=np.uint64)
        self.lib().ebc_oracle_bfs(self.h, source, _ptr(d, _u32p), _ptr(q, _u32p), _ptr(out, _u64p))
        return d, int(out[0]), int(out[1]), int(out[2])

    def diameter(self, sweeps=4, seed=0):
        out = np.zeros(3, dtype=np.uint64)
        rc = self.lib().ebc_oracle_diameter(self.h, sweeps, seed, _ptr(out, _u64p))
        if rc != 0:
            raise ValueError("diameter_upper_bound: graph is disconnected")
        return int(out[0]), int(out[1]), int(out[2])

    def brandes(self, workers=None):
        """Exact normalised betweenness; source blocks run in worker threads (ctypes drops the GIL)."""
        import concurrent.futures as cf
        workers = workers or os.cpu_count() or 1
        workers = max(1, min(workers, self.n))
        parts = [np.zeros(self.n, dtype=np.float64) for _ in range(workers)]
        L = self.lib()

        def job(w):
            b, e = self.n * w // workers, self.n * (w + 1) // workers
            L.ebc_oracle_brandes_block(self.h, b, e, _ptr(parts[w], _f64p))

        with cf.ThreadPoolExecutor(workers) as ex:
            list(ex.map(job, range(workers)))
        tot = np.sum(parts, axis=0)
        L.ebc_oracle_brandes_finish(self.n, _ptr(tot, _f64p))
        return tot

    # ---- stateless helpers ----
    @classmethod
    def compute_omega(cls, vd, eps, delta):
        return int(cls.lib().ebc_oracle_compute_omega(vd, eps, delta))

    @classmethod
    def epoch_length(cls, ranks, threads, base=1000.0, exponent=1.33):
        return int(cls.lib().ebc_oracle_epoch_length(ranks, threads, base, exponent))

    @classmethod
    def calibrate(cls, calib_words, n, delta, kind=0):
        w = _as(calib_words, np.uint64)
        dl = np.zeros(n, dtype=np.float64)
        du = np.zeros(n, dtype=np.float64)
        cls.lib().ebc_oracle_calibrate(_ptr(w, _u64p), n, delta, kind, _ptr(dl, _f64p),
                                       _ptr(du, _f64p))
        return dl, du

    @classmethod
    def bound_width(cls, b, delta_v, tau, bound=0):
        return float(cls.lib().ebc_oracle_bound_width(b, delta_v, tau, bound))

    @classmethod
    def check_stop(cls, words, eps, omega, dl, du, bound=0):
        w = _as(words, np.uint64)
        dl = _as(dl, np.float64)
        du = _as(du, np.float64)
        return bool(cls.lib().ebc_oracle_check_stop(_ptr(w, _u64p), len(w) - 1, eps, omega,
                                                    _ptr(dl, _f64p), _ptr(du, _f64p), bound))

    @classmethod
    def mt_draws(cls, master, rank, thread, bounds):
        b = _as(bounds, np.uint64)
        out = np.zeros(len(b), dtype=np.uint64)
        cls.lib().ebc_oracle_mt_draws(master, rank, thread, _ptr(b, _u64p), len(b), _ptr(out, _u64p))
        return out

    @classmethod
    def philox_block(cls, ctr, key):
        c = _as(ctr, np.uint32)
        k = _as(key, np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        cls.lib().ebc_oracle_philox_block(_ptr(c, _u32p), _ptr(k, _u32p), _ptr(out, _u32p))
        return out

    @classmethod
    def stream_draws(cls, seed, tag, index, bounds):
        b = _as(bounds, np.uint64)
        out = np.zeros(len(b), dtype=np.uint64)
        cls.lib().ebc_oracle_stream_draws(seed, tag, index, _ptr(b, _u64p), len(b), _ptr(out, _u64p))
        return out


# --------------------------------------------------------------------------------------
class RefShim:
    """UNMODIFIED reference sampler.cpp/stopping.cpp/graph.cpp driven by the Philox shim."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(os.path.join(HERE, "_ref", "libebc_ref_shim.so"))
            L.refshim_last_error.restype = C.c_char_p
            L.refshim_graph_from_csr.restype = C.c_void_p
            L.refshim_graph_from_csr.argtypes = [C.c_uint64, _u64p, _u32p]
            L.refshim_graph_free.argtypes = [C.c_void_p]
            L.refshim_graph_n.restype = C.c_uint64
            L.refshim_graph_n.argtypes = [C.c_void_p]
            L.refshim_graph_m.restype = C.c_uint64
            L.refshim_graph_m.argtypes = [C.c_void_p]
            L.refshim_graph_csr.argtypes = [C.c_void_p, _u64p, _u64p]
            L.refshim_sample.restype = C.c_int64
            L.refshim_sample.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                         C.c_uint64, C.c_uint64, _u32p, C.c_uint64, _u64p]
            L.refshim_last_search_state.argtypes = [C.c_void_p, C.c_int, _u32p, _u64p]
            L.refshim_last_meet.restype = C.c_uint64
            L.refshim_last_meet.argtypes = [C.c_void_p, _u32p, C.c_uint64]
            L.refshim_accumulate.restype = C.c_int
            L.refshim_accumulate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                             C.c_uint64, _u64p]
            L.refshim_compute_omega.restype = C.c_uint64
            L.refshim_compute_omega.argtypes = [C.c_uint64, C.c_double, C.c_double]
            L.refshim_calibrate.restype = C.c_int
            L.refshim_calibrate.argtypes = [_u64p, C.c_uint64, C.c_double, C.c_int, _f64p, _f64p]
            L.refshim_check_stop.restype = C.c_int
            L.refshim_check_stop.argtypes = [_u64p, C.c_uint64, C.c_double, C.c_uint64, _f64p, _f64p,
                                             C.c_int]
            L.refshim_bound.restype = C.c_double
            L.refshim_bound.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int]
            cls._lib = L
        return cls._lib

    def __init__(self, offsets, targets):
        self.offsets = _as(offsets, np.uint64)
        self.targets = _as(targets, np.uint32)
        self.n = len(self.offsets) - 1
        L = self.lib()
        self.h = L.refshim_graph_from_csr(self.n, _ptr(self.offsets, _u64p),
                                          _ptr(self.targets, _u32p))
        if not self.h:
            raise RuntimeError(L.refshim_last_error().decode())
        self._path = np.zeros(max(self.n, 1), dtype=np.uint32)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib().refshim_graph_free(self.h)
                self.h = None
        except Exception:
            pass

    def csr(self):
        off = np.zeros(self.n + 1, dtype=np.uint64)
        m2 = int(self.lib().refshim_graph_m(self.h)) * 2
        tg = np.zeros(m2, dtype=np.uint64)
        self.lib().refshim_graph_csr(self.h, _ptr(off, _u64p), _ptr(tg, _u64p))
        return off, tg

    def sample(self, seed, index, tag=0, pair=None):
        info = np.zeros(3, dtype=np.uint64)
        s, t = (0, 0) if pair is None else pair
        L = self.lib()
        ln = L.refshim_sample(self.h, seed, tag, index, 0 if pair is None else 1, s, t,
                              _ptr(self._path, _u32p), len(self._path), _ptr(info, _u64p))
        if ln < 0:
            raise RuntimeError(L.refshim_last_error().decode())
        return dict(s=int(info[0]), t=int(info[1]), draws=int(info[2]), path=self._path[:ln].copy())

    def last_state(self, side):
        d = np.zeros(self.n, dtype=np.uint32)
        s = np.zeros(self.n, dtype=np.uint64)
        self.lib().refshim_last_search_state(self.h, side, _ptr(d, _u32p), _ptr(s, _u64p))
        return d, s

    def last_meet_set(self):
        buf = np.zeros(self.n, dtype=np.uint32)
        k = self.lib().refshim_last_meet(self.h, _ptr(buf, _u32p), self.n)
        return buf[:k].copy()

    def accumulate(self, seed, first, count, tag=0, frame=None):
        if frame is None:
            frame = np.zeros(self.n + 1, dtype=np.uint64)
        L = self.lib()
        if L.refshim_accumulate(self.h, seed, tag, first, count, _ptr(frame, _u64p)) != 0:
            raise RuntimeError(L.refshim_last_error().decode())
        return frame

    @classmethod
    def compute_omega(cls, vd, eps, delta):
        return int(cls.lib().refshim_compute_omega(vd, eps, delta))

    @classmethod
    def calibrate(cls, calib_words, n, delta, kind=0):
        w = _as(calib_words, np.uint64)
        dl = np.zeros(n, dtype=np.float64)
        du = np.zeros(n, dtype=np.float64)
        L = cls.lib()
        if L.refshim_calibrate(_ptr(w, _u64p), n, delta, kind, _ptr(dl, _f64p), _ptr(du, _f64p)):
            raise RuntimeError(L.refshim_last_error().decode())
        return dl, du

    @classmethod
    def check_stop(cls, words, eps, omega, dl, du, bound=0):
        w = _as(words, np.uint64)
        dl = _as(dl, np.float64)
        du = _as(du, np.float64)
        L = cls.lib()
        r = L.refshim_check_stop(_ptr(w, _u64p), len(w) - 1, eps, omega, _ptr(dl, _f64p),
                                 _ptr(du, _f64p), bound)
        if r < 0:
            raise RuntimeError(L.refshim_last_error().decode())
        return bool(r)

    @classmethod
    def bound(cls, b, delta_v, tau, bound=0):
        return float(cls.lib().refshim_bound(b, delta_v, tau, bound))


# --------------------------------------------------------------------------------------
class _RunArgs(C.Structure):
    _fields_ = [("eps", C.c_double), ("delta", C.c_double), ("seed", C.c_uint64),
                ("ranks", C.c_int), ("threads", C.c_int), ("algo", C.c_int), ("bound", C.c_int),
                ("allocator", C.c_int), ("real_clock", C.c_int), ("omega_override", C.c_uint64),
                ("calib_samples_per_worker", C.c_uint64), ("diameter_sweeps", C.c_int),
                ("sample_cost_ms", C.c_double)]


class _RunStats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("epochs", "samples", "tau", "omega", "calibration_samples",
                                          "discarded_samples", "n0", "diameter_upper_bound",
                                          "vertex_diameter_bound")] + \
               [(k, C.c_double) for k in ("adaptive_s", "diameter_s", "calibration_s", "transition_s",
                                          "reduce_s", "check_s", "wall_s", "wall_ms")]


class RefPlain:
    """UNMODIFIED reference library (mt19937_64): pipeline, Brandes, diameter, graph ingestion."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(os.path.join(HERE, "_ref", "libebc_ref_plain.so"))
            L.refplain_last_error.restype = C.c_char_p
            for f in ("refplain_graph_from_csr", "refplain_graph_from_edges", "refplain_graph_load",
                      "refplain_lcc"):
                getattr(L, f).restype = C.c_void_p
            L.refplain_graph_from_csr.argtypes = [C.c_uint64, _u64p, _u32p]
            L.refplain_graph_from_edges.argtypes = [C.c_uint64, _u64p, _u64p, C.c_uint64]
            L.refplain_graph_load.argtypes = [C.c_char_p]
            L.refplain_graph_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
            L.refplain_lcc.argtypes = [C.c_void_p]
            L.refplain_graph_free.argtypes = [C.c_void_p]
            L.refplain_graph_n.restype = C.c_uint64
            L.refplain_graph_n.argtypes = [C.c_void_p]
            L.refplain_graph_m.restype = C.c_uint64
            L.refplain_graph_m.argtypes = [C.c_void_p]
            L.refplain_graph_csr.argtypes = [C.c_void_p, _u64p, _u64p, _u64p]
            L.refplain_diameter.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _u64p]
            L.refplain_bfs.argtypes = [C.c_void_p, C.c_uint64, _u32p, _u64p]
            L.refplain_brandes.argtypes = [C.c_void_p, C.c_int, _f64p]
            L.refplain_compute_omega.restype = C.c_uint64
            L.refplain_compute_omega.argtypes = [C.c_uint64, C.c_double, C.c_double]
            L.refplain_epoch_length.restype = C.c_uint64
            L.refplain_epoch_length.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
            L.refplain_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p, C.c_uint64,
                                             _u64p]
            L.refplain_run.argtypes = [C.c_void_p, C.POINTER(_RunArgs), _f64p, C.POINTER(_RunStats)]
            L.refplain_write_scores.argtypes = [C.c_char_p, _u64p, _f64p, C.c_uint64, C.POINTER(C.c_char_p),
                                                C.POINTER(C.c_char_p), C.c_uint64]
            L.refplain_compare_files.argtypes = [C.c_char_p, C.c_char_p, C.c_double, _f64p, _u64p]
            cls._lib = L
        return cls._lib

    def __init__(self, handle):
        self.h = handle
        if not self.h:
            raise RuntimeError(self.lib().refplain_last_error().decode())
        self.n = int(self.lib().refplain_graph_n(self.h))
        self.m = int(self.lib().refplain_graph_m(self.h))

    @classmethod
    def from_csr(cls, offsets, targets):
        o = _as(offsets, np.uint64)
        t = _as(targets, np.uint32)
        return cls(cls.lib().refplain_graph_from_csr(len(o) - 1, _ptr(o, _u64p), _ptr(t, _u32p)))

    @classmethod
    def from_edges(cls, n, src, dst):
        s = _as(src, np.uint64)
        d = _as(dst, np.uint64)
        return cls(cls.lib().refplain_graph_from_edges(n, _ptr(s, _u64p), _ptr(d, _u64p), len(s)))

    @classmethod
    def load(cls, path):
        return cls(cls.lib().refplain_graph_load(path.encode()))

    def save(self, path, binary=False):
        if self.lib().refplain_graph_save(self.h, path.encode(), int(binary)) != 0:
            raise RuntimeError(self.lib().refplain_last_error().decode())

    def lcc(self):
        return RefPlain(self.lib().refplain_lcc(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib().refplain_graph_free(self.h)
                self.h = None
        except Exception:
            pass

    def csr(self):
        off = np.zeros(self.n + 1, dtype=np.uint64)
        tg = np.zeros(2 * self.m, dtype=np.uint64)
        ids = np.zeros(self.n, dtype=np.uint64)
        self.lib().refplain_graph_csr(self.h, _ptr(off, _u64p), _ptr(tg, _u64p), _ptr(ids, _u64p))
        return off, tg, ids

    def diameter(self, sweeps=4, seed=0):
        out = np.zeros(3, dtype=np.uint64)
        if self.lib().refplain_diameter(self.h, sweeps, seed, _ptr(out, _u64p)) != 0:
            raise ValueError(self.lib().refplain_last_error().decode())
        return int(out[0]), int(out[1]), int(out[2])

    def bfs(self, source):
        d = np.zeros(self.n, dtype=np.uint32)
        out = np.zeros(3, dtype=np.uint64)
        if self.lib().refplain_bfs(self.h, source, _ptr(d, _u32p), _ptr(out, _u64p)) != 0:
            raise ValueError(self.lib().refplain_last_error().decode())
        return d, int(out[0]), int(out[1]), int(out[2])

    def brandes(self, workers=0):
        s = np.zeros(self.n, dtype=np.float64)
        if self.lib().refplain_brandes(self.h, workers, _ptr(s, _f64p)) != 0:
            raise RuntimeError(self.lib().refplain_last_error().decode())
        return s

    def run(self, eps, delta, seed, threads=1, ranks=1, algo=2, bound=0, allocator=0,
            real_clock=True, omega_override=0, calib_samples_per_worker=0, diameter_sweeps=0,
            sample_cost_ms=0.0):
        """run_simulated (engine.cpp:405-434) -> (scores, stats dict)."""
        a = _RunArgs(eps, delta, seed, ranks, threads, algo, bound, allocator, int(real_clock),
                     omega_override, calib_samples_per_worker, diameter_sweeps, sample_cost_ms)
        st = _RunStats()
        scores = np.zeros(self.n, dtype=np.float64)
        if self.lib().refplain_run(self.h, C.byref(a), _ptr(scores, _f64p), C.byref(st)) != 0:
            raise RuntimeError(self.lib().refplain_last_error().decode())
        return scores, {k: getattr(st, k) for k, _ in _RunStats._fields_}

    @classmethod
    def compute_omega(cls, vd, eps, delta):
        return int(cls.lib().refplain_compute_omega(vd, eps, delta))

    @classmethod
    def epoch_length(cls, ranks, threads, base=1000.0, exponent=1.33):
        return int(cls.lib().refplain_epoch_length(ranks, threads, base, exponent))

    @classmethod
    def write_scores(cls, path, ids, scores, meta=None):
        ids = _as(ids, np.uint64)
        scores = _as(scores, np.float64)
        meta = meta or {}
        keys = (C.c_char_p * max(len(meta), 1))(*[str(k).encode() for k in meta])
        vals = (C.c_char_p * max(len(meta), 1))(*[str(v).encode() for v in meta.values()])
        if cls.lib().refplain_write_scores(path.encode(), _ptr(ids, _u64p), _ptr(scores, _f64p), len(ids), keys, vals,
                                           len(meta)) != 0:
            raise RuntimeError(cls.lib().refplain_last_error().decode())

    @classmethod
    def compare_files(cls, approx, exact, eps):
        out = np.zeros(3, dtype=np.float64)
        cnt = np.zeros(2, dtype=np.uint64)
        if cls.lib().refplain_compare_files(approx.encode(), exact.encode(), eps, _ptr(out, _f64p), _ptr(cnt, _u64p)) != 0:
            raise ValueError(cls.lib().refplain_last_error().decode())
        return dict(max_abs_error=float(out[0]), top10_overlap=float(out[1]), top100_overlap=float(out[2]),
                    vertices_above_eps=int(cnt[0]), vertices=int(cnt[1]))

    @classmethod
    def rng_draws(cls, master, rank, thread, bounds):
        b = _as(bounds, np.uint64)
        out = np.zeros(len(b), dtype=np.uint64)
        cls.lib().refplain_rng_draws(master, rank, thread, _ptr(b, _u64p), len(b), _ptr(out, _u64p))
        return out
