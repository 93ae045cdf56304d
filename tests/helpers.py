"""Test-only helpers: small numpy graph builders (independent of the product's ingestion code)."""
from __future__ import annotations

import numpy as np


def csr_from_edges(n, src, dst):
    """Symmetrise, drop loops/duplicates, sort rows ascending -> (offsets u64[n+1], targets u32[2m])."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    a = np.concatenate([src, dst])
    b = np.concatenate([dst, src])
    key = np.unique(a * n + b)
    a, b = key // n, key % n
    offsets = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(offsets, a + 1, 1)
    offsets = np.cumsum(offsets).astype(np.uint64)
    return offsets, b.astype(np.uint32)


def random_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    return csr_from_edges(n, rng.integers(0, n, m), rng.integers(0, n, m))


def grid_graph(w, h, drop=0.0, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.arange(w * h).reshape(h, w)
    e = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                        np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
    if drop > 0:
        e = e[rng.random(len(e)) >= drop]
    return csr_from_edges(w * h, e[:, 0], e[:, 1])


def path_graph(n):
    return csr_from_edges(n, np.arange(n - 1), np.arange(1, n))


def cycle_graph(n):
    return csr_from_edges(n, np.arange(n), (np.arange(n) + 1) % n)


def star_graph(n):
    return csr_from_edges(n, np.zeros(n - 1, dtype=np.int64), np.arange(1, n))


def complete_bipartite_chain(widths):
    """Layered graph: consecutive layers fully connected -> sigma grows as a product of widths."""
    starts = np.concatenate([[0], np.cumsum(widths)])
    src, dst = [], []
    for i in range(len(widths) - 1):
        a = np.arange(starts[i], starts[i + 1])
        b = np.arange(starts[i + 1], starts[i + 2])
        aa, bb = np.meshgrid(a, b, indexing="ij")
        src.append(aa.ravel())
        dst.append(bb.ravel())
    return csr_from_edges(int(starts[-1]), np.concatenate(src), np.concatenate(dst))


def largest_component(offsets, targets):
    """numpy/scipy LCC (ties -> component with the smallest vertex id), order-preserving remap."""
    import scipy.sparse as sp
    import scipy.sparse.csgraph as csg
    n = len(offsets) - 1
    A = sp.csr_matrix((np.ones(len(targets), dtype=np.int8), targets.astype(np.int64),
                       offsets.astype(np.int64)), shape=(n, n))
    nc, lab = csg.connected_components(A, directed=False)
    sizes = np.bincount(lab, minlength=nc)
    first = np.full(nc, n, dtype=np.int64)
    np.minimum.at(first, lab, np.arange(n))
    best = max(range(nc), key=lambda c: (sizes[c], -first[c]))
    keep = np.nonzero(lab == best)[0]
    remap = np.full(n, -1, dtype=np.int64)
    remap[keep] = np.arange(len(keep))
    rows = np.repeat(np.arange(n), np.diff(offsets.astype(np.int64)))
    mask = (lab[rows] == best)
    return csr_from_edges(len(keep), remap[rows[mask]], remap[targets[mask].astype(np.int64)]), keep


def oracle_frame(offsets, targets, seed, first, count, workers=None, tag=0):
    """Frame (u64[n+1]) of sample indices [first, first+count) from the CPU oracle, the index range split
    over worker threads (each with its own Oracle state; ctypes drops the GIL; frames are sums)."""
    import concurrent.futures as cf
    import os
    from oracle import Oracle
    workers = max(1, min(workers or os.cpu_count() or 1, 32, count // 64 or 1))
    cuts = [first + count * w // workers for w in range(workers + 1)]

    def job(w):
        o = Oracle(offsets, targets)
        return o.accumulate(seed, cuts[w], cuts[w + 1] - cuts[w], tag=tag)

    with cf.ThreadPoolExecutor(workers) as ex:
        parts = list(ex.map(job, range(workers)))
    return np.sum(parts, axis=0, dtype=np.uint64)
