"""ctypes front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker
or the timed CPU baseline.  The product package (paper_2010_01542_b200)
never imports it.

Every function restates a reference function; see the header of
``pregel_oracle.c`` for the file:line map.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_np_sum.restype = ctypes.c_double
        L.orc_np_sum.argtypes = [_p, _i64]
        L.orc_np_reduceat_segment.restype = ctypes.c_double
        L.orc_np_reduceat_segment.argtypes = [_p, _i64]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_rmat_keys.restype = _i64
        L.orc_rmat_keys.argtypes = [ctypes.c_int, _i64, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double,
                                    ctypes.c_uint64, ctypes.c_int, _p,
                                    ctypes.c_int]
        L.orc_keys_to_csr.restype = None
        L.orc_keys_to_csr.argtypes = [_p, _i64, _i64, _p, _p]
        L.orc_transpose.restype = None
        L.orc_transpose.argtypes = [_i64, _p, _p, _p, _p]
        L.orc_run_sssp.restype = ctypes.c_int
        L.orc_run_sssp.argtypes = [_i64, _p, _p, _i64, _i64, ctypes.c_int,
                                   _p, _p, _p]
        L.orc_run_cc.restype = ctypes.c_int
        L.orc_run_cc.argtypes = [_i64, _p, _p, _p, _p, _i64, ctypes.c_int,
                                 _p, _p, _p]
        L.orc_run_pagerank.restype = ctypes.c_int
        L.orc_run_pagerank.argtypes = [_i64, _p, _p, _p, _p, _i64,
                                       ctypes.c_double, _i64, ctypes.c_int,
                                       _p, _p, _p]
        L.orc_components_ref.restype = None
        L.orc_components_ref.argtypes = [_i64, _i64, _p, _p, _p]
        L.orc_bfs_ref.restype = ctypes.c_int
        L.orc_bfs_ref.argtypes = [_i64, _i64, _p, _p, _i64, _p]
        L.orc_pagerank_ref.restype = None
        L.orc_pagerank_ref.argtypes = [_i64, _i64, _p, _p, _i64,
                                       ctypes.c_double, _p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ----------------------------------------------------------------------
# numpy rounding orders
# ----------------------------------------------------------------------

def np_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_np_sum(_ptr(a), a.size))


def np_reduceat_segment(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_np_reduceat_segment(_ptr(a), a.size))


# ----------------------------------------------------------------------
# inputs
# ----------------------------------------------------------------------

@dataclass(frozen=True)
class RmatSpec:
    """One R-MAT input of SURVEY.md 8(d) / BASELINE.json configs."""

    scale: int
    edge_factor: int
    a: float
    b: float
    c: float
    seed: int
    symmetric: bool

    @property
    def n(self) -> int:
        return 1 << self.scale


#: BASELINE.json configs C1..C5
CONFIGS = {
    "C1": RmatSpec(16, 16, 0.57, 0.19, 0.19, 1, False),
    "C2": RmatSpec(22, 8, 0.57, 0.19, 0.19, 2, True),
    "C3": RmatSpec(22, 16, 0.57, 0.19, 0.19, 3, False),
    "C4": RmatSpec(22, 28, 0.45, 0.22, 0.22, 4, False),
    "C5": RmatSpec(26, 14, 0.57, 0.19, 0.19, 5, True),
    # test-only: C5's shape at scale 16 (bench.py functional multi-rank runs)
    "C5S": RmatSpec(16, 14, 0.57, 0.19, 0.19, 5, True),
}


def rmat_csr(spec: RmatSpec, threads: int = 0):
    """(n, out_offsets int64[n+1], out_targets int32[m]) of an R-MAT spec."""
    n = spec.n
    cap = spec.edge_factor * n * (2 if spec.symmetric else 1)
    keys = np.empty(max(cap, 1), dtype=np.uint64)
    m = int(lib().orc_rmat_keys(spec.scale, spec.edge_factor, spec.a, spec.b,
                                spec.c, spec.seed, int(spec.symmetric),
                                _ptr(keys), threads))
    off = np.empty(n + 1, dtype=np.int64)
    tgt = np.empty(max(m, 1), dtype=np.int32)
    lib().orc_keys_to_csr(_ptr(keys), m, n, _ptr(off), _ptr(tgt))
    del keys
    return n, off, tgt[:m].copy()


def csr_from_edges(src, dst, n: int, undirected: bool = False):
    """graph.py:141-187 semantics: duplicates/self-loops kept, rows sorted."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if undirected and src.size:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    order = np.lexsort((dst, src))
    off = np.zeros(n + 1, dtype=np.int64)
    if src.size:
        np.cumsum(np.bincount(src, minlength=n), out=off[1:])
    return off, dst[order].astype(np.int32)


def transpose(n: int, off, tgt):
    off = np.ascontiguousarray(off, dtype=np.int64)
    tgt = np.ascontiguousarray(tgt, dtype=np.int32)
    in_off = np.empty(n + 1, dtype=np.int64)
    in_tgt = np.empty(max(tgt.size, 1), dtype=np.int32)
    lib().orc_transpose(n, _ptr(off), _ptr(tgt), _ptr(in_off), _ptr(in_tgt))
    return in_off, in_tgt[:tgt.size].copy()


def stored_edges(n: int, off, tgt):
    """CSR back to the stored directed edge arrays (harness.py:233-237)."""
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    return src, np.asarray(tgt, dtype=np.int64)


# ----------------------------------------------------------------------
# engine restatement
# ----------------------------------------------------------------------

@dataclass
class OracleRun:
    values: np.ndarray
    superstep_count: int
    hit_superstep_cap: bool
    active_counts: list
    messages_sent: list
    edges: list


def _finish(values, stats, hdr) -> OracleRun:
    k = int(hdr[0])
    st = stats[:3 * k].reshape(k, 3) if k else np.zeros((0, 3), np.int64)
    return OracleRun(values, k, bool(hdr[1]), st[:, 0].tolist(),
                     st[:, 1].tolist(), st[:, 2].tolist())


def run_sssp(n, off, tgt, source, max_steps=10_000, threads=0) -> OracleRun:
    off = np.ascontiguousarray(off, np.int64)
    tgt = np.ascontiguousarray(tgt, np.int32)
    dist = np.empty(n, np.uint32)
    stats = np.zeros(3 * max_steps, np.int64)
    hdr = np.zeros(2, np.int64)
    rc = lib().orc_run_sssp(n, _ptr(off), _ptr(tgt) if tgt.size else None,
                            source, max_steps, threads, _ptr(dist),
                            _ptr(stats), _ptr(hdr))
    if rc != 0:
        raise ValueError(f"orc_run_sssp failed ({rc})")
    return _finish(dist, stats, hdr)


def run_cc(n, off, tgt, in_off=None, in_tgt=None, max_steps=10_000,
           threads=0) -> OracleRun:
    off = np.ascontiguousarray(off, np.int64)
    tgt = np.ascontiguousarray(tgt, np.int32)
    if in_off is None:
        in_off, in_tgt = transpose(n, off, tgt)
    in_off = np.ascontiguousarray(in_off, np.int64)
    in_tgt = np.ascontiguousarray(in_tgt, np.int32)
    labels = np.empty(max(n, 1), np.int64)
    stats = np.zeros(3 * max_steps, np.int64)
    hdr = np.zeros(2, np.int64)
    rc = lib().orc_run_cc(n, _ptr(off), _ptr(tgt) if tgt.size else None,
                          _ptr(in_off), _ptr(in_tgt) if in_tgt.size else None,
                          max_steps, threads, _ptr(labels), _ptr(stats),
                          _ptr(hdr))
    if rc != 0:
        raise ValueError(f"orc_run_cc failed ({rc})")
    return _finish(labels[:n], stats, hdr)


def run_pagerank(n, off, tgt, iterations=10, damping=0.85, in_off=None,
                 in_tgt=None, max_steps=10_000, threads=0) -> OracleRun:
    off = np.ascontiguousarray(off, np.int64)
    tgt = np.ascontiguousarray(tgt, np.int32)
    if in_off is None:
        in_off, in_tgt = transpose(n, off, tgt)
    in_off = np.ascontiguousarray(in_off, np.int64)
    in_tgt = np.ascontiguousarray(in_tgt, np.int32)
    rank = np.empty(max(n, 1), np.float64)
    stats = np.zeros(3 * max_steps, np.int64)
    hdr = np.zeros(2, np.int64)
    rc = lib().orc_run_pagerank(n, _ptr(off), _ptr(tgt) if tgt.size else None,
                                _ptr(in_off),
                                _ptr(in_tgt) if in_tgt.size else None,
                                iterations, damping, max_steps, threads,
                                _ptr(rank), _ptr(stats), _ptr(hdr))
    if rc != 0:
        raise ValueError(f"orc_run_pagerank failed ({rc})")
    return _finish(rank[:n], stats, hdr)


# ----------------------------------------------------------------------
# independent validators (oracles.py)
# ----------------------------------------------------------------------

def components_reference(src, dst, n):
    src = np.ascontiguousarray(src, np.int64)
    dst = np.ascontiguousarray(dst, np.int64)
    out = np.empty(max(n, 1), np.int64)
    lib().orc_components_ref(n, src.size, _ptr(src), _ptr(dst), _ptr(out))
    return out[:n]


def bfs_distances_reference(src, dst, n, source):
    src = np.ascontiguousarray(src, np.int64)
    dst = np.ascontiguousarray(dst, np.int64)
    out = np.empty(max(n, 1), np.uint32)
    if lib().orc_bfs_ref(n, src.size, _ptr(src), _ptr(dst), source,
                         _ptr(out)) != 0:
        raise IndexError(f"source {source} out of range [0, {n})")
    return out[:n]


def pagerank_reference(src, dst, n, iterations=10, damping=0.85):
    src = np.ascontiguousarray(src, np.int64)
    dst = np.ascontiguousarray(dst, np.int64)
    out = np.empty(max(n, 1), np.float64)
    lib().orc_pagerank_ref(n, src.size, _ptr(src), _ptr(dst), iterations,
                           damping, _ptr(out))
    return out[:n]
