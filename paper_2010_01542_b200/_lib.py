"""ctypes binding of libpgx.so (include/pgx.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing, unloadable or no CUDA device is present, every run
raises -- the product path is the CUDA kernel or nothing.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, ExecutionError

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGX_LIB") or os.path.join(PKG_DIR, "libpgx.so")

PGX_ABI_VERSION = 6
PGX_OK, PGX_EINVAL, PGX_ECUDA, PGX_ENOMEM = 0, -1, -2, -3
PGX_APP_PAGERANK, PGX_APP_CC, PGX_APP_SSSP, PGX_APP_PAGERANK_PULL = 0, 1, 2, 3
PGX_OP_MIN_U32, PGX_OP_SUM_F64 = 0, 1
PGX_STAT_HDR, PGX_STAT_FIELDS = 4, 8
PGX_OPT_READ_FILTER, PGX_OPT_CTAS_PER_SM, PGX_OPT_CAS_LOOP, PGX_OPT_VERTEX_SCHED = 0, 1, 2, 3
PGX_OPT_LAYOUT = 4
PGX_OPT_SEG_MIN_EDGES = 5
PGX_OPT_SEG_PREDICT = 6
PGX_OPT_PULL_MIN_EDGES = 7
PGX_SEG_LOG2_DEFAULT = 14
PGX_IPC_HANDLE_BYTES = 64
PGX_LAYOUT_EXTERNALISED, PGX_LAYOUT_INTERLEAVED = 0, 1


def set_option(key: int, value: int) -> None:
    """Process-wide tuning knob of libpgx.so (A/B experiments)."""
    check(load().pgx_set_option(key, value), "pgx_set_option")

#: every symbol include/pgx.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "pgx_abi_version", "pgx_last_error", "pgx_set_option", "pgx_device_sm_count",
    "pgx_offsets_to_i32", "pgx_graph_workspace_bytes", "pgx_graph_prepare",
    "pgx_run_workspace_bytes", "pgx_hub_capacity", "pgx_sssp_run", "pgx_cc_run",
    "pgx_pagerank_run", "pgx_pagerank_pull_run", "pgx_pr_hub_capacity",
    "pgx_pagerank_pull_hubs_run", "pgx_cc_prescatter_init", "pgx_cc_source_scatter",
    "pgx_cc_run_prescattered", "pgx_rmat_keys", "pgx_microbench",
    "pgx_slice_init", "pgx_scatter", "pgx_slice_counters_bytes", "pgx_apply_slice",
    "pgx_pr_apply_slice", "pgx_touched_scratch_bytes", "pgx_touched", "pgx_scatter_pairs",
    "pgx_scatter_peer", "pgx_reset_touched", "pgx_peer_alloc", "pgx_peer_open",
    "pgx_peer_close", "pgx_peer_free", "pgx_seg_workspace_bytes", "pgx_seg_max_items",
    "pgx_seg_count", "pgx_seg_build", "pgx_sssp_run_ex", "pgx_cc_run_ex",
    "pgx_gather_slice", "pgx_fold_spanning", "pgx_peer_enable", "pgx_seg_scatter",
    "pgx_seg_count_ex", "pgx_seg_build_ex", "pgx_scatter_peer_bfs", "pgx_apply_slice_bfs",
    "pgx_sssp_run_dir",
)


class PgxSegIndex(ctypes.Structure):
    """include/pgx.h PgxSegIndex: the destination-segmented index."""

    _fields_ = [("seg_log2", ctypes.c_int32), ("nent", ctypes.c_int32),
                ("nitems", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("ent_src", ctypes.c_void_p), ("ent_eb", ctypes.c_void_p),
                ("col16", ctypes.c_void_p), ("tile_ent", ctypes.c_void_p),
                ("items", ctypes.c_void_p)]

_lib = None

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_up = ctypes.c_size_t  # uintptr_t stream

_SIGS = {
    "pgx_abi_version": (ctypes.c_int, []),
    "pgx_last_error": (ctypes.c_char_p, []),
    "pgx_set_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "pgx_device_sm_count": (ctypes.c_int, [ctypes.c_int, _p]),
    "pgx_offsets_to_i32": (ctypes.c_int, [_p, _p, _i64, _up]),
    "pgx_graph_workspace_bytes": (ctypes.c_int, [_i64, _i64, _p]),
    "pgx_graph_prepare": (ctypes.c_int, [_i32, _i64, _p, _p, _sz, _up]),
    "pgx_run_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i32, _p]),
    "pgx_hub_capacity": (ctypes.c_int, [_p]),
    "pgx_sssp_run": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _sz,
                                    _p, _up]),
    "pgx_cc_run": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _i32, _i32, _p, _p, _sz, _p,
                                  _up]),
    "pgx_pagerank_run": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _i32, _f64, _f64, _f64,
                                        _i32, _p, _p, _sz, _p, _up]),
    "pgx_pagerank_pull_run": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _i32, _f64, _f64,
                                             _f64, _i32, _p, _p, _sz, _p, _up]),
    "pgx_pr_hub_capacity": (ctypes.c_int, [_p]),
    "pgx_cc_prescatter_init": (ctypes.c_int, [_i32, _i64, _i32, _p, _sz, _up]),
    "pgx_cc_source_scatter": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _i64, _i64, _i32, _p, _sz,
                                             _up]),
    "pgx_cc_run_prescattered": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _i32, _p, _p, _sz, _p,
                                               _up]),
    "pgx_pagerank_pull_hubs_run": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _p, _i32, _i32,
                                                  _f64, _f64, _f64, _i32, _p, _p, _sz, _p, _up]),
    "pgx_slice_init": (ctypes.c_int, [ctypes.c_int, _i32, _i32, _p, _p, _p, _f64, _up]),
    "pgx_scatter": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _p, _p, _p, _p, _i32, _p, _p,
                                   _i32, _i64, _p, _p, ctypes.c_uint32, _up]),
    "pgx_touched_scratch_bytes": (ctypes.c_int, [_i32, _p]),
    "pgx_touched": (ctypes.c_int, [_i32, _i32, _i32, _p, _p, ctypes.c_uint32, _p, _p, _p, _up]),
    "pgx_scatter_pairs": (ctypes.c_int, [_p, _i64, _p, _up]),
    "pgx_scatter_peer": (ctypes.c_int, [ctypes.c_int, _p, _p, _p, _p, _i32, _p, _p, _i32, _i64,
                                        _p, _p, ctypes.c_uint32, _p, _p, _i32, _i32, _i32, _up]),
    "pgx_reset_touched": (ctypes.c_int, [_i32, _i32, _i32, _p, _p, ctypes.c_uint32, _up]),
    "pgx_scatter_peer_bfs": (ctypes.c_int, [_p, _p, _p, _p, _p, _i32, _i64, _p, _p, _p, _i32,
                                            _i32, _i32, _up]),
    "pgx_apply_slice_bfs": (ctypes.c_int, [_i32, _p, _p, _p, _p, _p, _p, _p, _p, _i32,
                                           ctypes.c_uint32, _up]),
    "pgx_peer_alloc": (ctypes.c_int, [_sz, _p, _p]),
    "pgx_peer_open": (ctypes.c_int, [_p, _p]),
    "pgx_peer_close": (ctypes.c_int, [_p]),
    "pgx_peer_free": (ctypes.c_int, [_p]),
    "pgx_slice_counters_bytes": (ctypes.c_int, [_p]),
    "pgx_apply_slice": (ctypes.c_int, [ctypes.c_int, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
                                       _i32, ctypes.c_uint32, _p, _up]),
    "pgx_seg_scatter": (ctypes.c_int, [ctypes.c_int, _p, _i64, _i32, _i32, _p, _p, _p,
                                       ctypes.c_uint32, _p, _up]),
    "pgx_seg_count_ex": (ctypes.c_int, [_i32, _i32, _i64, _p, _p, _p, _i32, _p, _sz, _p, _up]),
    "pgx_seg_build_ex": (ctypes.c_int, [_i32, _i32, _i64, _p, _p, _p, _i32, _i64, _p, _sz, _p,
                                        _p, _p, _p, _p, _p, _i32, _up]),
    "pgx_pr_apply_slice": (ctypes.c_int, [_i32, _p, _p, _p, _p, _f64, _f64, _p, _f64, _i32,
                                          _p, _up]),
    "pgx_gather_slice": (ctypes.c_int, [_i32, _i64, _p, _p, _i32, _p, _p, _p, _p, _up]),
    "pgx_fold_spanning": (ctypes.c_int, [_i32, _p, _p, _p, _p, _p, _p, _up]),
    "pgx_peer_enable": (ctypes.c_int, [_i32]),
    "pgx_microbench": (ctypes.c_int, [ctypes.c_int, _p, _i64, _i64, _u64, _p, _up]),
    "pgx_seg_workspace_bytes": (ctypes.c_int, [_i32, _i64, _i64, _i32, _p]),
    "pgx_seg_max_items": (ctypes.c_int, [_i32, _i64, _i32, _p]),
    "pgx_seg_count": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _i32, _p, _sz, _p, _up]),
    "pgx_seg_build": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _i32, _i64, _p, _sz, _p, _p, _p,
                                     _p, _p, _p, _i32, _up]),
    "pgx_sssp_run_ex": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _i32, _i32, _p, _p, _sz, _p,
                                       _up]),
    "pgx_sssp_run_dir": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _p, _p, _i32, _i32, _p, _p,
                                        _sz, _p, _up]),
    "pgx_cc_run_ex": (ctypes.c_int, [_i32, _i64, _p, _p, _p, _p, _i32, _p, _p, _sz, _p, _up]),
    "pgx_rmat_keys": (ctypes.c_int, [_i32, _i64, _i64, _f64, _f64, _f64, _u64, _i32,
                                     _i64, _i64, _p, _i64, _p, _up]),
}


def load():
    """Load libpgx.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExecutionError(
            f"{LIB_PATH} is missing: build it with "
            f"`python -c 'import __graft_entry__ as g; g.build()'` "
            f"(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pgx_abi_version() != PGX_ABI_VERSION:
        raise ExecutionError("libpgx.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a PGX status code onto the reference exception taxonomy."""
    if rc == PGX_OK:
        return
    msg = (_lib.pgx_last_error() or b"").decode(errors="replace") if _lib else ""
    if rc == PGX_EINVAL:
        raise ConfigError(f"{what}: {msg}")
    raise ExecutionError(f"{what} failed ({rc}): {msg}")


def out_size(fn, *args) -> int:
    v = ctypes.c_size_t(0)
    check(fn(*args, ctypes.byref(v)), fn.__name__)
    return int(v.value)
