"""The C ABI library loads and exports every symbol include/pgx.h declares
(no compute calls: CPU container), and the product path refuses to run
without a CUDA device (no CPU fallback)."""

import ctypes
import os
import re
import subprocess

import pytest

import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgx.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pgx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_exactly_the_bound_symbols():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (pgx_\w+)", out))
    for sym in declared_symbols():
        assert sym in exported, sym
        assert getattr(lib, sym) is not None
    assert lib.pgx_abi_version() == _lib.PGX_ABI_VERSION


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_size_queries_and_error_codes():
    lib = _lib.load()
    v = ctypes.c_size_t(0)
    assert lib.pgx_graph_workspace_bytes(1 << 22, 65_000_000, ctypes.byref(v)) == 0
    assert v.value > (1 << 22) * 8
    for app in (0, 1, 2):
        assert lib.pgx_run_workspace_bytes(app, 1000, 5000, 16, ctypes.byref(v)) == 0
        assert v.value > 1000 * 4
    assert lib.pgx_run_workspace_bytes(7, 10, 10, 1, ctypes.byref(v)) == _lib.PGX_EINVAL
    assert b"bad run workspace" in lib.pgx_last_error()
    with pytest.raises(pgx.ConfigError):
        _lib.check(_lib.PGX_EINVAL, "probe")
    with pytest.raises(pgx.ExecutionError):
        _lib.check(_lib.PGX_ECUDA, "probe")


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback():
    g = pgx.from_edges([0, 1], [1, 2], 3)
    for prog in (pgx.pagerank(), pgx.connected_components(), pgx.sssp(0)):
        with pytest.raises(pgx.ExecutionError):
            pgx.run(g, prog)


def test_header_constants_match_the_binding():
    defines = dict(re.findall(r"#define (PGX_[A-Z0-9_]+) (-?\d+)", open(HEADER).read()))
    bound = {k: getattr(_lib, k) for k in defines if hasattr(_lib, k)}
    assert {"PGX_OPT_LAYOUT", "PGX_LAYOUT_INTERLEAVED", "PGX_OPT_READ_FILTER"} <= set(bound)
    for k, v in bound.items():
        assert int(defines[k]) == v, k


def test_interleaved_layout_sizes_the_record_array():
    lib = _lib.load()
    soa, aos = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.pgx_run_workspace_bytes(1, 1 << 20, 1 << 24, 16, ctypes.byref(soa)) == 0
    _lib.set_option(_lib.PGX_OPT_LAYOUT, _lib.PGX_LAYOUT_INTERLEAVED)
    try:
        assert lib.pgx_run_workspace_bytes(1, 1 << 20, 1 << 24, 16, ctypes.byref(aos)) == 0
    finally:
        _lib.set_option(_lib.PGX_OPT_LAYOUT, _lib.PGX_LAYOUT_EXTERNALISED)
    assert aos.value - soa.value >= 4 * (1 << 20)


def test_pull_pagerank_rejects_a_misaligned_in_col():
    """The fold loads neighbour ids 32 bytes at a time: a misaligned in_col
    is refused with PGX_EINVAL before anything touches the device."""
    lib = _lib.load()
    fake = 1 << 20  # never dereferenced: the argument checks come first
    rc = lib.pgx_pagerank_pull_run(10, 20, fake, fake, fake + 4, fake, 10, 0.85, 0.015, 0.1,
                                   10, fake, fake, 1 << 20, fake, 0)
    assert rc == _lib.PGX_EINVAL
    assert b"32-byte aligned" in lib.pgx_last_error()


def test_direction_optimising_sssp_rejects_a_bad_in_csr():
    """pgx_sssp_run_dir checks its in-CSR before anything touches the
    device: a null in_row_ptr (or in_col with edges) and a misaligned
    in_col (256-bit sector loads) are PGX_EINVAL."""
    lib = _lib.load()
    fake = 1 << 20  # never dereferenced: the argument checks come first
    args = lambda irp, ic: (10, 20, fake, fake, fake, None, irp, ic, 0, 10, fake, fake, 1 << 20,
                            fake, 0)
    assert lib.pgx_sssp_run_dir(*args(None, fake)) == _lib.PGX_EINVAL
    assert b"in-CSR" in lib.pgx_last_error()
    assert lib.pgx_sssp_run_dir(*args(fake, None)) == _lib.PGX_EINVAL
    assert lib.pgx_sssp_run_dir(*args(fake, fake + 4)) == _lib.PGX_EINVAL
    assert b"32-byte aligned" in lib.pgx_last_error()


def test_integration_doc_covers_every_entry_point():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    assert [s for s in _lib.EXPORTS if s not in doc] == []
