"""Host-side mirror of the pregelite API (CPU): graph construction
semantics, cache format, partition rule, program validation, lowering."""

import os

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from oracle import oracle as O


def test_from_edges_keeps_duplicates_and_sorts_rows():
    # reference tests/test_graph.py:23-42
    g = pgx.from_edges([0, 0, 0, 2], [2, 1, 2, 0], 3)
    assert g.out_offsets.tolist() == [0, 3, 3, 4]
    assert g.out_targets.tolist() == [1, 2, 2, 0]
    assert g.out_targets.dtype == torch.int32
    u = pgx.from_edges([0, 1], [1, 1], 2, undirected=True)
    assert u.edge_count == 4
    assert u.out_neighbors(1).tolist() == [0, 1, 1]


@pytest.mark.parametrize("seed", range(4))
def test_from_edges_matches_reference_csr(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 200))
    m = int(rng.integers(0, 4 * n))
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    for und in (False, True):
        g = pgx.from_edges(src, dst, n, undirected=und)
        off, tgt = O.csr_from_edges(src, dst, n, und)
        assert np.array_equal(g.out_offsets.numpy(), off)
        assert np.array_equal(g.out_targets.numpy(), tgt)
        ioff, itgt = O.transpose(n, off, tgt)
        assert np.array_equal(g.in_offsets.numpy(), ioff)
        assert np.array_equal(g.in_targets.numpy(), itgt)


def test_from_edges_validation():
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_edges([0, 5], [1, 1], 3)
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_edges([0, -1], [1, 1], 3)
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_edges([0], [1, 2], 3)
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_edges([0], [1], -1)
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_edges([0], [1], 2, id_dtype=np.float32)


def test_cache_round_trip_and_corruption(tmp_path):
    g = pgx.from_edges([0, 1, 2, 2], [1, 2, 0, 0], 3, undirected=True)
    p = tmp_path / "g.bin"
    pgx.save_cache(g, p)
    h = pgx.load_cache(p)
    assert h.vertex_count == 3
    assert h.out_targets.tolist() == g.out_targets.tolist()
    assert h.in_offsets.tolist() == g.in_offsets.tolist()
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(pgx.GraphLoadError):
        pgx.load_cache(p)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"nonsense" * 8)
    with pytest.raises(pgx.GraphLoadError):
        pgx.load_cache(bad)


def test_load_edge_list(tmp_path):
    p = tmp_path / "e.txt"
    p.write_text("# comment\n10 20\n20 30\n\n30 10\n")
    g = pgx.load_edge_list(p)
    assert g.vertex_count == 3 and g.edge_count == 3
    assert g.original_ids(np.array([0, 1, 2])).tolist() == [10, 20, 30]
    p.write_text("1 2\n3\n")
    with pytest.raises(pgx.GraphLoadError, match=":2:"):
        pgx.load_edge_list(p)


def test_partition_bounds_balance():
    """The multi-GPU owner ranges (distributed.partition_bounds): contiguous,
    covering, each carrying < total / W + max work of out_degree + 1."""
    from paper_2010_01542_b200.distributed import partition_bounds
    assert partition_bounds(np.empty(0, int), 4).tolist() == [0] * 5
    assert partition_bounds(np.array([5, 1, 1, 1]), 1).tolist() == [0, 4]
    rng = np.random.default_rng(1)
    for w in (2, 3, 8, 32):
        deg = rng.zipf(2.3, size=2000).clip(max=2000)
        b = partition_bounds(deg, w)
        assert b[0] == 0 and b[-1] == deg.size and np.all(np.diff(b) >= 0)
        work = deg + 1
        total, mx = int(work.sum()), int(work.max())
        for k in range(w):
            assert int(work[b[k]:b[k + 1]].sum()) * w < total + mx * w
    with pytest.raises(ValueError):
        partition_bounds(np.array([1]), 0)


def test_gather_adjacency_matches_slices():
    g = pgx.from_edges([0, 0, 1, 2, 2, 2], [1, 2, 2, 0, 1, 2], 3)
    flat, lens = pgx.gather_adjacency(g.out_offsets, g.out_targets, [2, 0, 2])
    assert flat.tolist() == [0, 1, 2, 1, 2, 0, 1, 2]
    assert lens.tolist() == [3, 2, 3]


def test_program_validation_and_lowering():
    with pytest.raises(pgx.ConfigError):
        pgx.pagerank(iterations=0)
    with pytest.raises(pgx.ConfigError):
        pgx.pagerank(damping=1.5)
    with pytest.raises(pgx.ConfigError):
        pgx.sssp(-1)
    g = pgx.from_edges([0], [1], 2)
    custom = pgx.VertexProgram(compute=lambda ctx: None, comm_mode=pgx.CommMode.PUSH,
                               message_dtype=np.int64, state_dtype=np.int64,
                               combine=pgx.min_combine(np.int64))
    with pytest.raises(pgx.ConfigError, match="no device lowering"):
        pgx.run(g, custom)
    pr = pgx.pagerank(iterations=4)
    hooked = pgx.VertexProgram(compute=pr.compute, comm_mode=pr.comm_mode,
                               message_dtype=pr.message_dtype, state_dtype=pr.state_dtype,
                               combine=pr.combine, setup=pr.setup,
                               on_superstep_end=lambda s, st: None, track_active=False)
    with pytest.raises(pgx.ConfigError, match="on_superstep_end"):
        pgx.run(g, hooked)
    no_combine = pgx.VertexProgram(compute=lambda c: None, comm_mode=pgx.CommMode.PUSH,
                                   message_dtype=np.int64, state_dtype=np.int64)
    with pytest.raises(pgx.ConfigError):
        pgx.run(g, no_combine)
    with pytest.raises(pgx.ConfigError):
        pgx.run(g, pgx.sssp(0), pgx.EngineConfig(workers=0))
    with pytest.raises(pgx.ConfigError):
        pgx.run(g, pgx.sssp(0), pgx.EngineConfig(max_supersteps=0))
    for bad in (dict(segments="yes"), dict(direction="pull"), dict(pagerank_mode="both"),
                dict(hub_cache="maybe"), dict(pagerank_hubs="yes"), dict(overlap_upload="on")):
        with pytest.raises(pgx.ConfigError):
            pgx.run(g, pgx.sssp(0), pgx.EngineConfig(**bad))
    with pytest.raises(pgx.ConfigError):
        pgx.run(g, pgx.sssp(2))


def test_empty_graph_runs_without_device():
    e = pgx.from_edges(np.empty(0, int), np.empty(0, int), 0)
    r = pgx.run(e, pgx.pagerank())
    assert r.values.shape == (0,) and r.superstep_count == 1
    r = pgx.run(e, pgx.connected_components())
    assert r.values.dtype == np.int64
    with pytest.raises(pgx.ConfigError):
        pgx.run(e, pgx.sssp(0))


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _reference_caches():
    import json
    return json.load(open(os.path.join(GOLDEN, "reference_cache.json")))["graphs"]


@pytest.mark.parametrize("name", sorted(_reference_caches()))
def test_cache_files_written_by_the_reference(name, tmp_path):
    """load_cache reads pregelite's own snapshots (graph.py:298-373) and
    save_cache writes them back byte for byte."""
    want = _reference_caches()[name]
    path = os.path.join(GOLDEN, f"reference_cache_{name}.pglcsr")
    g = pgx.load_cache(path)
    assert g.vertex_count == want["n"] and g.edge_count == want["m"]
    assert g.out_offsets.tolist() == want["out_offsets"]
    assert g.out_targets.tolist() == want["out_targets"]
    assert g.in_offsets.tolist() == want["in_offsets"]
    assert g.in_targets.tolist() == want["in_targets"]
    assert str(g.out_targets.cpu().numpy().dtype) == want["id_dtype"]
    if want["id_map"] is None:
        assert g.id_map is None
    else:
        assert list(g.id_map) == want["id_map"]
    out = tmp_path / "again.pglcsr"
    pgx.save_cache(g, out)
    assert out.read_bytes() == open(path, "rb").read()


def test_cache_of_our_graphs_matches_the_reference_bytes(tmp_path):
    """The same graphs built with this package's from_edges / load_edge_list
    serialise to the reference's exact bytes."""
    ours = {
        "dup_loops_d": pgx.from_edges([0, 0, 0, 1, 2, 2, 4], [0, 1, 1, 2, 2, 0, 1], 5),
        "tri_tail_u": pgx.from_edges([0, 1, 2, 3], [1, 2, 0, 4], 6, undirected=True),
        "ids64_d": pgx.from_edges([3, 1, 2, 0], [0, 0, 3, 2], 4, id_dtype=np.int64),
        "empty3": pgx.from_edges([], [], 3),
    }
    el = tmp_path / "edges.txt"
    el.write_text("# sparse ids\n1000 7\n7 42\n42 1000\n99 7\n")
    ours["edgelist_idmap_u"] = pgx.load_edge_list(str(el), undirected=True)
    for name, g in ours.items():
        out = tmp_path / f"{name}.pglcsr"
        pgx.save_cache(g, out)
        ref = open(os.path.join(GOLDEN, f"reference_cache_{name}.pglcsr"), "rb").read()
        assert out.read_bytes() == ref, name


def test_load_cache_rejects_short_and_odd_files(tmp_path):
    src = os.path.join(GOLDEN, "reference_cache_dup_loops_d.pglcsr")
    blob = open(src, "rb").read()
    cases = {"short36": (blob[:36], "truncated"), "short20": (blob[:20], "bad magic"),
             "cut": (blob[:-4], "truncated"), "extra": (blob + b"\0" * 8, "trailing"),
             "dtype": (blob[:8] + b"<f8".ljust(8, b"\0") + blob[16:], "unsupported id dtype")}
    for name, (data, msg) in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(pgx.GraphLoadError, match=msg):
            pgx.load_cache(p)


@pytest.mark.parametrize("off,tgt", [([1, 2], [0, 0]), ([0, 3], [0, 0]), ([0, 2, 1], [0, 1]),
                                     ([0, 1], [5]), ([0, 1], [-1])])
def test_from_csr_rejects_malformed_input(off, tgt):
    with pytest.raises(pgx.GraphLoadError):
        pgx.from_csr(np.array(off), np.array(tgt, dtype=np.int32))


def test_huge_superstep_cap_is_cheap():
    """A cap used to mean 'unbounded' must not size device buffers by it."""
    from paper_2010_01542_b200.engine import _validate
    _validate(pgx.connected_components(), pgx.EngineConfig(max_supersteps=2 ** 31 - 2))
