"""Parity of the B200 engine (through libpgx.so's C ABI) with the reference.

* every reference run recorded in tests/golden (values, superstep counts,
  cap flag, per-superstep active / message counts);
* the GPU R-MAT builder against BASELINE.md's CSR hashes;
* full-size configs against BASELINE.md known answers (C2 labels hash, C3
  distances hash, per-superstep counts) and against the pinned CPU oracle
  (C1 and C4 PageRank, relative error <= 1e-9 per vertex, the north-star
  tolerance).

Tolerance: CC labels and SSSP distances bit-exact; PageRank per-vertex
relative error <= 1e-9 (BASELINE.json north_star) -- the push scatter adds
shares with red.add.f64 in arrival order, the reference folds them in
adjacency order.
"""

import ctypes
import hashlib

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200 import engine as engine_mod
from golden_cases import DANGLING_RANKS, PATH3_RANKS, load_runs
from oracle import oracle as O
from paper_2010_01542_b200.rmat import rmat_graph

pytestmark = pytest.mark.gpu

PR_RTOL = 1e-9
RUNS = load_runs()


def sha(t, dt):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else t
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def program(app, kw):
    kw = dict(kw)
    kw.pop("max_supersteps", None)
    return {"sssp": pgx.sssp, "components": pgx.connected_components,
            "pagerank": pgx.pagerank}[app](**kw)


def rel_err(got, want):
    if len(want) == 0:
        return 0.0
    return float(np.max(np.abs(got - want) / np.abs(want)))


@pytest.fixture
def seg_threshold():
    """Set PGX_OPT_SEG_MIN_EDGES (and optionally the gate / fused-apply
    knobs) for one test, restore the shipped values."""
    def set_(v, pred=1):
        _lib.set_option(_lib.PGX_OPT_SEG_MIN_EDGES, v)
        _lib.set_option(_lib.PGX_OPT_SEG_PREDICT, pred)
    yield set_
    set_(256)


@pytest.fixture
def pull_threshold():
    """Set PGX_OPT_PULL_MIN_EDGES (bottom-up SSSP supersteps from m * v /
    1024 sender edges) for one test, restore the shipped value."""
    def set_(v):
        _lib.set_option(_lib.PGX_OPT_PULL_MIN_EDGES, v)
    yield set_
    set_(128)


# modes: pull / push (PageRank lowering, min programs with the shipped
# segment policy: device graphs get the segmented scatter for supersteps
# with >= m/4 sender edges), hubs (hub-cache arm), k1 (segments off: K1 in
# every superstep), segall (the segmented scatter whenever its send values
# are exact: every superstep until the first K1 one), segskip (default
# threshold, the apply never builds a frontier after a segmented superstep,
# so every superstep after one runs segmented too), bu / buall (unit-weight
# SSSP direction-optimising at the shipped threshold / bottom-up in every
# superstep after the first), push1 (SSSP push only), prhubs / prhubs3
# (pull PageRank with the shared-memory hub-source table: every source of
# out-degree >= 2 a hub / only the top 3)
@pytest.mark.parametrize("mode", ["pull", "push", "hubs", "k1", "segall", "segskip", "bu",
                                  "buall", "push1", "prhubs", "prhubs3", "hostcc"])
@pytest.mark.parametrize("r", RUNS, ids=lambda r: r.id)
def test_golden_reference_runs(r, mode, seg_threshold, pull_threshold, monkeypatch):
    if mode in ("push", "prhubs", "prhubs3") and r.app != "pagerank":
        pytest.skip("pagerank_mode / pagerank_hubs only change the PageRank lowering")
    if mode == "prhubs3":
        monkeypatch.setenv("PGX_PR_HUBS", "3")
    if mode in ("hubs", "k1", "segall", "segskip") and r.app == "pagerank":
        pytest.skip("hub_cache / segments only change the min combiner")
    if mode in ("bu", "buall", "push1") and r.app != "sssp":
        pytest.skip("direction only changes unit-weight SSSP")
    if mode == "hostcc" and r.app != "components":
        pytest.skip("the upload pipeline runs connected components")
    if mode == "hostcc":  # host graph: superstep 0 under the upload, 7-edge chunks
        monkeypatch.setattr(engine_mod, "_OVERLAP_CHUNK", 7)
    g = pgx.from_edges(r.src, r.dst, r.n, undirected=r.undirected,
                       device="cpu" if mode == "hostcc" else "cuda")
    cap = r.kwargs.get("max_supersteps")
    cfg = pgx.EngineConfig(max_supersteps=cap if cap else pgx.DEFAULT_MAX_SUPERSTEPS,
                           pagerank_mode="push" if mode == "push" else "pull",
                           pagerank_hubs="on" if mode.startswith("prhubs") else "off",
                           hub_cache="on" if mode == "hubs" else "off",
                           segments="off" if mode == "k1" else
                           "on" if mode.startswith("seg") else "auto",
                           direction="on" if mode.startswith("bu") else
                           "off" if mode == "push1" else "auto")
    if mode == "buall":
        pull_threshold(0)
    if mode == "segall":
        seg_threshold(0)
    elif mode == "segskip":
        seg_threshold(256, pred=2)
    rep = pgx.run(g, program(r.app, r.kwargs), cfg)
    if r.app == "pagerank":
        assert rep.values.dtype == np.float64
        assert rel_err(rep.values, r.values) <= PR_RTOL
    elif r.app == "sssp":
        assert rep.values.dtype == np.uint32
        assert np.array_equal(rep.values, r.values)
    else:
        assert rep.values.dtype == np.int64
        assert np.array_equal(rep.values, r.values)
    assert rep.superstep_count == r.superstep_count
    assert rep.hit_superstep_cap == r.hit_superstep_cap
    assert [s.active_count for s in rep.supersteps] == r.active_counts
    assert [s.messages_sent for s in rep.supersteps] == r.messages_sent


def test_reference_golden_vectors():
    # reference tests/test_algorithms.py:27-43
    g = pgx.from_edges([0, 1], [1, 2], 3, undirected=True)
    got = pgx.run(g, pgx.pagerank()).values
    assert np.max(np.abs(got - np.array(PATH3_RANKS))) < 1e-9
    g = pgx.from_edges([0, 0, 1], [1, 2, 2], 3)
    got = pgx.run(g, pgx.pagerank()).values
    assert np.max(np.abs(got - np.array(DANGLING_RANKS))) < 1e-9
    assert abs(got.sum() - 1.0) < 1e-12
    # reference tests/test_engine.py:29-37
    g = pgx.from_edges([0, 1, 2], [1, 2, 3], 4, undirected=True)
    rep = pgx.run(g, pgx.sssp(0))
    assert rep.values.tolist() == [0, 1, 2, 3]
    assert [s.active_count for s in rep.supersteps] == [4, 1, 2, 2, 1]
    assert [s.messages_sent for s in rep.supersteps] == [1, 2, 2, 1, 0]


def test_n_path_takes_n_plus_one_supersteps():
    # reference tests/test_acceptance.py:490-511
    for n in range(1, 65):
        src = np.arange(n - 1)
        g = pgx.from_edges(src, src + 1, n, undirected=True)
        rep = pgx.run(g, pgx.sssp(0))
        assert rep.values.tolist() == list(range(n))
        assert rep.superstep_count == (n + 1 if n >= 2 else 1)


def test_errors_and_edge_cases():
    g = pgx.from_edges([0, 1], [1, 2], 3)
    with pytest.raises(pgx.ConfigError):
        pgx.run(g, pgx.sssp(3))
    empty = pgx.from_edges(np.empty(0, int), np.empty(0, int), 0)
    assert pgx.run(empty, pgx.pagerank()).values.shape == (0,)
    assert pgx.run(empty, pgx.connected_components()).values.shape == (0,)
    with pytest.raises(pgx.ConfigError):
        pgx.run(empty, pgx.sssp(0))
    # extract override (reference tests/test_engine.py:144-155)
    prog = pgx.sssp(0)
    prog = pgx.VertexProgram(compute=prog.compute, comm_mode=prog.comm_mode,
                             message_dtype=prog.message_dtype,
                             state_dtype=prog.state_dtype, combine=prog.combine,
                             setup=prog.setup,
                             extract=lambda store: store.state.astype(np.int64) * 10)
    g = pgx.from_edges([0, 1], [1, 2], 3, undirected=True)
    assert pgx.run(g, prog).values.tolist() == [0, 10, 20]


def test_host_graph_and_device_graph_agree():
    n, off, tgt = O.rmat_csr(O.RmatSpec(13, 16, .57, .19, .19, 9, True))
    host = pgx.from_csr(torch.from_numpy(off), torch.from_numpy(tgt)).pin_memory()
    dev = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    for prog in (pgx.connected_components(), pgx.sssp(0)):
        a, b = pgx.run(host, prog), pgx.run(dev, prog)
        assert np.array_equal(a.values, b.values)
        assert a.supersteps == b.supersteps or \
            [s.active_count for s in a.supersteps] == [s.active_count for s in b.supersteps]


def test_repeat_runs_deterministic():
    n, off, tgt = O.rmat_csr(O.RmatSpec(14, 8, .57, .19, .19, 11, True))
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    a = pgx.run(g, pgx.connected_components())
    for _ in range(3):
        b = pgx.run(g, pgx.connected_components())
        assert np.array_equal(a.values, b.values)
        assert [s.active_count for s in a.supersteps] == \
            [s.active_count for s in b.supersteps]
    p = pgx.run(g, pgx.pagerank()).values
    q = pgx.run(g, pgx.pagerank()).values
    assert np.array_equal(p, q)  # pull mode: no atomics, fixed fold order
    q = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(pagerank_mode="push")).values
    assert rel_err(p, q) <= 1e-12


# ----------------------------------------------------------------------
# full-size configs
# ----------------------------------------------------------------------

CSR_HASHES = {
    "C1": ("8e2c9c7ecc7087595f3b3d6738c80e0eea0c7f3edb30b9397604cad1b0ebabac",
           "b920d8fe143abe02a3459674d13419b061340af5008426612925db3b8efaec08"),
    "C2": ("aa2ac4555df0c0fb7c1a95773d688be797f718cf6164f925d28de9c02318bf36",
           "ff82f71753fbeba1d1a651bfa6015d922da2d9d9e4357a4c5687cdcceccbba7c"),
    "C3": ("d170d3d509c9a166499b435e9565471846461f06c5b593f302326618f14da385",
           "11f2969e2050ea91eac527b41fdabad7ecb5640246aa4dfa12f023605737e5d6"),
    "C4": ("c1decf3c223d3503206518c3b0b8d2e94779f7ae38ec59192ce9691b4b4b5627",
           "142655f978f140e96c91626b7e4314416d90625024a609f0c9f02949d7d92d4d"),
}


@pytest.fixture(scope="module")
def graphs():
    cache = {}

    def get(name):
        if name not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[name] = rmat_graph(name)
        return cache[name]
    return get


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_gpu_rmat_matches_baseline_hashes(graphs, name):
    g = graphs(name)
    assert sha(g.out_offsets, "<i8") == CSR_HASHES[name][0]
    assert sha(g.out_targets, "<i4") == CSR_HASHES[name][1]


@pytest.mark.parametrize("mode", ["pull", "push", "pull-hubs"])
def test_c1_pagerank_vs_oracle(graphs, mode):
    g = graphs("C1")
    off = g.out_offsets.cpu().numpy()
    tgt = g.out_targets.cpu().numpy()
    want = O.run_pagerank(g.vertex_count, off, tgt)
    rep = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(
        pagerank_mode=mode[:4], pagerank_hubs="on" if mode == "pull-hubs" else "auto"))
    assert rel_err(rep.values, want.values) <= PR_RTOL
    assert rep.superstep_count == 10
    assert [s.messages_sent for s in rep.supersteps] == [40_445] * 9 + [0]
    assert int(np.argmax(rep.values)) == 0
    assert abs(rep.values[0] - 0.005883584525755893) / 0.005883584525755893 <= PR_RTOL


@pytest.mark.parametrize("hubs", ["off", "on"])
def test_c2_components_known_answer(graphs, hubs):
    g = graphs("C2")
    rep = pgx.run(g, pgx.connected_components(), pgx.EngineConfig(hub_cache=hubs))
    assert sha(rep.values.astype(np.uint32), "<u4") == \
        "c4e2cc1d7b5db62b9818e1cd41611649a294c5623d7e29804c175f904c40bf98"
    assert [s.active_count for s in rep.supersteps] == \
        [4194304, 2009754, 2004276, 1499157, 208894, 2173, 23]
    assert [s.messages_sent for s in rep.supersteps] == \
        [4194304, 1816650, 1905145, 269866, 2165, 23, 0]
    assert [s.edges for s in rep.supersteps] == \
        [65242574, 64803511, 28608953, 348075, 2192, 23, 0]
    assert len(np.unique(rep.values)) == 2_186_257


@pytest.mark.parametrize("hubs", ["off", "on"])
def test_c3_sssp_known_answer(graphs, hubs):
    g = graphs("C3")
    src = int(torch.argmax(g.out_degrees))
    assert src == 0
    rep = pgx.run(g, pgx.sssp(src), pgx.EngineConfig(hub_cache=hubs))
    assert sha(rep.values, "<u4") == \
        "bd08774026f70bbd29b80c977187f880654c0d8cbd2b42ba0988fed279ffa1e2"
    assert [s.active_count for s in rep.supersteps] == \
        [4194304, 97364, 1730927, 1490812, 146756, 2024, 6]
    assert [s.messages_sent for s in rep.supersteps] == \
        [97364, 36379100, 27861844, 339319, 2142, 6, 0]


@pytest.mark.parametrize("direction", ["off", "on", "all", "never"])
def test_c3_sssp_directions(graphs, direction, pull_threshold):
    """Bottom-up supersteps (pgx_pull.cuh) at C3's size: push only, the
    shipped threshold (supersteps 1 and 2 bottom-up), every superstep after
    the first bottom-up, and the threshold above m (no bottom-up with the
    in-CSR bound): one distance vector, one set of statistics."""
    g = graphs("C3")
    if direction == "all":
        pull_threshold(0)
    elif direction == "never":
        pull_threshold(1025)
    rep = pgx.run(g, pgx.sssp(0), pgx.EngineConfig(direction="off" if direction == "off"
                                                   else "on"))
    assert sha(rep.values, "<u4") == \
        "bd08774026f70bbd29b80c977187f880654c0d8cbd2b42ba0988fed279ffa1e2"
    assert [s.active_count for s in rep.supersteps] == \
        [4194304, 97364, 1730927, 1490812, 146756, 2024, 6]
    assert [s.messages_sent for s in rep.supersteps] == \
        [97364, 36379100, 27861844, 339319, 2142, 6, 0]
    assert [s.recipients for s in rep.supersteps] == \
        [97364, 1730927, 1490812, 146756, 2024, 6, 0]


@pytest.mark.parametrize("mode", ["pull", "push", "pull-nohubs"])
def test_c4_pagerank_vs_oracle(graphs, mode):
    g = graphs("C4")
    rep = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(
        pagerank_mode=mode[:4], pagerank_hubs="off" if mode == "pull-nohubs" else "auto"))
    off = g.out_offsets.cpu().numpy()
    tgt = g.out_targets.cpu().numpy()
    want = O.run_pagerank(g.vertex_count, off, tgt)
    assert rel_err(rep.values, want.values) <= PR_RTOL
    assert [s.messages_sent for s in rep.supersteps] == [3_751_426] * 9 + [0]
    assert abs(rep.values[0] - 0.0001216244232021811) / 0.0001216244232021811 <= PR_RTOL


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_pagerank_hub_table_bit_identical(graphs, name):
    """The shared-memory hub-source table changes where a hub's share is
    read from, not the values or the summation order: ranks are
    bit-identical with and without it (C4's default takes the table)."""
    g = graphs(name)
    on = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(pagerank_hubs="on"))
    off = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(pagerank_hubs="off"))
    assert np.array_equal(on.values, off.values)
    cap = ctypes.c_int32(0)
    _lib.check(_lib.load().pgx_pr_hub_capacity(ctypes.byref(cap)), "pgx_pr_hub_capacity")
    csr = g.device_csr(torch.device("cuda", 0))
    assert csr.pr_nhubs == cap.value
    enc = csr.pr_hub_col
    assert int((enc < 0).sum()) > 0


@pytest.mark.parametrize("chunk", [1 << 26, 1 << 20, 100_003])
def test_cc_upload_pipeline_matches(graphs, chunk, monkeypatch):
    """C2 from pinned host memory with superstep 0 combined while the
    targets upload (engine._upload_overlapped): labels and every
    per-superstep statistic equal the plain upload and the device graph."""
    monkeypatch.setattr(engine_mod, "_OVERLAP_CHUNK", chunk)
    g = graphs("C2")
    host = pgx.Graph(g.vertex_count, g.out_offsets.cpu(), g.out_targets.cpu()).pin_memory()
    ref = pgx.run(g, pgx.connected_components())
    for cfg in (pgx.EngineConfig(), pgx.EngineConfig(overlap_upload="off")):
        host.drop_device_cache()
        plan = pgx.plan_run(host, pgx.connected_components(), cfg)
        assert plan.prescattered == (cfg.overlap_upload == "auto")
        plan.launch()
        rep = pgx.collect(plan, pgx.connected_components())
        assert np.array_equal(rep.values, ref.values)
        assert rep.superstep_count == ref.superstep_count
        for a, b in zip(rep.supersteps, ref.supersteps):
            assert (a.active_count, a.messages_sent, a.edges, a.senders, a.recipients) == \
                (b.active_count, b.messages_sent, b.edges, b.senders, b.recipients)
        # a second launch of the same plan runs superstep 0 itself
        plan.launch()
        assert np.array_equal(pgx.collect(plan, pgx.connected_components()).values, ref.values)
    host.drop_device_cache()


def test_load_cache_pinned_and_on_device(tmp_path):
    """load_cache(device=...) reads into page-locked buffers and uploads;
    the device CSR equals the host one and runs through the engine."""
    import os
    g = rmat_graph("C1")
    p = tmp_path / "c1.pglcsr"
    pgx.save_cache(g, p)
    host = pgx.load_cache(p)
    pinned = pgx.load_cache(p, pin_memory=True)
    dev = pgx.load_cache(p, device="cuda")
    assert pinned.out_targets.is_pinned() and dev.out_targets.is_cuda
    for a in ("out_offsets", "out_targets", "in_offsets", "in_targets"):
        assert torch.equal(getattr(host, a), getattr(pinned, a))
        assert torch.equal(getattr(host, a), getattr(dev, a).cpu())
    want = pgx.run(host, pgx.pagerank()).values
    assert np.array_equal(pgx.run(dev, pgx.pagerank()).values, want)
    golden = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                          "reference_cache_edgelist_idmap_u.pglcsr")
    d = pgx.load_cache(golden, device="cuda")
    assert d.id_map is not None and d.out_targets.is_cuda


@pytest.mark.gpu
def test_unbounded_cap_sizes_buffers_by_n():
    """a cap of 2^31 - 2 ('unbounded') must not allocate per-cap
    statistics; CC / SSSP quiesce within n + 1 supersteps."""
    g = pgx.from_edges(np.arange(63), np.arange(1, 64), 64, undirected=True, device="cuda")
    cfg = pgx.EngineConfig(max_supersteps=2 ** 31 - 2)
    plan = pgx.plan_run(g, pgx.sssp(0), cfg)
    assert plan.stats.numel() <= _lib.PGX_STAT_HDR + _lib.PGX_STAT_FIELDS * (64 + 2)
    r = pgx.run(g, pgx.sssp(0), cfg)
    assert r.superstep_count == 65 and not r.hit_superstep_cap
    assert r.values.tolist() == list(range(64))
