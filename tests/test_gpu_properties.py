"""Size-independent properties at BASELINE sizes, and a randomized sweep.

Full-size configs are pinned by known answers elsewhere (test_gpu.py,
test_gpu_c5.py); these checks hold for ANY correct result and catch
classes of bugs a hash would only flag as "different":

* CC: labels are constant along every edge and every label is the minimum
  id of its class (so each label names a vertex labelled by itself);
* SSSP: dist[source] = 0, dist[v] <= dist[u] + 1 along every edge u->v,
  and every reached vertex != source has a predecessor at dist - 1;
* PageRank: ranks are positive and sum to 1 (mass conservation, ref test
  tests/test_algorithms.py:43), and one more superstep of the reference
  recurrence applied on the host to the 9-superstep result reproduces the
  10-superstep result.

The randomized sweep compares the GPU with the oracle on many small
adversarial graphs: stars, chains, cliques, self-loops, duplicate edges,
isolated vertices, one-vertex and edgeless graphs, random multigraphs.
"""

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from oracle import oracle as O
from paper_2010_01542_b200.rmat import rmat_graph

pytestmark = pytest.mark.gpu


def edge_arrays(g):
    off = g.out_offsets.to(torch.int64)
    src = torch.repeat_interleave(torch.arange(g.vertex_count, device=off.device),
                                  torch.diff(off))
    return src, g.out_targets.to(torch.int64)


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


def test_c2_components_properties(graphs):
    g = graphs("C2")
    lab = torch.from_numpy(pgx.run(g, pgx.connected_components()).values).cuda()
    src, dst = edge_arrays(g)
    assert torch.equal(lab[src], lab[dst])                    # constant on edges
    assert torch.equal(lab[lab], lab)                          # label is a fixed point
    ids = torch.arange(g.vertex_count, device=lab.device)
    assert bool((lab <= ids).all())                            # min id of the class


def test_c3_sssp_properties(graphs):
    g = graphs("C3")
    s = int(torch.argmax(g.out_degrees))
    d = torch.from_numpy(pgx.run(g, pgx.sssp(s)).values.astype(np.int64)).cuda()
    unreached = 2 ** 32 - 1
    src, dst = edge_arrays(g)
    assert int(d[s]) == 0
    fin = d[src] != unreached
    assert bool((d[dst][fin] <= d[src][fin] + 1).all())       # triangle inequality
    # every reached non-source vertex has an in-neighbour exactly one closer
    ok = torch.zeros(g.vertex_count, dtype=torch.bool, device=d.device)
    tight = fin & (d[dst] == d[src] + 1)
    ok[dst[tight]] = True
    reached = (d != unreached)
    reached[s] = False
    assert bool(ok[reached].all())


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_pagerank_properties(graphs, name):
    g = graphs(name)
    r10 = pgx.run(g, pgx.pagerank(10)).values
    r9 = pgx.run(g, pgx.pagerank(9)).values
    assert (r10 > 0).all()
    assert abs(r10.sum() - 1.0) < 1e-12
    # one host-side superstep of the reference recurrence (algorithms.py:61-78)
    n = g.vertex_count
    off = g.out_offsets.cpu().numpy()
    tgt = g.out_targets.cpu().numpy()
    deg = np.diff(off)
    src = np.repeat(np.arange(n), deg)
    share = np.where(deg > 0, r9 / np.maximum(deg, 1), 0.0)
    folded = np.bincount(tgt, weights=share[src], minlength=n)
    dangling = r9[deg == 0].sum()
    nxt = (1 - 0.85) / n + 0.85 * (folded + dangling / n)
    assert np.max(np.abs(nxt - r10) / r10) < 1e-9


def _adversarial_graphs(rng):
    yield "one_vertex", np.empty(0, int), np.empty(0, int), 1, False
    yield "edgeless", np.empty(0, int), np.empty(0, int), 17, False
    yield "self_loops", np.arange(5), np.arange(5), 5, False
    k = 40
    yield "star_out", np.zeros(k - 1, int), np.arange(1, k), k, False
    yield "star_in", np.arange(1, k), np.zeros(k - 1, int), k, False
    yield "chain_long", np.arange(299), np.arange(1, 300), 300, False
    c = 24
    a, b = np.meshgrid(np.arange(c), np.arange(c))
    yield "clique", a.ravel(), b.ravel(), c, False
    yield "dup_edges", np.repeat([0, 1, 2], 50), np.repeat([1, 2, 0], 50), 3, False
    yield "two_hubs", np.r_[np.zeros(600, int), np.full(600, 1)], \
        np.r_[np.arange(600) + 2, np.arange(600) + 2], 602, False
    for i in range(25):
        n = int(rng.integers(2, 3000 if i < 10 else 30_000))
        m = int(rng.integers(0, 6 * n))
        skew = rng.random() < 0.5
        if skew:
            p = 1.0 / np.arange(1, n + 1) ** 1.2
            p /= p.sum()
            src, dst = rng.choice(n, m, p=p), rng.choice(n, m, p=p)
        else:
            src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        yield f"random{i}", src, dst, n, bool(rng.random() < 0.5)


@pytest.mark.parametrize("case", list(_adversarial_graphs(np.random.default_rng(2026))),
                         ids=lambda c: c[0])
def test_randomized_gpu_vs_oracle(case):
    name, src, dst, n, und = case
    off, tgt = O.csr_from_edges(src, dst, n, und)
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    cc = pgx.run(g, pgx.connected_components())
    want = O.run_cc(n, off, tgt)
    assert np.array_equal(cc.values, want.values)
    assert [s.active_count for s in cc.supersteps] == want.active_counts
    assert [s.messages_sent for s in cc.supersteps] == want.messages_sent
    source = int(np.argmax(np.diff(off)))
    want = O.run_sssp(n, off, tgt, source)
    # push only, direction-optimising (shipped threshold), bottom-up in
    # every superstep after the first
    for direction, thr in (("off", 128), ("on", 128), ("on", 0)):
        _lib.set_option(_lib.PGX_OPT_PULL_MIN_EDGES, thr)
        try:
            sp = pgx.run(g, pgx.sssp(source), pgx.EngineConfig(direction=direction))
        finally:
            _lib.set_option(_lib.PGX_OPT_PULL_MIN_EDGES, 128)
        assert np.array_equal(sp.values, want.values), (direction, thr)
        assert [s.active_count for s in sp.supersteps] == want.active_counts
        assert [s.messages_sent for s in sp.supersteps] == want.messages_sent
    for mode in ("pull", "push"):
        pr = pgx.run(g, pgx.pagerank(), pgx.EngineConfig(pagerank_mode=mode))
        want = O.run_pagerank(n, off, tgt)
        assert np.max(np.abs(pr.values - want.values) / np.abs(want.values)) <= 1e-9
        assert pr.superstep_count == want.superstep_count


def _big_cases():
    k = 300_001
    yield "star_out_300k", np.zeros(k - 1, int), np.arange(1, k), k, False
    yield "star_in_300k", np.arange(1, k), np.zeros(k - 1, int), k, False
    yield "star_sym_300k", np.zeros(k - 1, int), np.arange(1, k), k, True
    n = 20_003  # a long chain: 20k tiny supersteps, n not a multiple of 32
    yield "chain_20k", np.arange(n - 1), np.arange(1, n), n, True
    rng = np.random.default_rng(7)
    n = 100_003
    hubs = rng.integers(0, 50, 400_000)
    yield "hubby_dir", hubs, rng.integers(0, n, 400_000), n, False


@pytest.mark.parametrize("case", list(_big_cases()), ids=lambda c: c[0])
def test_large_hub_rows_and_long_runs_vs_oracle(case):
    """Rows spanning thousands of 256-edge tiles, in-hubs receiving 300k
    messages per superstep, and 20k-superstep runs: CC / SSSP exact with
    per-superstep counts (the unit-weight SSSP bitmap kernel included)."""
    name, src, dst, n, und = case
    off, tgt = O.csr_from_edges(src, dst, n, und)
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    cap = 30_000
    for source in (0, n - 1):
        want = O.run_sssp(n, off, tgt, source, cap)
        for thr in (128, 0):  # shipped direction threshold / bottom-up throughout
            _lib.set_option(_lib.PGX_OPT_PULL_MIN_EDGES, thr)
            try:
                sp = pgx.run(g, pgx.sssp(source), pgx.EngineConfig(max_supersteps=cap))
            finally:
                _lib.set_option(_lib.PGX_OPT_PULL_MIN_EDGES, 128)
            assert np.array_equal(sp.values, want.values), (name, source, thr)
            assert [s.active_count for s in sp.supersteps] == want.active_counts
            assert [s.messages_sent for s in sp.supersteps] == want.messages_sent
    cc = pgx.run(g, pgx.connected_components(), pgx.EngineConfig(max_supersteps=cap))
    want = O.run_cc(n, off, tgt, max_steps=cap)
    assert np.array_equal(cc.values, want.values)
    assert [s.active_count for s in cc.supersteps] == want.active_counts


def test_unaligned_views_of_the_csr():
    """col_idx may be any 4-byte-aligned view (a user's slice, a rank's
    share of the targets): the dense superstep's L2 bulk prefetch widens
    its range to 16-byte granules instead of faulting."""
    n, off, tgt = O.rmat_csr(O.RmatSpec(12, 8, .57, .19, .19, 5, True))
    want = O.run_cc(n, off, tgt)
    for shift in (1, 2, 3):
        buf = torch.zeros(tgt.size + shift, dtype=torch.int32, device="cuda")
        buf[shift:] = torch.from_numpy(tgt).cuda()
        view = buf[shift:]
        assert view.data_ptr() % 16 != 0
        g = pgx.from_csr(torch.from_numpy(off).cuda(), view)
        rep = pgx.run(g, pgx.connected_components())
        assert np.array_equal(rep.values, want.values)
        assert [s.active_count for s in rep.supersteps] == want.active_counts
