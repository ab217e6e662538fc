"""CUDA phase kernels of the partitioned superstep on one GPU.

W ranks run as threads (tests/thread_dist.py) sharing cuda:0; each owns a
CudaBackend (local CSR, full-width mailbox, owned slice) and the driver is
the production PartitionedRun, with each mailbox exchange: the fused peer
scatter (pgx_scatter_peer combining straight into the owners' mailboxes),
the per-superstep dense / sparse collectives, dense only.  Results must equal the oracle's (CC / SSSP
exact with per-superstep counts, PageRank within 1e-9) for W = 1, 2, 4, 8.
"""

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from oracle import oracle as O
from paper_2010_01542_b200.distributed import (CudaBackend, PartitionedRun,
                                               partition_bounds)
from thread_dist import run_ranks

pytestmark = pytest.mark.gpu

SPECS = [O.RmatSpec(14, 8, .57, .19, .19, 31, True),
         O.RmatSpec(13, 16, .45, .22, .22, 32, False)]


def _run(off, tgt, app, kw, world, exchange="auto", pr_mode="pull", d=None):
    n = off.size - 1
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    bounds = partition_bounds(np.diff(off), world)

    def rank_fn(r, d):
        be = CudaBackend(g, int(bounds[r]), int(bounds[r + 1]), "cuda:0", pr_mode=pr_mode)
        run = PartitionedRun(be, d, bounds, n, int(tgt.size))
        run.exchange = exchange
        cap = kw.get("max_supersteps", 10_000)
        if app == "pagerank":
            return run.run_pagerank(10, 0.85, cap)
        return run.run_min(app, kw.get("source", 0), cap)
    return run_ranks(world, rank_fn, d)[0]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("pr_mode", ["pull", "push"])
def test_partitioned_pagerank_modes(world, pr_mode):
    """Partitioned PageRank on the pull fold (pgx_gather_slice +
    pgx_fold_spanning, default) and on the red.add.f64 push arm: both
    within 1e-9 of the oracle, through the equal-block reduce_scatter."""
    from thread_dist import ThreadDist
    for spec in SPECS:
        n, off, tgt = O.rmat_csr(spec)
        want = O.run_pagerank(n, off, tgt)
        d = ThreadDist(world)
        vals, stats, hit, _ = _run(off, tgt, "pagerank", {}, world, pr_mode=pr_mode, d=d)
        v = vals.cpu().numpy()
        assert np.max(np.abs(v - want.values) / np.abs(want.values)) <= 1e-9
        assert [s["messages_sent"] for s in stats] == want.messages_sent
        assert d.calls.get("reduce_scatter_tensor") == 10  # one per superstep


def test_collectives_of_the_production_branch():
    """The thread stand-in reports the NCCL backend, so the driver takes the
    device-tensor branch: dense supersteps are one reduce_scatter_tensor,
    sparse ones all_to_all_single."""
    from thread_dist import ThreadDist
    n, off, tgt = O.rmat_csr(SPECS[0])
    d = ThreadDist(2)
    vals, stats, hit, _ = _run(off, tgt, "components", {}, 2, exchange="hybrid", d=d)
    ex = [s["exchange"] for s in stats]
    assert d.calls.get("reduce_scatter_tensor") == ex.count("dense") > 0
    assert d.calls.get("all_to_all_single") == 2 * ex.count("sparse") > 0
    assert np.array_equal(vals.cpu().numpy().view(np.uint32).astype(np.int64),
                          O.run_cc(n, off, tgt).values.astype(np.int64))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("spec", SPECS, ids=["sym", "dir"])
@pytest.mark.parametrize("exchange", ["auto", "peer", "hybrid", "dense"])
def test_partitioned_cuda_matches_oracle(spec, world, exchange):
    n, off, tgt = O.rmat_csr(spec)
    src = int(np.argmax(np.diff(off)))
    for app, kw, want in (
            ("components", {}, O.run_cc(n, off, tgt)),
            ("sssp", {"source": src}, O.run_sssp(n, off, tgt, src)),
            ("components", {"max_supersteps": 2}, O.run_cc(n, off, tgt, max_steps=2)),
            ("pagerank", {}, O.run_pagerank(n, off, tgt))):
        vals, stats, hit, _ = _run(off, tgt, app, kw, world, exchange)
        v = vals.cpu().numpy()
        if app == "pagerank":
            assert np.max(np.abs(v - want.values) / np.abs(want.values)) <= 1e-9
        else:
            assert np.array_equal(v.view(np.uint32).astype(np.int64),
                                  want.values.astype(np.int64)), (app, world)
        assert [s["active_count"] for s in stats] == want.active_counts, (app, world)
        assert [s["messages_sent"] for s in stats] == want.messages_sent, (app, world)
        assert hit == want.hit_superstep_cap
        if app != "pagerank":
            used = {s["exchange"] for s in stats}
            assert used <= {"peer": {"peer"}, "auto": {"dense", "sparse", "peer"}}.get(
                exchange, {"dense", "sparse"})


@pytest.mark.parametrize("exchange", ["peer", "hybrid"])
def test_partitioned_from_pinned_host_graph(exchange):
    """Each rank uploads only its own rows of a page-locked host graph (the
    end-to-end path of bench.py under torchrun)."""
    spec = SPECS[0]
    n, off, tgt = O.rmat_csr(spec)
    host = pgx.from_csr(torch.from_numpy(off), torch.from_numpy(tgt)).pin_memory()
    bounds = partition_bounds(np.diff(off), 2)
    want = O.run_cc(n, off, tgt)

    def rank_fn(r, d):
        be = CudaBackend(host, int(bounds[r]), int(bounds[r + 1]), "cuda:0")
        assert be.col.numel() == int(off[bounds[r + 1]] - off[bounds[r]])
        run = PartitionedRun(be, d, bounds, n, int(tgt.size))
        run.exchange = exchange
        return run.run_min("components", 0, 10_000)
    vals, stats, hit, _ = run_ranks(2, rank_fn)[0]
    assert np.array_equal(vals.cpu().numpy().view(np.uint32).astype(np.int64),
                          want.values.astype(np.int64))
    assert [s["active_count"] for s in stats] == want.active_counts


@pytest.mark.parametrize("exchange", ["auto", "hybrid"])
def test_partition_slices_at_unaligned_offsets(exchange):
    """Rank boundaries whose first edge offset is not a multiple of 4: each
    rank's col_idx is then an unaligned view of the targets."""
    n, off, tgt = O.rmat_csr(SPECS[0])
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    k = next(v for v in range(n // 3, n) if off[v] % 4 == 1)
    k2 = next(v for v in range(2 * n // 3, n) if off[v] % 4 == 3)
    bounds = np.array([0, k, k2, n], dtype=np.int64)
    want = O.run_cc(n, off, tgt)

    def rank_fn(r, d):
        be = CudaBackend(g, int(bounds[r]), int(bounds[r + 1]), "cuda:0")
        run = PartitionedRun(be, d, bounds, n, int(tgt.size))
        run.exchange = exchange
        return run.run_min("components", 0, 10_000)
    vals, stats, hit, _ = run_ranks(3, rank_fn)[0]
    assert np.array_equal(vals.cpu().numpy().view(np.uint32).astype(np.int64),
                          want.values.astype(np.int64))
    assert [s["active_count"] for s in stats] == want.active_counts


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_c2_full_size_known_answer(world):
    """BASELINE config C2 (65M edges) through the partitioned superstep:
    the labels hash and per-superstep counts of BASELINE.md, bit-exact."""
    import hashlib
    from paper_2010_01542_b200.rmat import rmat_graph
    g = rmat_graph("C2")
    n, m = g.vertex_count, g.edge_count
    bounds = partition_bounds(torch.diff(g.out_offsets).cpu().numpy(), world)

    def rank_fn(r, d):
        be = CudaBackend(g, int(bounds[r]), int(bounds[r + 1]), "cuda:0")
        run = PartitionedRun(be, d, bounds, n, m)
        return run.run_min("components", 0, 10_000)
    vals, stats, hit, _ = run_ranks(world, rank_fn)[0]
    lab = vals.cpu().numpy().view(np.uint32)
    assert hashlib.sha256(lab.astype("<u4").tobytes()).hexdigest() == \
        "c4e2cc1d7b5db62b9818e1cd41611649a294c5623d7e29804c175f904c40bf98"
    assert [s["active_count"] for s in stats] == \
        [4194304, 2009754, 2004276, 1499157, 208894, 2173, 23]
    assert [s["edges"] for s in stats] == \
        [65242574, 64803511, 28608953, 348075, 2192, 23, 0]
    assert {s["exchange"] for s in stats} == {"dense", "peer"}


def test_partitioned_c3_and_c4_full_size():
    """C3 SSSP (distances hash of BASELINE.md) and C4 PageRank (per-vertex
    relative error <= 1e-9 against the single-GPU pull run, rank[0] of
    BASELINE.md) through the partitioned superstep with 3 ranks."""
    import hashlib
    from paper_2010_01542_b200.rmat import rmat_graph
    world = 3
    for cfg in ("C3", "C4"):
        g = rmat_graph(cfg)
        n, m = g.vertex_count, g.edge_count
        bounds = partition_bounds(torch.diff(g.out_offsets).cpu().numpy(), world)

        def rank_fn(r, d):
            be = CudaBackend(g, int(bounds[r]), int(bounds[r + 1]), "cuda:0")
            run = PartitionedRun(be, d, bounds, n, m)
            if cfg == "C3":
                return run.run_min("sssp", 0, 10_000)
            return run.run_pagerank(10, 0.85, 10_000)
        vals, stats, hit, _ = run_ranks(world, rank_fn)[0]
        if cfg == "C3":
            d = vals.cpu().numpy().view(np.uint32)
            assert hashlib.sha256(d.astype("<u4").tobytes()).hexdigest() == \
                "bd08774026f70bbd29b80c977187f880654c0d8cbd2b42ba0988fed279ffa1e2"
            assert [s["messages_sent"] for s in stats] == \
                [97364, 36379100, 27861844, 339319, 2142, 6, 0]
        else:
            got = vals.cpu().numpy()
            want = pgx.run(g, pgx.pagerank()).values
            assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-9
            assert abs(got[0] - 0.0001216244232021811) / 0.0001216244232021811 <= 1e-9
        del g
        torch.cuda.empty_cache()


def _adversarial(rng):
    yield "star_out", np.zeros(499, int), np.arange(1, 500), 500, False
    yield "star_in", np.arange(1, 500), np.zeros(499, int), 500, False
    yield "isolated_heavy", np.array([3, 3, 7]), np.array([7, 9, 3]), 4000, True
    yield "tiny_many_ranks", np.array([0, 1]), np.array([1, 2]), 3, True
    for i in range(8):
        n = int(rng.integers(2, 5000))
        m = int(rng.integers(0, 8 * n))
        if i % 2:
            p = 1.0 / np.arange(1, n + 1) ** 1.1
            p /= p.sum()
            src, dst = rng.choice(n, m, p=p), rng.choice(n, m, p=p)
        else:
            src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        yield f"random{i}", src, dst, n, bool(i % 3 == 0)


@pytest.mark.parametrize("case", list(_adversarial(np.random.default_rng(99))),
                         ids=lambda c: c[0])
def test_partitioned_randomized_vs_oracle(case):
    """Adversarial shapes for the partition: ranks whose range is empty,
    hubs owning a whole range, isolated vertices, more ranks than vertices;
    CC / SSSP exact with per-superstep counts, PageRank <= 1e-9."""
    name, src, dst, n, und = case
    off, tgt = O.csr_from_edges(src, dst, n, und)
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    source = int(np.argmax(np.diff(off)))
    want = {"components": O.run_cc(n, off, tgt), "sssp": O.run_sssp(n, off, tgt, source),
            "pagerank": O.run_pagerank(n, off, tgt)}
    for world, exchange in ((2, "auto"), (3, "peer"), (5, "hybrid"), (7, "auto")):
        bounds = partition_bounds(np.diff(off), world)
        for app in ("components", "sssp", "pagerank"):
            def rank_fn(r, d):
                be = CudaBackend(g, int(bounds[r]), int(bounds[r + 1]), "cuda:0")
                run = PartitionedRun(be, d, bounds, n, int(tgt.size))
                run.exchange = exchange
                if app == "pagerank":
                    return run.run_pagerank(10, 0.85, 10_000)
                return run.run_min(app, source, 10_000)
            vals, stats, hit, _ = run_ranks(world, rank_fn)[0]
            w = want[app]
            v = vals.cpu().numpy()
            if app == "pagerank":
                assert np.max(np.abs(v - w.values) / np.abs(w.values)) <= 1e-9, (name, world)
            else:
                assert np.array_equal(v.view(np.uint32).astype(np.int64),
                                      w.values.astype(np.int64)), (name, world, app)
                assert [s["active_count"] for s in stats] == w.active_counts, (name, world, app)
                assert [s["messages_sent"] for s in stats] == w.messages_sent, (name, world, app)
