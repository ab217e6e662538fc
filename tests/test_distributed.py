"""Partitioned multi-GPU host logic over gloo (world sizes 2 and 3, CPU).

The driver (paper_2010_01542_b200.distributed.PartitionedRun) is the one
the CUDA backend uses under torchrun; here the per-rank phases run on the
CPU test backend (tests/dist_backend.py), for every mailbox exchange: the
collective ones (dense reduction, sparse pairs, chosen per superstep) and
the fused peer exchange (shared-memory mailboxes standing in for CUDA IPC).  Results must equal the oracle's
(and therefore the reference's): CC labels / SSSP distances exact, per-
superstep active and message counts exact, PageRank within 1e-9.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2010_01542_b200.distributed import PartitionedRun, partition_bounds

CASES = [
    ("rmat11_sym", O.RmatSpec(11, 8, .57, .19, .19, 21, True)),
    ("rmat11_dir", O.RmatSpec(11, 16, .57, .19, .19, 22, False)),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, jobs, out_dir, exchange="hybrid"):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from dist_backend import CpuBackend
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    results = []
    backends = []
    for (off, tgt, app, kw) in jobs:
        n = off.size - 1
        bounds = partition_bounds(np.diff(off), world)
        be = CpuBackend(off, tgt, int(bounds[rank]), int(bounds[rank + 1]))
        backends.append(be)
        run = PartitionedRun(be, dist, bounds, n, int(tgt.size))
        run.exchange = exchange
        cap = kw.get("max_supersteps", 10_000)
        if app == "pagerank":
            vals, stats, hit, _ = run.run_pagerank(kw.get("iterations", 10),
                                                   kw.get("damping", 0.85), cap)
        else:
            vals, stats, hit, _ = run.run_min(app, kw.get("source", 0), cap)
        results.append((vals.numpy(), [(s["active_count"], s["messages_sent"])
                                        for s in stats], hit,
                        [s.get("exchange") for s in stats]))
    if rank == 0:
        torch.save(results, os.path.join(out_dir, "results.pt"))
    dist.barrier()
    for be in backends:
        be.close()
    dist.destroy_process_group()


def _jobs():
    jobs = []
    for name, spec in CASES:
        n, off, tgt = O.rmat_csr(spec)
        src = int(np.argmax(np.diff(off)))
        jobs += [(off, tgt, "components", {}), (off, tgt, "sssp", {"source": src}),
                 (off, tgt, "pagerank", {}), (off, tgt, "components", {"max_supersteps": 2}),
                 (off, tgt, "pagerank", {"max_supersteps": 3})]
    # path with more ranks than some ranges can fill, and a dangling graph
    off, tgt = O.csr_from_edges(np.arange(9), np.arange(1, 10), 10, undirected=True)
    jobs += [(off, tgt, "sssp", {"source": 0}), (off, tgt, "components", {})]
    off, tgt = O.csr_from_edges([0, 0, 1], [1, 2, 2], 3)
    jobs += [(off, tgt, "pagerank", {}), (off, tgt, "sssp", {"source": 0})]
    return jobs


def _expected(off, tgt, app, kw):
    n = off.size - 1
    cap = kw.get("max_supersteps", 10_000)
    if app == "components":
        return O.run_cc(n, off, tgt, max_steps=cap)
    if app == "sssp":
        return O.run_sssp(n, off, tgt, kw["source"], cap)
    return O.run_pagerank(n, off, tgt, kw.get("iterations", 10), kw.get("damping", 0.85),
                          max_steps=cap)


@pytest.mark.parametrize("world,exchange", [(2, "hybrid"), (3, "hybrid"), (2, "dense"),
                                            (2, "peer"), (3, "peer"), (2, "auto"),
                                            (3, "auto")])
def test_partitioned_run_matches_oracle(world, exchange, tmp_path):
    jobs = _jobs()
    mp.start_processes(_worker, args=(world, _free_port(), jobs, str(tmp_path), exchange),
                       nprocs=world, start_method="spawn")
    results = torch.load(os.path.join(tmp_path, "results.pt"), weights_only=False)
    modes = set()
    for (off, tgt, app, kw), (vals, stats, hit, ex) in zip(jobs, results):
        modes.update(m for m in ex if m)
        want = _expected(off, tgt, app, kw)
        if app == "pagerank":
            assert np.max(np.abs(vals - want.values) / np.abs(want.values)) <= 1e-9
        else:
            assert np.array_equal(vals.astype(np.int64), want.values.astype(np.int64)), (app, kw)
        assert [a for a, _ in stats] == want.active_counts, (app, kw)
        assert [m for _, m in stats] == want.messages_sent, (app, kw)
        assert hit == want.hit_superstep_cap
    # hybrid: both collective exchanges ran (sparse on the late supersteps);
    # peer: the min programs never reduce the mailbox (PageRank records none)
    # auto: the dense collective for the big supersteps, the peer exchange
    # for the rest (every transition between the two is exercised)
    if exchange == "auto":
        assert {"dense", "peer"} <= modes <= {"dense", "sparse", "peer"}
    else:
        assert modes == {"hybrid": {"dense", "sparse"}, "dense": {"dense"},
                         "peer": {"peer"}}[exchange]


def test_partition_bounds_edge_balanced():
    deg = np.array([50, 1, 1, 1, 1, 1, 1, 1, 1, 40])
    b = partition_bounds(deg, 2)
    assert b[0] == 0 and b[-1] == deg.size
    total = int((deg + 1).sum())
    for r in range(2):
        load = int((deg[b[r]:b[r + 1]] + 1).sum())
        assert load * 2 < total + int((deg + 1).max()) * 2


def test_owner_blocked_layout():
    """Padded owner blocks: block = the largest range rounded up to 64;
    vertex v of owner r sits at r * B + (v - lo_r); positions are ordered
    like the vertices and never land in a block's padding."""
    from paper_2010_01542_b200.distributed import owner_block, padded_positions
    bounds = np.array([0, 70, 75, 200], dtype=np.int64)
    B = owner_block(bounds)
    assert B == 128 and B % 64 == 0
    v = torch.arange(200, dtype=torch.int32)
    pos = padded_positions(v, bounds, B, chunk=17).numpy()
    owner = np.searchsorted(bounds[1:-1], np.arange(200), side="right")
    assert np.array_equal(pos, owner * B + np.arange(200) - bounds[owner])
    assert np.all(np.diff(pos) > 0)
    sizes = np.diff(bounds)
    assert np.all(pos - owner * B < sizes[owner])
    assert owner_block(np.array([0, 0, 0])) == 64       # empty graph: one line
