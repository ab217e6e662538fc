"""The fused peer exchange across PROCESSES: CUDA IPC mailboxes.

Two ranks run as separate processes (gloo process group for the small
collectives) on the one GPU of the test box; each maps the other's mailbox
with pgx_peer_open (cudaIpcOpenMemHandle) and pgx_scatter_peer combines
foreign messages straight into it -- the code path torchrun uses on an
NVLink / NVSwitch node, where the mapping crosses GPUs.  No kernel waits on
another rank: ranks synchronise only through host collectives.  Results
must equal the oracle's: labels / distances exact, per-superstep counts
exact; runs forced to "peer" use it in every superstep, "auto" runs mix it
with the dense collective.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SPEC = O.RmatSpec(15, 8, .57, .19, .19, 41, True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    import paper_2010_01542_b200 as pgx
    from paper_2010_01542_b200.distributed import (CudaBackend, PartitionedRun,
                                                   partition_bounds)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    n, off, tgt = O.rmat_csr(SPEC)
    g = pgx.from_csr(torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda())
    bounds = partition_bounds(np.diff(off), world)
    be = CudaBackend(g, int(bounds[rank]), int(bounds[rank + 1]), "cuda:0")
    out = {}
    src = int(np.argmax(np.diff(off)))
    for ex, app, kw in (("peer", "components", {}), ("peer", "sssp", {"source": src}),
                        ("peer", "components", {"max_supersteps": 3}),
                        ("auto", "components", {}), ("auto", "sssp", {"source": src})):
        be2 = be if ex == "peer" else CudaBackend(g, int(bounds[rank]), int(bounds[rank + 1]),
                                                  "cuda:0")
        run = PartitionedRun(be2, dist, bounds, n, int(tgt.size))
        run.exchange = ex
        vals, stats, hit, _ = run.run_min(app, kw.get("source", 0),
                                          kw.get("max_supersteps", 10_000))
        out[(ex, app, kw.get("max_supersteps"))] = (
            vals.cpu().numpy().view(np.uint32).astype(np.int64),
            [s["active_count"] for s in stats], [s["messages_sent"] for s in stats],
            hit, {s["exchange"] for s in stats}, len(be._opened))
    # the public API under the same process group (run() -> run_partitioned)
    rep = pgx.run(g, pgx.connected_components())
    out["api"] = rep.values
    if rank == 0:
        torch.save(out, os.path.join(out_dir, "peer.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_exchange_across_processes(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    out = torch.load(os.path.join(tmp_path, "peer.pt"), weights_only=False)
    n, off, tgt = O.rmat_csr(SPEC)
    src = int(np.argmax(np.diff(off)))
    for (ex, app, cap), (vals, active, sent, hit, modes, opened) in (
            (k, v) for k, v in out.items() if k != "api"):
        want = (O.run_cc(n, off, tgt, max_steps=cap or 10_000) if app == "components"
                else O.run_sssp(n, off, tgt, src))
        assert np.array_equal(vals, want.values.astype(np.int64)), app
        assert active == want.active_counts, app
        assert sent == want.messages_sent, app
        assert hit == want.hit_superstep_cap
        if ex == "peer":
            assert modes == {"peer"}
        else:  # dense collective for the big supersteps, peer for the tail
            assert "peer" in modes and modes <= {"dense", "sparse", "peer"}
        # the other rank's mailbox and has-bitmap came through IPC
        assert opened == 2 * (world - 1)
    assert np.array_equal(out["api"], O.run_cc(n, off, tgt).values.astype(np.int64))
