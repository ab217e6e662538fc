"""Input side of the path on the GPU box: from_edges (CSR build on the
device) for C2 / C4 edge lists, and load_cache of the C2 snapshot (host,
pinned + device).  The reference's host build took 47 s (C2) and 112 s
(C4) in the survey."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = fn(); torch.cuda.synchronize()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return r, best


for cfg, und in (("C2", True), ("C4", False)):
    g = rmat_graph(cfg)
    off = g.out_offsets
    src = torch.repeat_interleave(torch.arange(g.vertex_count, device=off.device), torch.diff(off))
    dst = g.out_targets.to(torch.int64)
    if und:  # the stored graph is symmetric: feed one direction, rebuild both
        keep = src < dst
        src, dst = src[keep], dst[keep]
    h, t = timed(lambda: pgx.from_edges(src, dst, g.vertex_count, undirected=und))
    same = torch.equal(h.out_offsets, g.out_offsets) and torch.equal(h.out_targets, g.out_targets)
    print(f"{cfg}: from_edges on the GPU, {src.numel()} input edges -> m={h.edge_count}: "
          f"{t*1e3:.1f} ms (CSR identical to the generator's: {same})")
    if cfg == "C2":
        d = tempfile.mkdtemp()
        p = os.path.join(d, "c2.pglcsr")
        g.in_offsets  # build the in-CSR once before saving
        pgx.save_cache(g, p)
        sz = os.path.getsize(p)
        _, t1 = timed(lambda: pgx.load_cache(p))
        _, t2 = timed(lambda: pgx.load_cache(p, device="cuda"))
        print(f"C2 load_cache ({sz/1e6:.0f} MB, page cache warm): host {t1*1e3:.0f} ms, "
              f"pinned + device {t2*1e3:.0f} ms")
        os.unlink(p)
    del g, h, src, dst
    torch.cuda.empty_cache()
