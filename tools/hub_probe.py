"""PageRank pull fold with hub-aware L1 hints (exp build with bit 31 of an
in-edge = hub source): mark the top-K out-degree sources in the in-CSR and
time C4.  Needs PGX_LIB=exp/libpgx_v13.so.  usage: hub_probe.py C4 0,4096,16384"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
Ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,4096,16384,65536").split(",")]
g = rmat_graph(cfg)
prog = pgx.pagerank(10, 0.85)
plan = pgx.plan_run(g, prog)
csr = plan.csr
base_col = csr.in_col.clone()
deg = torch.diff(csr.row_ptr.to(torch.int64))
order = torch.argsort(deg, descending=True)
ref = None
for K in Ks:
    col = base_col.clone()
    if K > 0:
        hub = torch.zeros(csr.n, dtype=torch.bool, device=col.device)
        hub[order[:K]] = True
        col = torch.where(hub[col.long()], col | (-2 ** 31), col)
    csr.in_col.copy_(col)
    best = None
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(plan.stream); plan.launch(); b.record(plan.stream); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    rep = pgx.collect(plan, prog)
    if ref is None:
        ref = rep.values.copy()
    same = bool((rep.values == ref).all())
    print(f"{cfg} K={K}: {best:.3f} ms  identical={same}", flush=True)
