"""Pull PageRank with the shared-memory hub-source table: time a config for
several table sizes (0 = the plain fold) and check the ranks are
bit-identical.  usage: pr_hub_probe.py C4 0,4096,8192,16384,20480"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
Ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,4096,8192,16384,20480").split(",")]
g = rmat_graph(cfg)
prog = pgx.pagerank(10, 0.85)
ref = None
for K in Ks:
    conf = pgx.EngineConfig(pagerank_hubs="off" if K == 0 else "on")
    csr = g.device_csr(torch.device("cuda", 0))
    csr.pr_hub_col = csr.pr_hub_slot = None
    csr.pr_nhubs = 0
    if K:
        os.environ["PGX_PR_HUBS"] = str(K)
    plan = pgx.plan_run(g, prog, conf)
    ms = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(plan.stream); plan.launch(); b.record(plan.stream); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    rep = pgx.collect(plan, prog)
    if ref is None:
        ref = rep.values.copy()
    same = bool(np.array_equal(rep.values, ref))
    E = sum(x.edges for x in rep.supersteps)
    print(f"{cfg} hubs={K} (used {csr.pr_nhubs}): median {np.median(ms):.3f} ms, "
          f"min {min(ms):.3f} ms, {E / np.median(ms) / 1e6:.1f} GTEPS, identical={same}", flush=True)
