"""usage: relabel_probe.py C2,C3,C4 in|out|sum
Experiment: does a degree-descending vertex relabelling (hot recipients
packed into few cache lines) speed up the scatter?  Timing only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.graph import Graph
from paper_2010_01542_b200.rmat import rmat_graph


KEY = sys.argv[2] if len(sys.argv) > 2 else "in"   # in | out | sum


def relabel(g):
    n, m = g.vertex_count, g.edge_count
    off = g.out_offsets
    col = g.out_targets.to(torch.int64)
    indeg = torch.bincount(col, minlength=n)
    outdeg = torch.diff(off.to(torch.int64))
    key = {"in": indeg, "out": outdeg, "sum": indeg + outdeg}[KEY]
    order = torch.argsort(-key, stable=True)             # new -> old
    new_id = torch.empty_like(order)
    new_id[order] = torch.arange(n, device=order.device)  # old -> new
    src = torch.repeat_interleave(torch.arange(n, device=off.device), torch.diff(off))
    key = (new_id[src] << 32) | new_id[col]
    key, _ = torch.sort(key)
    s2 = key >> 32
    offs = torch.zeros(n + 1, dtype=torch.int64, device=off.device)
    offs[1:] = torch.cumsum(torch.bincount(s2, minlength=n), 0)
    return Graph(n, offs, (key & 0xFFFFFFFF).to(torch.int32)), new_id


def time_run(g, prog, reps=5):
    plan = pgx.plan_run(g, prog)
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.launch(); b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    rep = pgx.collect(plan, prog)
    return float(np.median(ms)), rep


for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C2,C3,C4").split(","):
    g = rmat_graph(cfg)
    r, new_id = relabel(g)
    if cfg == "C2":
        progs = (pgx.connected_components(), pgx.connected_components())
    elif cfg == "C3":
        s = int(torch.argmax(g.out_degrees))
        progs = (pgx.sssp(s), pgx.sssp(int(new_id[s])))
    else:
        progs = (pgx.pagerank(), pgx.pagerank())
    t0, r0 = time_run(g, progs[0])
    t1, r1 = time_run(r, progs[1])
    E0 = sum(x.edges for x in r0.supersteps); E1 = sum(x.edges for x in r1.supersteps)
    print(f"{cfg}: original {t0:.3f} ms ({E0/t0/1e6:.1f} GTEPS, {r0.superstep_count} steps) | "
          f"relabelled {t1:.3f} ms ({E1/t1/1e6:.1f} GTEPS, {r1.superstep_count} steps)", flush=True)
    if cfg == "C3":
        d0 = r0.values; d1 = r1.values[new_id.cpu().numpy()]
        print("   sssp distances identical after un-permuting:", np.array_equal(d0, d1))
    del g, r
    torch.cuda.empty_cache()
