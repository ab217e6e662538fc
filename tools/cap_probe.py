"""One device run of a BASELINE config with a superstep cap (ncu target:
profile the first supersteps alone).  usage: cap_probe.py C5 1 [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph

cfg, cap = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = rmat_graph(cfg)
app = {"C2": "components", "C3": "sssp", "C5": "components"}[cfg]
prog = pgx.connected_components() if app == "components" else \
    pgx.sssp(int(torch.argmax(g.out_degrees)))
plan = pgx.plan_run(g, prog, pgx.EngineConfig(max_supersteps=cap))
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(plan.stream); plan.launch(); b.record(plan.stream); torch.cuda.synchronize()
    rep = pgx.collect(plan, prog)
    print(f"{cfg} cap={cap}: {a.elapsed_time(b):.3f} ms, steps={rep.superstep_count}, "
          f"per-step us={[round(s.seconds * 1e6, 1) for s in rep.supersteps]}", flush=True)
