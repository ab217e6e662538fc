import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph
g = rmat_graph("C5")
prog = pgx.connected_components()
for _ in range(2):
    rep = pgx.run(g, prog, pgx.EngineConfig(segments="off"))
print("total", rep.device_seconds * 1e3, "ms")
for s in rep.supersteps:
    print(f"s{s.index}: {s.seconds*1e6:.1f} us edges={s.edges}")
