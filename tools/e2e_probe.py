"""Break down the end-to-end run() from pinned host memory (C2 CC)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200.rmat import rmat_graph

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
g = rmat_graph(cfg)
host = g.pin_memory()
prog = pgx.connected_components() if cfg in ("C2", "C5") else pgx.pagerank() if cfg in ("C1", "C4") \
    else pgx.sssp(int(torch.argmax(g.out_degrees)))
def T():
    torch.cuda.synchronize(); return time.perf_counter()
for it in range(4):
    host.drop_device_cache()
    t0 = T()
    csr = host.device_csr()
    t1 = T()
    plan = pgx.plan_run(host, prog)
    t2 = T()
    plan.launch(); t3 = T()
    rep = pgx.collect(plan, prog); t4 = T()
    host.drop_device_cache()
    t5 = T(); r = pgx.run(host, prog); t6 = T()
    print(f"it{it}: device_csr {1e3*(t1-t0):.2f} ms  plan {1e3*(t2-t1):.2f}  kernel {1e3*(t3-t2):.2f}  "
          f"collect {1e3*(t4-t3):.2f}  | run() total {1e3*(t6-t5):.2f} ms")
# raw H2D bandwidth from pinned
x = host.out_targets
t0 = T(); y = x.to("cuda", non_blocking=True); t1 = T()
print(f"H2D targets {x.numel()*4/1e6:.0f} MB: {1e3*(t1-t0):.2f} ms = {x.numel()*4/(t1-t0)/1e9:.1f} GB/s")
z = torch.empty(g.vertex_count, dtype=torch.int64, pin_memory=True)
d = torch.zeros(g.vertex_count, dtype=torch.int64, device="cuda")
t0 = T(); z.copy_(d, non_blocking=True); t1 = T()
print(f"D2H pinned {g.vertex_count*8/1e6:.0f} MB: {1e3*(t1-t0):.2f} ms")
t0 = T(); w = d.cpu(); t1 = T()
print(f"D2H pageable .cpu() {g.vertex_count*8/1e6:.0f} MB: {1e3*(t1-t0):.2f} ms")
