import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PGX_LIB"] = "exp/dbg_count.so"
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph
lib = _lib.load()
lib.pgx_debug_counts.argtypes = [ctypes.c_void_p]
out = (ctypes.c_ulonglong * 3)()
for cfg in sys.argv[1].split(","):
    g = rmat_graph(cfg)
    prog = pgx.connected_components() if cfg == "C2" else pgx.sssp(int(torch.argmax(g.out_degrees)))
    plan = pgx.plan_run(g, prog)
    lib.pgx_debug_counts(out)
    plan.launch(); torch.cuda.synchronize()
    lib.pgx_debug_counts(out)
    rep = pgx.collect(plan, prog)
    E = sum(s.edges for s in rep.supersteps)
    print(cfg, f"edges={out[2]} (stats {E}) reds={out[0]} ({out[0]/out[2]:.3f}/edge) bit-reds={out[1]} recipients={sum(s.recipients for s in rep.supersteps)}")
