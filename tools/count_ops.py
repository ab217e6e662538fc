"""Operation mix of the scatter (debug build): red.min and has-bit red.or
per edge on full C2 / C3 runs.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \\
         -shared -Iinclude -DPGX_COUNT_OPS=1 paper_2010_01542_b200/csrc/*.cu \\
         -o exp/dbg_count.so
    python tools/count_ops.py C2,C3
"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PGX_LIB"] = os.environ.get("PGX_LIB", "exp/dbg_count.so")
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph
lib = _lib.load()
lib.pgx_debug_counts.argtypes = [ctypes.c_void_p]
out = (ctypes.c_ulonglong * 3)()
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C2,C3").split(","):
    g = rmat_graph(cfg)
    prog = pgx.connected_components() if cfg in ("C2", "C5") else \
        pgx.sssp(int(torch.argmax(g.out_degrees)))
    plan = pgx.plan_run(g, prog)
    lib.pgx_debug_counts(out)                      # reset
    plan.launch(); torch.cuda.synchronize()
    lib.pgx_debug_counts(out)
    rep = pgx.collect(plan, prog)
    E = sum(s.edges for s in rep.supersteps)
    R = sum(s.recipients for s in rep.supersteps)
    print(f"{cfg}: edges={out[2]} (stats {E})  red.min={out[0]} ({out[0]/max(out[2],1):.4f}/edge)  "
          f"has-bit red.or={out[1]} ({out[1]/max(out[2],1):.4f}/edge)  recipients={R}")
