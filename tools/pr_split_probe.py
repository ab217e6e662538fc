"""Fold / compute split of the pull PageRank kernel per superstep (needs a
build with -DPGX_PR_FOLD_STAMP=1: tools/build_variant.sh stamp
-DPGX_PR_FOLD_STAMP=1; PGX_LIB=ab/libpgx_stamp.so).  usage: pr_split_probe.py C4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
g = rmat_graph(cfg)
prog = pgx.pagerank(10, 0.85)
plan = pgx.plan_run(g, prog)
for _ in range(3):
    plan.launch()
torch.cuda.synchronize()
k = 10
st = plan.stats[_lib.PGX_STAT_HDR:_lib.PGX_STAT_HDR + k * _lib.PGX_STAT_FIELDS]
st = st.view(k, _lib.PGX_STAT_FIELDS).cpu().numpy().astype(np.int64)
for s in range(k):
    fold = (st[s, 6] - st[s, 7]) * 1e-3
    comp = (st[s, 5] - st[s, 6]) * 1e-3
    print(f"{cfg} s{s}: fold {fold:7.1f} us  compute+reduce {comp:6.1f} us")
