"""Share of in-edges whose source is among the top-K out-degree vertices
(what an L1 / shared-memory cache of hot shares could serve in the
PageRank pull fold), and the segmented index's edges per entry at several
segment sizes.  usage: hub_share.py C4,C2  -> profiles/hub_share_r2.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle as O

out = {}
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C4,C2").split(","):
    n, off, tgt = O.rmat_csr(O.CONFIGS[cfg])
    m = tgt.size
    deg = np.diff(off)
    top = np.cumsum(np.sort(deg)[::-1])
    row = {"top_k_out_degree_share": {str(k): round(float(top[k - 1] / m), 4)
                                      for k in (2048, 4096, 8192, 16384)}}
    starts = np.zeros(m, bool)
    starts[off[:-1][deg > 0]] = True
    epe = {}
    for L in (12, 13, 14, 15):
        key = tgt >> L
        ch = np.empty(m, bool)
        ch[0] = True
        ch[1:] = key[1:] != key[:-1]
        epe[str(L)] = round(m / float((ch | starts).sum()), 3)
    row["edges_per_entry_by_seg_log2"] = epe
    out[cfg] = row
    print(cfg, row, flush=True)
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                 "hub_share_r2.json"), "w"), indent=1)
