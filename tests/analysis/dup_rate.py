"""How often a warp's 32-edge round holds duplicate destinations (the only
messages a warp-aggregated combine -- __match_any_sync + __reduce_min_sync /
a shuffle sum -- can remove before the atomic).  Rounds = 32 consecutive
edges of the dense superstep's edge space (the CSR order every K1 tile and
the PR push arm walk).  Reports the fraction of edges whose destination
already occurs earlier in the same round, and the mean distinct
destinations per round.  usage: dup_rate.py C2,C4"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle as O

out = {}
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "C2,C4").split(","):
    n, off, tgt = O.rmat_csr(O.CONFIGS[cfg])
    m = tgt.size - tgt.size % 32
    r = tgt[:m].reshape(-1, 32).astype(np.int64)
    s = np.sort(r, axis=1)
    dup = (s[:, 1:] == s[:, :-1]).sum()
    distinct = 32 - (s[:, 1:] == s[:, :-1]).sum(axis=1)
    rounds_with_dup = int(((s[:, 1:] == s[:, :-1]).any(axis=1)).sum())
    out[cfg] = {"edges": int(m), "duplicate_fraction": round(float(dup) / m, 5),
                "mean_distinct_per_round": round(float(distinct.mean()), 3),
                "rounds_with_a_duplicate": round(rounds_with_dup / r.shape[0], 5)}
    print(cfg, out[cfg], flush=True)
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                 "dup_rate_r2.json"), "w"), indent=1)
