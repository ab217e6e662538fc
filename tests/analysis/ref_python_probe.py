"""The reference package itself (pregelite, installed unmodified into
baseline/_ref) timed on this host: the paper's "final" variant
EngineConfig(workers=1, EXTERNALISED, dynamic(256), HYBRID)
(reference harness.py:288-291), T = RunReport.wall_seconds (excludes setup,
engine.py:258-266), GTEPS = edges traversed by the senders / T, "1
effective core of N" (the engine's worker threads are GIL-bound; BASELINE.md
section 5).  Inputs: the BASELINE configs' CSR (oracle generator, sha-pinned),
handed to pregelite.from_edges as stored edge arrays.

usage: ref_python_probe.py C1:3,C2:1   (config:repeats)"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
import numpy as np
import pregelite as P
from oracle import oracle as O

spec = sys.argv[1] if len(sys.argv) > 1 else "C1:3,C2:1"
out = []
for item in spec.split(","):
    cfg, reps = item.split(":")
    s = O.CONFIGS[cfg]
    n, off, tgt = O.rmat_csr(s)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    t = time.perf_counter()
    # the CSR is already symmetric and deduplicated: build it as directed
    g = P.from_edges(src, tgt.astype(np.int64), n)
    t_build = time.perf_counter() - t
    app = {"C1": "pagerank", "C2": "components", "C3": "sssp", "C4": "pagerank",
           "C5": "components"}[cfg]
    prog = (P.pagerank(10, 0.85) if app == "pagerank" else
            P.connected_components() if app == "components" else
            P.sssp(int(np.argmax(np.diff(off)))))
    ec = P.EngineConfig(workers=1, layout=P.LayoutMode.EXTERNALISED,
                        scheduler=P.SchedulerMode.dynamic(256), combiner=P.CombinerKind.HYBRID)
    # edges traversed by the senders (the GTEPS numerator of both arms)
    edges = sum(O.run_pagerank(n, off, tgt).edges if app == "pagerank" else
                O.run_cc(n, off, tgt, off, tgt).edges if app == "components" else
                O.run_sssp(n, off, tgt, int(np.argmax(np.diff(off)))).edges)
    walls = []
    for _ in range(int(reps)):
        rep = P.run(g, prog, ec)
        walls.append(rep.wall_seconds)
    T = float(np.median(walls))
    row = {"config": cfg, "app": app, "n": n, "m": int(tgt.size), "edges": int(edges),
           "repeats": int(reps), "wall_seconds": [round(w, 3) for w in walls],
           "median_s": round(T, 3), "GTEPS": round(edges / T / 1e9, 6),
           "graph_build_s": round(t_build, 1), "cores": f"1 effective core of {os.cpu_count()}",
           "call": "pregelite.run(g, prog, EngineConfig(workers=1, EXTERNALISED, dynamic(256), HYBRID))"}
    print(json.dumps(row), flush=True)
    out.append(row)
