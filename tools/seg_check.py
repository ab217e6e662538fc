"""Segmented scatter vs K1 on BASELINE configs: identical values and
per-superstep statistics, and the device time of both (probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3"]
thr = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256]
for c in cfgs:
    g = rmat_graph(c)
    app = {"C2": "components", "C3": "sssp", "C5": "components"}[c]
    prog = pgx.connected_components() if app == "components" else pgx.sssp(int(torch.argmax(g.out_degrees)))
    res = {}
    for mode in ["off"] + [f"on{t}" for t in thr]:
        if mode.startswith("on"):
            _lib.set_option(_lib.PGX_OPT_SEG_MIN_EDGES, int(mode[2:]))
        t0 = time.time()
        plan = pgx.plan_run(g, prog, pgx.EngineConfig(segments="off" if mode == "off" else "on"))
        torch.cuda.synchronize()
        tprep = time.time() - t0
        best = None
        for r in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(plan.stream); plan.launch(); b.record(plan.stream); torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            rep = pgx.collect(plan, prog)
            if best is None or ms < best[0]:
                best = (ms, rep)
        ms, rep = best
        E = sum(s.edges for s in rep.supersteps)
        st = plan.stats.cpu().numpy()
        res[mode] = rep
        print(f"{c} {mode}: {ms:.3f} ms  GTEPS={E/ms/1e6:.1f}  prep={tprep:.3f}s", flush=True)
        for x in rep.supersteps:
            row = st[4 + 8 * x.index: 4 + 8 * x.index + 8]
            print(f"   s{x.index}: {x.seconds*1e6:9.1f} us (scatter {(row[5]-row[7])*1e-3:8.1f}) "
                  f"act={x.active_count} F={x.broadcasters} E={x.edges} R={x.recipients}")
        del plan
    base = res["off"]
    for k, rep in res.items():
        same = (rep.values == base.values).all() and \
            [(s.active_count, s.messages_sent, s.edges, s.recipients) for s in rep.supersteps] == \
            [(s.active_count, s.messages_sent, s.edges, s.recipients) for s in base.supersteps]
        print(f"{c} {k}: identical to K1 = {bool(same)}", flush=True)
    _lib.set_option(_lib.PGX_OPT_SEG_MIN_EDGES, 256)
    del g
    torch.cuda.empty_cache()
