"""Segmented scatter variants vs K1 on BASELINE configs: identical values
and per-superstep statistics, and the device time of each (probe).

usage: seg_check.py C2,C5 [variant ...]
  variant = comma-separated key=value: L=<seg_log2>, min=<PGX_OPT_SEG_MIN_EDGES>,
"off" = K1 only.  Default: off and the
            shipped options."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3"]
variants = sys.argv[2:] or ["off", "shipped"]
OPTS = {"min": _lib.PGX_OPT_SEG_MIN_EDGES, "pred": _lib.PGX_OPT_SEG_PREDICT}
DEFAULTS = {"min": 256, "pred": 1}
for c in cfgs:
    g = rmat_graph(c)
    app = {"C2": "components", "C3": "sssp", "C5": "components", "C5S": "components"}[c]
    prog = pgx.connected_components() if app == "components" else pgx.sssp(int(torch.argmax(g.out_degrees)))
    res = {}
    for var in variants:
        kv = dict(x.split("=") for x in var.split(",") if "=" in x)
        for k, o in OPTS.items():
            _lib.set_option(o, int(kv.get(k, DEFAULTS[k])))
        L = int(kv.get("L", _lib.PGX_SEG_LOG2_DEFAULT))
        csr = g.device_csr()
        if var != "off" and csr.seg is not None and csr.seg.seg_log2 != L:
            csr.seg, csr.seg_arrays = None, ()
        t0 = time.time()
        if var != "off":
            csr.ensure_segments(seg_log2=L)
        plan = pgx.plan_run(g, prog, pgx.EngineConfig(segments="off" if var == "off" else "on"))
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
        res[var] = rep
        print(f"{c} {var}: {ms:.3f} ms  GTEPS={E/ms/1e6:.1f}  prep={tprep:.3f}s ctas={rep.ctas}",
              flush=True)
        for x in rep.supersteps:
            row = st[4 + 8 * x.index: 4 + 8 * x.index + 8]
            print(f"   s{x.index}: {x.seconds*1e6:9.1f} us (scatter {(row[5]-row[7])*1e-3:8.1f}) "
                  f"act={x.active_count} F={x.broadcasters} E={x.edges} R={x.recipients}")
        del plan
    base = res[variants[0]]
    for k, rep in res.items():
        same = (rep.values == base.values).all() and \
            [(s.active_count, s.messages_sent, s.edges, s.recipients) for s in rep.supersteps] == \
            [(s.active_count, s.messages_sent, s.edges, s.recipients) for s in base.supersteps]
        print(f"{c} {k}: identical to {variants[0]} = {bool(same)}", flush=True)
    for k, o in OPTS.items():
        _lib.set_option(o, DEFAULTS[k])
    del g
    torch.cuda.empty_cache()
