"""B200 ablation grid mirroring the reference harness's grid_variants
(harness.py:273-292: baseline, then each optimisation alone, then all):

  layout     interleaved {mailbox, value} records  ->  externalised SoA
  combiner   lock-style CAS retry per message       ->  hybrid (read-filter + red.min)
  scheduler  one thread per sender                  ->  edge-balanced 256-edge warp tiles

Every arm must reproduce the shipped arm's values and per-superstep counts.
Writes profiles/ablation_<tag>.json and prints a markdown table.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

IL, EX = _lib.PGX_LAYOUT_INTERLEAVED, _lib.PGX_LAYOUT_EXTERNALISED
ARMS = [  # name, read_filter, cas_loop, vertex_sched, layout
    ("baseline (interleaved, vertex-per-thread, CAS loop)", 0, 1, 1, IL),
    ("+ hybrid combiner only", 1, 0, 1, IL),
    ("+ externalised layout only", 0, 1, 1, EX),
    ("+ edge-balanced tiles only", 0, 1, 0, IL),
    ("final (externalised + edge tiles + hybrid)", 1, 0, 0, EX),
    ("final with the interleaved layout", 1, 0, 0, IL),
    ("final, red.min without read-filter", 0, 0, 0, EX),
    ("final, K1 only (no segmented scatter)", 1, 0, 0, EX, "off"),
]
FINAL = 4


def set_arm(rf, cas, vs, layout, segments="auto"):
    _lib.set_option(_lib.PGX_OPT_READ_FILTER, rf)
    _lib.set_option(_lib.PGX_OPT_CAS_LOOP, cas)
    _lib.set_option(_lib.PGX_OPT_VERTEX_SCHED, vs)
    _lib.set_option(_lib.PGX_OPT_LAYOUT, layout)


def time_plan(plan, prog, reps):
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(plan.stream); plan.launch(); b.record(plan.stream); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms)), pgx.collect(plan, prog)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "arms": [a[0] for a in ARMS], "results": []}
    rows = []
    for cfg in ("C2", "C3"):
        g = rmat_graph(cfg)
        prog = pgx.connected_components() if cfg == "C2" else pgx.sssp(int(torch.argmax(g.out_degrees)))
        ref = None
        res = {}
        order = [ARMS[FINAL]] + [a for i, a in enumerate(ARMS) if i != FINAL]
        for name, *opts in order:   # final first: the reference arm
            set_arm(*opts)
            seg = opts[4] if len(opts) > 4 else "auto"
            plan = pgx.plan_run(g, prog, pgx.EngineConfig(segments=seg))
            ms, rep = time_plan(plan, prog, reps)
            if ref is None:
                ref = rep
            same = np.array_equal(rep.values, ref.values) and \
                [s.active_count for s in rep.supersteps] == [s.active_count for s in ref.supersteps]
            E = sum(s.edges for s in rep.supersteps)
            res[name] = {"ms": round(ms, 3), "GTEPS": round(E / ms / 1e6, 2), "identical": bool(same)}
            print(cfg, name, res[name], flush=True)
        set_arm(*ARMS[FINAL][1:])
        base = res[ARMS[0][0]]["ms"]
        for name, *_ in ARMS:
            res[name]["speedup_vs_baseline"] = round(base / res[name]["ms"], 2)
        out["results"].append({"config": cfg, "app": "components" if cfg == "C2" else "sssp", "arms": res})
        rows.append((cfg, res))
        del g
        torch.cuda.empty_cache()
    # PageRank: the paper's PR is pull; push (red.add.f64) as the alternative
    g = rmat_graph("C4")
    res = {}
    for mode in ("push", "pull"):
        plan = pgx.plan_run(g, pgx.pagerank(), pgx.EngineConfig(pagerank_mode=mode))
        ms, rep = time_plan(plan, pgx.pagerank(), reps)
        res[mode] = {"ms": round(ms, 3), "GTEPS": round(10 * g.edge_count / ms / 1e6, 2)}
        print("C4", mode, res[mode], flush=True)
    out["results"].append({"config": "C4", "app": "pagerank", "arms": res})
    for d in ("profiles", "gpurun_out"):
        os.makedirs(d, exist_ok=True)
        json.dump(out, open(f"{d}/ablation_{tag}.json", "w"), indent=1)
    print("\n| arm | " + " | ".join(f"{c} ms (x)" for c, _ in rows) + " |")
    print("|---|" + "---|" * len(rows))
    for name, *_ in ARMS:
        print(f"| {name} | " + " | ".join(f"{r[name]['ms']} ({r[name]['speedup_vs_baseline']}x)"
                                          + ("" if r[name]["identical"] else " MISMATCH")
                                          for _, r in rows) + " |")


if __name__ == "__main__":
    main()
