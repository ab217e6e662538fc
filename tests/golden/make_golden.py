"""Regenerate tests/golden/reference_runs.npz by running the REFERENCE.

Imports the reference package read-only from /root/reference/pkg/src
(pregelite, pure Python) and records, for a fixed list of small graphs,
exactly what ``pregelite.run`` returns: values, superstep_count,
hit_superstep_cap and the per-superstep ``active_count`` /
``messages_sent``.  The GPU box has no /root/reference, so the tests read
only the committed .npz written here.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Graphs: the reference tests' own fixtures (tests/test_algorithms.py:31-184,
tests/test_engine.py:29-98, tests/test_acceptance.py:77-82, 490-511),
seeded random ER / power-law multigraphs (self-loops and duplicates kept,
as ``from_edges`` keeps them), and small R-MAT graphs from the SURVEY 8(d)
generator (the oracle's, whose C1-C3 CSR hashes are pinned to BASELINE.md).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _cases():
    sys.path.insert(0, REF_SRC)
    from pregelite.generate import erdos_renyi_edges, path_edges, power_law_edges

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    cases = []

    def add(name, src, dst, n, undirected, apps):
        cases.append(dict(name=name, src=np.asarray(src, np.int64),
                          dst=np.asarray(dst, np.int64), n=int(n),
                          undirected=bool(undirected), apps=apps))

    all3 = lambda s=0: [("sssp", dict(source=s)), ("components", {}),
                        ("pagerank", {})]
    # reference test fixtures
    add("path4_u", *path_edges(4), 4, True, all3())
    add("path3_u", *path_edges(3), 3, True, all3())
    add("dangling_d", [0, 0, 1], [1, 2, 2], 3, False, all3())
    add("two_edges_u", [0, 2], [1, 3], 4, True, all3())
    add("two_edges_5_u", [0, 2], [1, 3], 5, True, all3())
    add("two_triangles_u", [0, 1, 2, 3, 4, 5], [1, 2, 0, 4, 5, 3], 6, True,
        all3())
    add("isolated_u", [1], [2], 5, True, all3(1))
    add("directed_d", [0, 1, 3], [1, 2, 0], 4, False, all3())
    add("star_u", np.zeros(7, np.int64), np.arange(1, 8), 8, True, all3())
    add("empty4", [], [], 4, False, [("components", {}), ("pagerank", {})])
    add("empty0", [], [], 0, False, [("components", {}), ("pagerank", {})])
    add("single_vertex", [], [], 1, False, all3())
    add("self_loop_dup_d", [0, 0, 0, 1, 2, 2], [0, 1, 1, 2, 2, 0], 3, False,
        all3())
    for n in (2, 5, 7, 12, 30, 64):
        add(f"path{n}_u", *path_edges(n), n, True,
            [("sssp", dict(source=0)), ("sssp", dict(source=n // 2)),
             ("components", {}), ("pagerank", {})])
    add("path12_d", *path_edges(12), 12, False, all3())
    add("path50_u_cap", *path_edges(50), 50, True,
        [("components", dict(max_supersteps=3)),
         ("sssp", dict(source=0, max_supersteps=7)),
         ("pagerank", dict(max_supersteps=4))])
    add("path5_u_prk", *path_edges(5), 5, True,
        [("pagerank", dict(iterations=k)) for k in (1, 2, 3, 7)])
    # seeded random multigraphs
    for seed in range(6):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(5, 400))
        m = int(rng.integers(0, 3 * n))
        gen = power_law_edges if seed % 2 else erdos_renyi_edges
        src, dst = gen(n, m, rng)
        for und in (True, False):
            out_deg = np.bincount(np.concatenate([src, dst]) if und else src,
                                  minlength=n)
            hub = int(np.argmax(out_deg))
            add(f"rand{seed}_{'u' if und else 'd'}", src, dst, n, und,
                [("sssp", dict(source=hub)),
                 ("sssp", dict(source=int(rng.integers(0, n)))),
                 ("components", {}), ("pagerank", {}),
                 ("pagerank", dict(iterations=15, damping=0.7)),
                 ("pagerank", dict(damping=0.0))])
    # small R-MAT graphs from the SURVEY 8(d) generator
    for name, spec in (("rmat12_c1", O.RmatSpec(12, 16, .57, .19, .19, 1, False)),
                       ("rmat12_c2", O.RmatSpec(12, 8, .57, .19, .19, 2, True)),
                       ("rmat12_c4", O.RmatSpec(12, 28, .45, .22, .22, 4, False))):
        n, off, tgt = O.rmat_csr(spec)
        src, dst = O.stored_edges(n, off, tgt)
        hub = int(np.argmax(np.diff(off)))
        add(name, src, dst, n, False,
            [("sssp", dict(source=hub)), ("components", {}),
             ("pagerank", {})])
    return cases


def _run(case, app, kw):
    from pregelite import (EngineConfig, connected_components, from_edges,
                           pagerank, run, sssp)
    g = from_edges(case["src"], case["dst"], case["n"],
                   undirected=case["undirected"])
    kw = dict(kw)
    cap = kw.pop("max_supersteps", None)
    cfg = EngineConfig(max_supersteps=cap) if cap else EngineConfig()
    prog = {"sssp": lambda: sssp(**kw),
            "components": lambda: connected_components(**kw),
            "pagerank": lambda: pagerank(**kw)}[app]()
    rep = run(g, prog, cfg)
    return rep


def main():
    cases = _cases()
    arrays = {}
    manifest = []
    for ci, case in enumerate(cases):
        arrays[f"c{ci}_src"] = case["src"].astype(np.int32)
        arrays[f"c{ci}_dst"] = case["dst"].astype(np.int32)
        entry = dict(name=case["name"], n=case["n"],
                     undirected=case["undirected"], runs=[])
        for ri, (app, kw) in enumerate(case["apps"]):
            rep = _run(case, app, kw)
            key = f"c{ci}_r{ri}"
            arrays[key + "_values"] = np.asarray(rep.values)
            entry["runs"].append(dict(
                app=app, kwargs=kw, key=key,
                superstep_count=rep.superstep_count,
                hit_superstep_cap=bool(rep.hit_superstep_cap),
                active_counts=[s.active_count for s in rep.supersteps],
                messages_sent=[s.messages_sent for s in rep.supersteps]))
        manifest.append(entry)
    np.savez_compressed(os.path.join(HERE, "reference_runs.npz"), **arrays)
    with open(os.path.join(HERE, "reference_runs.json"), "w") as fh:
        json.dump(dict(generator="tests/golden/make_golden.py",
                       reference="/root/reference/pkg (pregelite 0.1.0)",
                       cases=manifest), fh, indent=1)
    print(f"{len(cases)} graphs, "
          f"{sum(len(c['runs']) for c in manifest)} reference runs")


if __name__ == "__main__":
    main()
