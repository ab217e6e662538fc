"""Regenerate tests/golden/reference_cache_*.pglcsr with the REFERENCE.

Imports pregelite read-only from /root/reference/pkg/src and writes its own
binary CSR snapshots (``save_cache``, graph.py:298-322) of small graphs --
duplicates and self-loops, an undirected graph, an edge-list file with
sparse ids (``load_edge_list`` -> id_map), int64 ids and an empty graph --
plus a JSON manifest of their CSR arrays.  tests/test_api.py checks that
``load_cache`` reads these files and that ``save_cache`` reproduces them
byte for byte.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cache_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import pregelite as P
    from pregelite.graph import load_edge_list, save_cache

    graphs = {
        "dup_loops_d": P.from_edges([0, 0, 0, 1, 2, 2, 4], [0, 1, 1, 2, 2, 0, 1], 5),
        "tri_tail_u": P.from_edges([0, 1, 2, 3], [1, 2, 0, 4], 6, undirected=True),
        "ids64_d": P.from_edges([3, 1, 2, 0], [0, 0, 3, 2], 4, id_dtype=np.int64),
        "empty3": P.from_edges([], [], 3),
    }
    with tempfile.TemporaryDirectory() as td:
        el = os.path.join(td, "edges.txt")
        with open(el, "w") as fh:
            fh.write("# sparse ids\n1000 7\n7 42\n42 1000\n99 7\n")
        graphs["edgelist_idmap_u"] = load_edge_list(el, undirected=True)
    manifest = {}
    for name, g in graphs.items():
        save_cache(g, os.path.join(HERE, f"reference_cache_{name}.pglcsr"))
        manifest[name] = dict(
            n=int(g.vertex_count), m=int(g.edge_count), id_dtype=str(g.id_dtype),
            out_offsets=g.out_offsets.tolist(), out_targets=g.out_targets.tolist(),
            in_offsets=g.in_offsets.tolist(), in_targets=g.in_targets.tolist(),
            id_map=None if g.id_map is None else g.id_map.tolist())
    with open(os.path.join(HERE, "reference_cache.json"), "w") as fh:
        json.dump(dict(generator="tests/golden/make_cache_golden.py",
                       reference="/root/reference/pkg (pregelite 0.1.0)",
                       graphs=manifest), fh, indent=1)
    print(len(graphs), "reference caches")


if __name__ == "__main__":
    main()
