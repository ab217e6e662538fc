"""Every ablation arm of the min engine computes the reference's answer.

The arms mirror the reference harness's grid (harness.py:273-292: layout
interleaved vs externalised, combiner lock vs hybrid, scheduler static vs
edge-balanced) and are selected through pgx_set_option.  Each arm must
reproduce the recorded reference runs (values, superstep counts, per-step
active / message counts) and, at full size, BASELINE.md's C2 labels and C3
distances hashes -- an A/B number is only meaningful if both arms compute
the same thing.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from golden_cases import load_runs
from paper_2010_01542_b200 import _lib
from paper_2010_01542_b200.rmat import rmat_graph

pytestmark = pytest.mark.gpu

IL, EX = _lib.PGX_LAYOUT_INTERLEAVED, _lib.PGX_LAYOUT_EXTERNALISED
ARMS = {  # read_filter, cas_loop, vertex_sched, layout
    "baseline": (0, 1, 1, IL),
    "hybrid_only": (1, 0, 1, IL),
    "externalised_only": (0, 1, 1, EX),
    "edge_tiles_only": (0, 1, 0, IL),
    "final_interleaved": (1, 0, 0, IL),
    "final_no_filter": (0, 0, 0, EX),
}
SHIPPED = (1, 0, 0, EX)
MIN_RUNS = [r for r in load_runs() if r.app != "pagerank"]


def set_arm(rf, cas, vs, layout):
    _lib.set_option(_lib.PGX_OPT_READ_FILTER, rf)
    _lib.set_option(_lib.PGX_OPT_CAS_LOOP, cas)
    _lib.set_option(_lib.PGX_OPT_VERTEX_SCHED, vs)
    _lib.set_option(_lib.PGX_OPT_LAYOUT, layout)


@pytest.fixture(params=list(ARMS), ids=list(ARMS))
def arm(request):
    set_arm(*ARMS[request.param])
    yield request.param
    set_arm(*SHIPPED)


def program(app, kw):
    kw = dict(kw)
    kw.pop("max_supersteps", None)
    return pgx.sssp(**kw) if app == "sssp" else pgx.connected_components(**kw)


@pytest.mark.parametrize("r", MIN_RUNS, ids=lambda r: r.id)
def test_arm_matches_reference_runs(arm, r):
    g = pgx.from_edges(r.src, r.dst, r.n, undirected=r.undirected, device="cuda")
    cap = r.kwargs.get("max_supersteps")
    cfg = pgx.EngineConfig(max_supersteps=cap if cap else pgx.DEFAULT_MAX_SUPERSTEPS)
    rep = pgx.run(g, program(r.app, r.kwargs), cfg)
    assert np.array_equal(rep.values, r.values)
    assert rep.superstep_count == r.superstep_count
    assert rep.hit_superstep_cap == r.hit_superstep_cap
    assert [s.active_count for s in rep.supersteps] == r.active_counts
    assert [s.messages_sent for s in rep.supersteps] == r.messages_sent


@pytest.fixture(scope="module")
def c2c3():
    return {"C2": rmat_graph("C2"), "C3": rmat_graph("C3")}


def test_arm_full_size_known_answers(arm, c2c3):
    g = c2c3["C2"]
    rep = pgx.run(g, pgx.connected_components())
    assert hashlib.sha256(rep.values.astype("<u4").tobytes()).hexdigest() == \
        "c4e2cc1d7b5db62b9818e1cd41611649a294c5623d7e29804c175f904c40bf98"
    assert [s.active_count for s in rep.supersteps] == \
        [4194304, 2009754, 2004276, 1499157, 208894, 2173, 23]
    g = c2c3["C3"]
    rep = pgx.run(g, pgx.sssp(0))
    assert hashlib.sha256(rep.values.astype("<u4").tobytes()).hexdigest() == \
        "bd08774026f70bbd29b80c977187f880654c0d8cbd2b42ba0988fed279ffa1e2"
    assert [s.messages_sent for s in rep.supersteps] == \
        [97364, 36379100, 27861844, 339319, 2142, 6, 0]
