"""Pin the CPU oracle before trusting it (CPU only).

* numpy rounding orders reproduced exactly (the reference folds PageRank
  with ``np.add.reduceat`` and sums dangling mass with ``ndarray.sum``);
* the SURVEY 8(d) R-MAT generator reproduces BASELINE.md section 3's CSR
  SHA-256 values;
* the engine restatement reproduces every reference run recorded in
  tests/golden (values bit-for-bit -- PageRank included -- superstep
  counts, cap flag, per-superstep active and message counts);
* at C2/C3 size it reproduces BASELINE.md's label / distance hashes and
  per-superstep counts (taken from the reference engine on those inputs).
"""

import hashlib
import os
import sys

import numpy as np
import pytest

from golden_cases import DANGLING_RANKS, PATH3_RANKS, load_runs
from oracle import oracle as O

RUNS = load_runs()


def sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def oracle_run(r, threads=0):
    off, tgt = O.csr_from_edges(r.src, r.dst, r.n, r.undirected)
    kw = dict(r.kwargs)
    cap = kw.pop("max_supersteps", 10_000)
    if r.app == "sssp":
        return O.run_sssp(r.n, off, tgt, kw["source"], cap, threads)
    if r.app == "components":
        return O.run_cc(r.n, off, tgt, max_steps=cap, threads=threads)
    return O.run_pagerank(r.n, off, tgt, kw.get("iterations", 10),
                          kw.get("damping", 0.85), max_steps=cap,
                          threads=threads)


def test_numpy_rounding_orders():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 1500))
        a = rng.random(n) * rng.random(n) ** 5
        assert O.np_sum(a) == float(a.sum())
        assert O.np_reduceat_segment(a) == float(np.add.reduceat(a, [0])[0])


def test_splitmix64_known_values():
    # SplitMix64 with state 0: first output of the canonical generator
    assert O.lib().orc_splitmix64(0) == 0xE220A8397B1DCDAF


def test_rmat_c1_matches_baseline_hashes():
    n, off, tgt = O.rmat_csr(O.CONFIGS["C1"])
    assert (n, tgt.size) == (65_536, 955_890)
    assert sha(off, "<i8") == ("8e2c9c7ecc7087595f3b3d6738c80e0e"
                               "ea0c7f3edb30b9397604cad1b0ebabac")
    assert sha(tgt, "<i4") == ("b920d8fe143abe02a3459674d13419b0"
                               "61340af5008426612925db3b8efaec08")
    deg = np.diff(off)
    assert int((deg == 0).sum()) == 25_091           # dangling
    assert int(np.argmax(deg)) == 0 and int(deg[0]) == 6_259


@pytest.mark.parametrize("r", RUNS, ids=lambda r: r.id)
def test_oracle_engine_matches_reference(r):
    got = oracle_run(r)
    want = r.values
    if r.app == "pagerank":
        # bit-identical: same fold order and rounding as the reference
        assert np.array_equal(got.values.view(np.uint64),
                              want.astype(np.float64).view(np.uint64))
    else:
        assert np.array_equal(got.values.astype(np.int64),
                              want.astype(np.int64))
    assert got.superstep_count == r.superstep_count
    assert got.hit_superstep_cap == r.hit_superstep_cap
    assert got.active_counts == r.active_counts
    assert got.messages_sent == r.messages_sent


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_oracle_thread_invariance(threads):
    for r in RUNS[::7]:
        a = oracle_run(r, threads=1)
        b = oracle_run(r, threads=threads)
        assert np.array_equal(a.values, b.values)
        assert a.active_counts == b.active_counts


def test_reference_golden_constants():
    # tests/test_algorithms.py:27-43 of the reference
    off, tgt = O.csr_from_edges([0, 1], [1, 2], 3, undirected=True)
    got = O.run_pagerank(3, off, tgt).values
    assert np.max(np.abs(got - np.array(PATH3_RANKS))) < 1e-9
    off, tgt = O.csr_from_edges([0, 0, 1], [1, 2, 2], 3)
    got = O.run_pagerank(3, off, tgt).values
    assert np.max(np.abs(got - np.array(DANGLING_RANKS))) < 1e-9
    assert abs(got.sum() - 1.0) < 1e-12
    # tests/test_engine.py:29-37: path-4 SSSP stats
    off, tgt = O.csr_from_edges([0, 1, 2], [1, 2, 3], 4, undirected=True)
    r = O.run_sssp(4, off, tgt, 0)
    assert r.values.tolist() == [0, 1, 2, 3]
    assert r.superstep_count == 5
    assert r.active_counts == [4, 1, 2, 2, 1]
    assert r.messages_sent == [1, 2, 2, 1, 0]


@pytest.mark.parametrize("r", [r for r in RUNS if r.app != "pagerank"
                               and not r.hit_superstep_cap],
                         ids=lambda r: r.id)
def test_validators_agree_with_reference_engine(r):
    off, tgt = O.csr_from_edges(r.src, r.dst, r.n, r.undirected)
    es, ed = O.stored_edges(r.n, off, tgt)
    if r.app == "components" and r.undirected:
        assert np.array_equal(O.components_reference(es, ed, r.n),
                              r.values.astype(np.int64))
    if r.app == "sssp":
        assert np.array_equal(
            O.bfs_distances_reference(es, ed, r.n, r.kwargs["source"]),
            r.values.astype(np.uint32))


@pytest.mark.parametrize("r", [r for r in RUNS if r.app == "pagerank"
                               and not r.hit_superstep_cap and r.n],
                         ids=lambda r: r.id)
def test_pagerank_validator_within_tolerance(r):
    off, tgt = O.csr_from_edges(r.src, r.dst, r.n, r.undirected)
    es, ed = O.stored_edges(r.n, off, tgt)
    ref = O.pagerank_reference(es, ed, r.n, r.kwargs.get("iterations", 10),
                               r.kwargs.get("damping", 0.85))
    assert np.max(np.abs(ref - r.values) / np.abs(r.values)) <= 1e-9


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="reference tree not mounted (GPU box)")
def test_validators_bitwise_vs_live_reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    from pregelite import oracles as ref
    rng = np.random.default_rng(7)
    for _ in range(5):
        n = int(rng.integers(2, 300))
        m = int(rng.integers(0, 4 * n))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        assert np.array_equal(O.components_reference(src, dst, n),
                              ref.components_reference(src, dst, n))
        s = int(rng.integers(0, n))
        assert np.array_equal(O.bfs_distances_reference(src, dst, n, s),
                              ref.bfs_distances_reference(src, dst, n, s))
        a = O.pagerank_reference(src, dst, n)
        b = ref.pagerank_reference(src, dst, n)
        assert np.max(np.abs(a - b) / b) < 1e-13


@pytest.mark.slow
def test_rmat_c2_c3_known_answers():
    """CSR hashes and the reference's outputs."""
    n, off, tgt = O.rmat_csr(O.CONFIGS["C2"])
    assert tgt.size == 65_242_574
    assert sha(off, "<i8").startswith("aa2ac4555df0c0fb")
    assert sha(tgt, "<i4").startswith("ff82f71753fbeba1")
    r = O.run_cc(n, off, tgt)
    assert sha(r.values, "<u4") == ("c4e2cc1d7b5db62b9818e1cd41611649"
                                    "a294c5623d7e29804c175f904c40bf98")
    assert r.active_counts == [4194304, 2009754, 2004276, 1499157, 208894,
                               2173, 23]
    assert r.messages_sent == [4194304, 1816650, 1905145, 269866, 2165, 23, 0]
    assert r.edges == [65242574, 64803511, 28608953, 348075, 2192, 23, 0]
    del off, tgt, r
    n, off, tgt = O.rmat_csr(O.CONFIGS["C3"])
    assert tgt.size == 65_242_824
    assert sha(off, "<i8").startswith("d170d3d509c9a166")
    assert sha(tgt, "<i4").startswith("11f2969e2050ea91")
    r = O.run_sssp(n, off, tgt, int(np.argmax(np.diff(off))))
    assert sha(r.values, "<u4") == ("bd08774026f70bbd29b80c977187f880"
                                    "654c0d8cbd2b42ba0988fed279ffa1e2")
    assert r.active_counts == [4194304, 97364, 1730927, 1490812, 146756,
                               2024, 6]
    assert r.messages_sent == [97364, 36379100, 27861844, 339319, 2142, 6, 0]
