"""CPU tests of the pull fold's hub-source encoding (graph.encode_hub_sources,
consumed by pgx_pagerank_pull_hubs_run).  The GPU parity of the encoded
fold is in tests/test_gpu.py (golden modes prhubs / prhubs3,
test_pagerank_hub_table_bit_identical)."""
import numpy as np
import torch

from paper_2010_01542_b200.graph import encode_hub_sources


def _csr(n, src, dst):
    order = np.lexsort((src, dst))            # in-CSR: rows = destinations
    deg_out = np.bincount(src, minlength=n)
    row_ptr = np.zeros(n + 1, np.int32)
    row_ptr[1:] = np.cumsum(deg_out)
    return torch.from_numpy(row_ptr), torch.from_numpy(src[order].astype(np.int32))


def test_top_out_degree_sources_are_encoded():
    rng = np.random.default_rng(7)
    n, m = 500, 6000
    src = (rng.pareto(1.2, m) * 7).astype(np.int64) % n    # skewed out-degrees
    dst = rng.integers(0, n, m)
    row_ptr, in_col = _csr(n, src, dst)
    enc, slot, nh = encode_hub_sources(row_ptr, in_col, 16)
    outdeg = np.diff(row_ptr.numpy())
    assert nh == 16
    hubs = np.flatnonzero(slot.numpy() >= 0)
    # the hubs are 16 vertices of maximal out-degree, slots in descending order
    assert len(hubs) == 16 and outdeg[hubs].min() >= np.sort(outdeg)[-16]
    by_slot = np.empty(16, np.int64)
    by_slot[slot.numpy()[hubs]] = hubs
    assert np.all(np.diff(outdeg[by_slot]) <= 0)
    e, c = enc.numpy(), in_col.numpy()
    is_hub = slot.numpy()[c] >= 0
    assert np.array_equal(e[~is_hub], c[~is_hub])                  # non-hub edges untouched
    assert np.all(e[is_hub] < 0)                                    # bit 31 set
    assert np.array_equal(by_slot[e[is_hub] & 0x7FFFFFFF], c[is_hub])  # decodes to the source


def test_sources_of_one_edge_are_never_hubs_and_capacity_is_respected():
    n = 8
    src = np.array([0, 0, 0, 1, 1, 2, 3, 4])
    dst = np.array([1, 2, 3, 0, 2, 5, 6, 7])
    row_ptr, in_col = _csr(n, src, dst)
    enc, slot, nh = encode_hub_sources(row_ptr, in_col, 100)
    assert nh == 2 and set(np.flatnonzero(slot.numpy() >= 0)) == {0, 1}
    assert slot[0] == 0 and slot[1] == 1                         # out-degree 3 before 2
    enc1, slot1, nh1 = encode_hub_sources(row_ptr, in_col, 1)
    assert nh1 == 1 and int((enc1 < 0).sum()) == 3               # the three edges of vertex 0
