"""The reference's host-side storage / combiner / scheduler contract
(layout.py, mailbox.py, scheduler.py of pregelite): same names, same
semantics, same errors -- and, on the GPU, the device combine reproduces
the hybrid strategy applied message by message."""

import threading

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib

MODES = [pgx.LayoutMode.INTERLEAVED, pgx.LayoutMode.EXTERNALISED]
STRATEGIES = [pgx.send_lock, pgx.send_cas, pgx.send_hybrid]


# ---- layout ------------------------------------------------------------

def test_record_dtypes_are_packed():
    assert pgx.hot_dtype(np.float64).itemsize == 9
    assert pgx.hot_dtype(np.uint32).itemsize == 5
    assert pgx.cold_dtype(np.int64).itemsize == 9
    assert pgx.hot_dtype(np.int64).names == ("flag", "msg")
    assert pgx.cold_dtype(np.uint32).names == ("state", "halted")


@pytest.mark.parametrize("mode", MODES)
def test_store_views_alias_and_start_zeroed(mode):
    st = pgx.VertexStore(6, np.int64, np.float64, mode)
    for p in (0, 1):
        assert not st.flags(p).any() and not st.values(p).any()
    st.values(1)[3] = 42
    st.flags(1)[3] = True
    assert st.hot(1)[3]["msg"] == 42 and st.hot(1)[3]["flag"]
    assert st.values(0)[3] == 0                       # parities are separate
    rec = st.cold(2)
    rec["state"] = 1.5
    rec["halted"] = True
    assert st.state[2] == 1.5 and st.halted[2]        # writes go through
    assert not st.flags(0).any() and st.values(1)[2] == 0


def test_layout_specific_storage():
    il = pgx.VertexStore(4, np.float64, np.float64, pgx.LayoutMode.INTERLEAVED)
    ex = pgx.VertexStore(4, np.float64, np.float64, pgx.LayoutMode.EXTERNALISED)
    assert il.record_nbytes == 9 + 9 + 9 and not il.buffers_contiguous()
    assert ex.record_nbytes == 9 + 9 + 9 and ex.buffers_contiguous()
    assert ex.hot_itemsize == 9


@pytest.mark.parametrize("mode", MODES)
def test_locks_lazy_stable_and_edge_cases(mode):
    st = pgx.VertexStore(3, np.uint32, np.uint32, mode)
    assert st._locks is None
    locks = st.locks
    assert len(locks) == 3 and st.locks is locks
    assert pgx.VertexStore(0, np.uint32, np.uint32, mode).locks == []
    with pytest.raises(pgx.ConfigError):
        pgx.VertexStore(-1, np.uint32, np.uint32, mode)


# ---- combiner strategies ------------------------------------------------

def _buf(dtype=np.int64, n=4, guarded=False):
    st = pgx.VertexStore(n, dtype, dtype, pgx.LayoutMode.EXTERNALISED)
    return pgx.MessageBuffer(st, 0, guarded)


@pytest.mark.parametrize("send", STRATEGIES, ids=lambda f: f.__name__)
def test_publish_then_combine(send):
    cmb = pgx.min_combine(np.int64)
    buf = _buf()
    if send is pgx.send_cas:
        buf.values[:] = cmb.neutral
    send(buf, 2, 9, cmb)
    send(buf, 2, 4, cmb)
    send(buf, 2, 7, cmb)
    assert buf.flags.tolist() == [False, False, True, False]
    assert buf.values[2] == 4


@pytest.mark.parametrize("send", STRATEGIES, ids=lambda f: f.__name__)
def test_opposite_sums_leave_a_flagged_zero(send):
    cmb = pgx.sum_combine(np.int64)
    buf = _buf()
    send(buf, 1, 5, cmb)
    send(buf, 1, -5, cmb)
    assert buf.flags[1] and buf.values[1] == 0       # zero is a value, not "empty"


def test_apply_cas_skips_noop_combines_and_counts_attempts():
    cmb = pgx.min_combine(np.int64)
    buf = _buf()
    pgx.send_hybrid(buf, 0, 3, cmb)
    assert pgx.apply_cas(buf, 0, 8, cmb) == 0       # min(3, 8) == 3: no write
    assert pgx.apply_cas(buf, 0, 1, cmb) == 1 and buf.values[0] == 1


def test_cas_primitive_and_consume():
    buf = _buf()
    buf.values[1] = 6
    assert not buf.cas(1, 5, 7) and buf.values[1] == 6
    assert buf.cas(1, 6, 7) and buf.values[1] == 7
    assert buf.read_and_consume(1) is None           # not flagged
    buf.flags[1] = True
    assert buf.read_and_consume(1) == 7 and not buf.flags[1]


def test_sender_dispatch_and_phase_guard():
    assert pgx.sender_for(pgx.CombinerKind.LOCK) is pgx.send_lock
    assert pgx.sender_for(pgx.CombinerKind.CAS) is pgx.send_cas
    assert pgx.sender_for(pgx.CombinerKind.HYBRID) is pgx.send_hybrid
    cmb = pgx.min_combine(np.int64)
    buf = _buf(guarded=True)
    for send in STRATEGIES:
        with pytest.raises(pgx.PhaseError):
            send(buf, 0, 1, cmb)
    buf.accepting = True
    pgx.send_hybrid(buf, 0, 1, cmb)
    free = _buf(guarded=False)
    pgx.send_lock(free, 0, 1, cmb)                   # unguarded: never raises


def test_mailbox_parities_prefill_and_errors():
    st = pgx.VertexStore(3, np.int64, np.int64, pgx.LayoutMode.INTERLEAVED)
    cmb = pgx.min_combine(np.int64)
    mb = pgx.Mailbox(st, cmb, pgx.CombinerKind.HYBRID)
    send = mb.sender()
    send(1, 5)
    assert mb.next.flags[1] and not mb.current.flags[1]
    nxt = mb.next
    mb.swap_buffers()
    assert mb.current is nxt and mb.current.values[1] == 5
    cas = pgx.Mailbox(pgx.VertexStore(3, np.int64, np.int64), cmb, pgx.CombinerKind.CAS)
    cas.prepare()
    assert (cas.next.values == cmb.neutral).all()
    cas.sender()(0, 4)
    cas.swap_buffers()
    cas.swap_buffers()                               # the retired parity is re-filled
    assert (cas.next.values == cmb.neutral).all() and not cas.next.flags.any()
    with pytest.raises(pgx.ConfigError):
        pgx.Mailbox(st, pgx.CombineFn(fn=min), pgx.CombinerKind.CAS)
    with pytest.raises(pgx.ConfigError):
        pgx.Mailbox(st, None, pgx.CombinerKind.HYBRID).sender()


@pytest.mark.parametrize("kind", list(pgx.CombinerKind))
def test_concurrent_folds_are_exact(kind):
    st = pgx.VertexStore(8, np.int64, np.int64, pgx.LayoutMode.EXTERNALISED)
    cmb = pgx.sum_combine(np.int64)
    mb = pgx.Mailbox(st, cmb, kind)
    mb.prepare()
    send = mb.sender()

    def worker(seed):
        rng = np.random.default_rng(seed)
        for dst in rng.integers(0, 8, 400):
            send(int(dst), 1)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert int(mb.next.values[mb.next.flags].sum()) == 6 * 400


# ---- scheduler -----------------------------------------------------------

def test_chunk_claimer_contract():
    c = pgx.dynamic_chunks(1000, 256)
    got = []
    while (r := c.claim()) is not None:
        got.append(r)
    assert got == [(0, 256), (256, 512), (512, 768), (768, 1000)]
    assert pgx.dynamic_chunks(10).chunk_size == pgx.DEFAULT_CHUNK_SIZE
    assert pgx.dynamic_chunks(0).claim() is None
    with pytest.raises(pgx.ConfigError):
        pgx.ChunkClaimer(10, 0)
    c = pgx.ChunkClaimer(10_000, 7)
    seen = []

    def worker():
        while (r := c.claim()) is not None:
            seen.extend(range(*r))

    ts = [threading.Thread(target=worker) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert sorted(seen) == list(range(10_000))     # every item exactly once


# ---- the device combine against the sequential strategy ------------------

@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_device_scatter_equals_hybrid_sends(seed):
    """pgx_scatter (one warp-tiled kernel, fire-and-forget red.min and
    has-bits) leaves exactly the flags / values that send_hybrid produces
    when the same messages are sent one by one."""
    rng = np.random.default_rng(seed)
    n, m = 3000, 40_000
    src = np.sort(rng.integers(0, n, m))
    dst = rng.integers(0, n, m)
    g = pgx.from_edges(src, dst, n, device="cuda")
    c = g.device_csr()
    al = lambda x: (x + 255) // 256 * 256
    o_id = al(16)
    o_eb = o_id + al(4 * (n + 1))
    o_tile = o_eb + al(4 * (n + 1))
    nz_id = c.ws[o_id:o_id + 4 * (n + 1)].view(torch.int32)
    nz_eb = c.ws[o_eb:o_eb + 4 * (n + 1)].view(torch.int32)
    tile = c.ws[o_tile:o_tile + 4 * ((m + 255) // 256 + 2)].view(torch.int32)
    nnz = int(c.ws[:16].view(torch.int32)[0])
    mb = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    has = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    _lib.check(lib.pgx_scatter(_lib.PGX_OP_MIN_U32, 1, c.col_idx.data_ptr(), nz_eb.data_ptr(),
                               None, nz_id.data_ptr(), 0, None, tile.data_ptr(), nnz, m,
                               mb.data_ptr(), has.data_ptr(), 0xFFFFFFFF,
                               torch.cuda.current_stream().cuda_stream), "pgx_scatter")
    torch.cuda.synchronize()
    buf = _buf(np.uint32, n)
    cmb = pgx.min_combine(np.uint32)
    off = g.out_offsets.cpu().numpy()
    tgt = g.out_targets.cpu().numpy()
    for u in range(n):                               # sender u broadcasts its id
        for w in tgt[off[u]:off[u + 1]]:
            pgx.send_hybrid(buf, int(w), u, cmb)
    bits = has.cpu().numpy().view(np.uint32)
    flags = ((bits[np.arange(n) >> 5] >> (np.arange(n) & 31)) & 1).astype(bool)
    assert np.array_equal(flags, buf.flags)
    assert np.array_equal(mb.cpu().numpy().view(np.uint32)[flags], buf.values[flags])
