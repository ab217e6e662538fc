"""The reference's combiner / layout / scheduler schema that EngineConfig
and VertexProgram accept (mailbox.py:43-79, layout.py:31-33,
scheduler.py:27-76) -- and, on the GPU, the device combine reproduces the
reference's hybrid strategy applied message by message (send_hybrid,
mailbox.py:180-199, restated below as the sequential specification)."""

import numpy as np
import pytest
import torch

import paper_2010_01542_b200 as pgx
from paper_2010_01542_b200 import _lib


def test_combine_declarations():
    mn = pgx.min_combine(np.uint32)
    assert mn.name == "min" and mn.neutral == 2 ** 32 - 1 and mn.fn(3, 5) == 3
    assert pgx.min_combine(np.float64).neutral == np.inf
    sm = pgx.sum_combine(np.float64)
    assert sm.name == "sum" and sm.neutral == 0.0 and sm.ufunc is np.add
    assert {k.value for k in pgx.CombinerKind} == {"lock", "cas", "hybrid"}


def test_layout_and_scheduler_modes():
    assert {m.value for m in pgx.LayoutMode} == {"interleaved", "externalised"}
    assert pgx.SchedulerMode.static().kind is pgx.SchedulerKind.STATIC
    d = pgx.SchedulerMode.dynamic()
    assert d.kind is pgx.SchedulerKind.DYNAMIC and d.chunk_size == pgx.DEFAULT_CHUNK_SIZE
    assert pgx.SchedulerMode.edge_balanced().kind is pgx.SchedulerKind.EDGE_BALANCED
    with pytest.raises(pgx.ConfigError):
        pgx.SchedulerMode.dynamic(0)


@pytest.mark.parametrize("kw", [dict(layout=pgx.LayoutMode.EXTERNALISED),
                                dict(scheduler=pgx.SchedulerMode.dynamic(64)),
                                dict(combiner=pgx.CombinerKind.LOCK), dict(workers=4)])
def test_engine_config_accepts_the_reference_knobs(kw):
    """Accepted and validated like the reference; inert on the device."""
    pgx.EngineConfig(**kw)


def test_engine_config_rejects_bad_knobs():
    g = pgx.from_edges([0], [1], 2)
    for cfg in (pgx.EngineConfig(workers=0), pgx.EngineConfig(scheduler="dynamic"),
                pgx.EngineConfig(layout="soa"), pgx.EngineConfig(combiner="cas")):
        with pytest.raises(pgx.ConfigError):
            pgx.run(g, pgx.connected_components(), cfg)


class _HybridSpec:
    """Sequential restatement of the reference's hybrid send (test
    specification only): the first message to an empty slot publishes
    value then flag; later ones combine only when that changes the value."""

    def __init__(self, n):
        self.flags = np.zeros(n, bool)
        self.values = np.zeros(n, np.uint32)

    def send(self, dst, msg):
        if not self.flags[dst]:
            self.values[dst] = msg
            self.flags[dst] = True
        elif min(int(self.values[dst]), msg) != int(self.values[dst]):
            self.values[dst] = msg


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_device_scatter_equals_hybrid_sends(seed):
    """pgx_scatter (one warp-tiled kernel, fire-and-forget red.min and
    has-bits) leaves exactly the flags / values that the hybrid strategy
    produces when the same messages are sent one by one."""
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
    spec = _HybridSpec(n)
    off = g.out_offsets.cpu().numpy()
    tgt = g.out_targets.cpu().numpy()
    for u in range(n):                               # sender u broadcasts its id
        for w in tgt[off[u]:off[u + 1]]:
            spec.send(int(w), u)
    bits = has.cpu().numpy().view(np.uint32)
    flags = ((bits[np.arange(n) >> 5] >> (np.arange(n) & 31)) & 1).astype(bool)
    assert np.array_equal(flags, spec.flags)
    assert np.array_equal(mb.cpu().numpy().view(np.uint32)[flags], spec.values[flags])
