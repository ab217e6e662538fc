"""Partitioned multi-GPU superstep, one process per GPU.

The reference has no distributed mode (SPEC.md:420 non-goal); this is the
B200 build's scale-out of the same superstep, with results identical to
one GPU (CC labels / SSSP distances bit-exact, PageRank within 1e-9):

* **partition**: 1-D by source vertex.  Rank r owns the contiguous vertex
  range ``[lo_r, hi_r)`` -- its out-edges and that block of the mailbox.
  Ranges balance ``out_degree + 1`` (edges + vertex work) across ranks
  (``partition_bounds``).
* **owner-blocked mailbox**: every rank's full-width mailbox is laid out as
  ``world`` equal blocks of ``B`` slots (B = the largest range, rounded up
  to 64): vertex v of owner r lives at position ``r * B + (v - lo_r)``.  The
  local CSR stores those positions (remapped once per graph), so the
  per-superstep reduction is ONE equal-block ``reduce_scatter_tensor``
  (ncclReduceScatter, in place, NVLS-eligible) instead of per-owner
  reduces, and the owner of a slot is ``slot // B``.  Messages stay global
  vertex ids (CC labels, SSSP distances).
* **per superstep** (min programs): every rank scatters its senders into
  its full-width mailbox (``pgx_scatter``; CC's dense supersteps -- sender
  edges >= a quarter of the rank's -- through the rank's own segmented
  index, ``pgx_seg_scatter``, as on one GPU); the mailbox is delivered to the
  owners by one of three exchanges (below); the owner applies on its block
  (``pgx_apply_slice``); ONE all-gather of every rank's (recipients,
  broadcasts, senders, edges) drives the halt test and the statistics and
  sizes the next scatter -- the only host read of the superstep (plus the
  split sizes on a sparse superstep).
* **exchanges** (min programs, chosen per superstep, collectively):
  - ``peer`` (the fused compute + collective): when every rank maps every
    other rank's mailbox (CUDA IPC over NVLink / NVSwitch, ``pgx_peer_*``),
    ``pgx_scatter_peer`` combines each message that passes the rank's local
    filter straight into the OWNER's slot with a system-scope
    ``red.min`` -- no reduction at all; a one-element all-reduce orders the
    combines before the owners' apply.  Used for supersteps that traverse
    at most n/2 edges ("auto") or always ("peer");
  - ``dense``: the equal-block ``reduce_scatter_tensor`` (MIN), used for the
    big supersteps;
  - ``sparse`` (when no peer mapping exists): if every
    rank's edges bound its touched foreign slots below a quarter of the
    dense volume, the touched slots are compacted into (slot, value) pairs
    (grouped by owner) and exchanged with ``all_to_all_single``.
* **PageRank**: the reference's pull fold (engine.py:425-457) per rank --
  a local in-CSR of the rank's out-edges (rows = mailbox positions,
  entries = local sources), folded with the K3 kernel into a full-width
  partial sum (``pgx_gather_slice`` + ``pgx_fold_spanning``), then the
  SUM ``reduce_scatter_tensor``.  The dangling mass is all-reduced on the
  device and read by the next apply from device memory: a PageRank
  superstep has no host synchronisation.  ``pr_mode="push"`` keeps the
  ``red.add.f64`` scatter as the A/B arm.
* has-message after the reduction is ``mailbox != neutral``: CC / SSSP
  messages are < n < 2^31 - 1 and never equal the exchange neutral
  INT32_MAX (the signed int32 MIN of NCCL / gloo is then exact).

The orchestration below is backend-agnostic: ``CudaBackend`` drives
libpgx.so on the rank's GPU (NCCL process group); tests/ drive the same
``PartitionedRun`` with a CPU test backend over a gloo process group and
with the CUDA backend on threads sharing one GPU.
"""

from __future__ import annotations

import ctypes
import os
import time
import weakref
from dataclasses import dataclass

import numpy as np
import torch

#: min neutral of the exchanged mailbox: INT32_MAX, so that the signed
#: int32 MIN reduction of NCCL / gloo is exact (messages are < n < 2^31 - 1)
EXCHANGE_NEUTRAL = 2 ** 31 - 1

#: mailbox blocks are padded to a multiple of this many slots (has-bitmask
#: words and 128-byte lines never straddle two owners)
BLOCK_ALIGN = 64


def distributed_context():
    """The active torch.distributed module when world_size > 1, else None."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    if dist.get_world_size() <= 1:
        return None
    return dist


def partition_bounds(out_degrees, world: int) -> np.ndarray:
    """Contiguous owner ranges ``bounds[r]..bounds[r+1]`` balancing
    ``out_degree + 1`` per vertex: range r ends at the first vertex whose
    inclusive work prefix reaches ``(r + 1) / world`` of the total (exact
    integer comparison), so every range carries less than
    ``total / world + max work`` and an empty graph gives empty ranges."""
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    w = torch.as_tensor(np.asarray(out_degrees, dtype=np.int64)) + 1
    n = int(w.numel())
    bounds = np.zeros(world + 1, dtype=np.int64)
    bounds[-1] = n
    if n == 0 or world == 1:
        return bounds
    prefix = torch.cumsum(w, 0)                       # inclusive work prefix
    total = int(prefix[-1])
    goal = torch.arange(1, world, dtype=torch.int64) * total
    cut = torch.searchsorted(prefix * world, goal, right=False) + 1
    bounds[1:-1] = np.minimum(cut.numpy(), n)
    return np.maximum.accumulate(bounds)


def owner_block(bounds) -> int:
    """Slots per owner block of the padded mailbox."""
    sizes = np.diff(np.asarray(bounds, dtype=np.int64))
    big = int(sizes.max()) if sizes.size else 0
    return max(BLOCK_ALIGN, -(-big // BLOCK_ALIGN) * BLOCK_ALIGN)


def padded_positions(col: torch.Tensor, bounds, block: int,
                     chunk: int = 1 << 27) -> torch.Tensor:
    """Global vertex ids -> owner-blocked mailbox positions (int32), in
    chunks (the int64 temporaries stay bounded)."""
    inner = torch.as_tensor(np.asarray(bounds[1:-1], dtype=np.int64), device=col.device)
    lo = torch.as_tensor(np.asarray(bounds[:-1], dtype=np.int64), device=col.device)
    out = torch.empty(col.numel(), dtype=torch.int32, device=col.device)
    for a in range(0, col.numel(), chunk):
        c = col[a:a + chunk].to(torch.int64)
        owner = torch.searchsorted(inner, c, right=True)
        out[a:a + chunk] = (owner * block + c - lo[owner]).to(torch.int32)
    return out


@dataclass
class StepCounts:
    recipients: int
    broadcasts: int
    senders: int
    edges: int


class PartitionedRun:
    """Backend-agnostic driver of one partitioned run on this rank."""

    def __init__(self, backend, dist, bounds, n: int, m: int):
        self.b = backend
        self.dist = dist
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.n, self.m = n, m
        self.lo = int(self.bounds[self.rank])
        self.hi = int(self.bounds[self.rank + 1])
        self.B = owner_block(self.bounds)
        self.npad = self.world * self.B
        self.b.bind(self.bounds, self.rank, self.B)
        # min-program exchange: "auto" (peer if every rank maps every peer,
        # else hybrid), "peer", "hybrid" (dense / sparse per superstep),
        # "dense" (A/B switches)
        self.exchange = "auto"
        be = str(getattr(dist, "get_backend", lambda: "")())
        # gloo has no CUDA collectives: stage device tensors through the host
        self._host_coll = be == "gloo" and self.b.device.type == "cuda"
        self._cdev = torch.device("cpu") if self._host_coll else self.b.device

    def _coll_sync(self):
        """Before a host-side collective: the rank's kernels have finished."""
        if self._host_coll:
            torch.cuda.current_stream(self.b.device).synchronize()

    def _to_coll(self, t: torch.Tensor) -> torch.Tensor:
        if self._host_coll:
            self._coll_sync()
            return t.cpu()
        return t

    def _peer_setup(self) -> bool:
        """Map every rank's mailbox on every rank (collective decision).

        The outcome is cached on the rank's backend (cached per graph, so
        every rank of a job holds the same cache state): later runs on the
        same backend skip the handle exchange."""
        cached = getattr(self.b, "_peer_decision", None)
        if cached is not None and cached[0] == self.exchange:
            self.b.peer_active = cached[1]
            return cached[1]
        want = self.exchange in ("auto", "peer") and hasattr(self.b, "peer_handle")
        h = self.b.peer_handle() if want else None
        handles = [None] * self.world
        self.dist.all_gather_object(handles, h)
        ok = all(x is not None for x in handles) and self.b.open_peers(handles)
        t = torch.tensor([1 if ok else 0], dtype=torch.int64, device=self._cdev)
        self._coll_sync()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        ok = bool(t.item())
        if not ok and self.exchange == "peer":
            raise RuntimeError("peer exchange requested but a rank cannot map its peers")
        self.b.peer_active = ok
        self.b._peer_decision = (self.exchange, ok)
        return ok

    def _fence(self):
        """All ranks' peer combines land before any owner applies."""
        t = torch.zeros(1, dtype=torch.int64, device=self._cdev)
        self._coll_sync()
        self.dist.all_reduce(t)

    # ---- collectives --------------------------------------------------

    def _reduce_slices(self, op):
        """Deliver every owner the reduction of its mailbox block: one
        equal-block reduce_scatter, in place (output = this rank's block of
        the input)."""
        full = self.b.mailbox
        mine = full[self.rank * self.B:(self.rank + 1) * self.B]
        if self._host_coll:  # gloo: stage the mailbox through the host
            self._coll_sync()
            host = full.cpu()
            out = torch.empty(self.B, dtype=host.dtype)
            self.dist.reduce_scatter_tensor(out, host, op=op)
            mine.copy_(out)
            return
        self.dist.reduce_scatter_tensor(mine, full, op=op)

    def _exchange_min(self, op, max_edges: int, allow_sparse: bool) -> str:
        """Dense block reduction or sparse pair exchange.  The choice uses
        every rank's edge count (a bound on its touched foreign slots, known
        to all ranks from the counters all-gather): collective without a
        further reduction."""
        if allow_sparse and self.exchange != "dense" and 16 * max_edges < 4 * self.npad:
            pairs, splits = self.b.compact_touched()           # one host read
            send = torch.tensor(splits, dtype=torch.int64, device=self._cdev)
            recv_n = torch.empty_like(send)
            self.dist.all_to_all_single(recv_n, send)
            recv_splits = recv_n.tolist()
            pairs = self._to_coll(pairs)
            recv = torch.empty(sum(recv_splits), dtype=torch.int64, device=pairs.device)
            self.dist.all_to_all_single(recv, pairs, recv_splits, list(splits))
            self.b.scatter_pairs(recv.to(self.b.device))
            return "sparse"
        self._reduce_slices(op)
        return "dense"

    def _gather_counts(self, local: torch.Tensor):
        """Every rank's (recipients, broadcasts, senders, edges) in ONE
        all-gather and one host read: the sums drive the halt test and the
        statistics, the rank's own senders / edges size its next scatter."""
        local = self._to_coll(local.to(torch.int64))
        parts = [torch.empty_like(local) for _ in range(self.world)]
        self.dist.all_gather(parts, local)
        rows = [self.b.decode_counts(r) for r in torch.stack(parts).tolist()]
        self.b.set_frontier(rows[self.rank][2], rows[self.rank][3])
        tot = [sum(r[i] for r in rows) for i in range(4)]
        return StepCounts(*tot), max(r[3] for r in rows)

    def _gather_values(self):
        local = self._to_coll(self.b.values())
        sizes = np.diff(self.bounds)
        mx = int(sizes.max()) if sizes.size else 0
        pad = torch.zeros(max(mx, 1), dtype=local.dtype, device=local.device)
        pad[:local.numel()] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad)
        return torch.cat([parts[r][:int(sizes[r])] for r in range(self.world)])

    # ---- min programs: CC / SSSP -------------------------------------

    def run_min(self, app: str, source: int, max_steps: int):
        """loop_min, then every rank's values gathered (rank order)."""
        stats, hit_cap, wall = self.loop_min(app, source, max_steps)
        return self._gather_values(), stats, hit_cap, wall

    def loop_min(self, app: str, source: int, max_steps: int):
        """The superstep loop of a CC / SSSP run; values stay on the rank."""
        op = self.dist.ReduceOp.MIN
        n = self.n
        peer_ok = self._peer_setup()
        self.b.init_min(app)
        if peer_ok:  # every mailbox is neutral before any peer combines into it
            self._fence()
        stats = []
        if app == "sssp":
            own = self.lo <= source < self.hi
            deg = self.b.global_out_degree(source)
            if own:
                self.b.seed_source(source - self.lo)
            nxt = StepCounts(0, 1, 1 if deg > 0 else 0, deg)
            max_edges = deg
        else:
            nxt = StepCounts(0, n, self.b.global_nonzero_degree(), self.m)
            max_edges = self.m
        hit_cap = False
        t0 = time.perf_counter()
        active = n  # superstep 0 runs every vertex
        for s in range(max_steps):
            ts = time.perf_counter()
            cur = nxt
            # "auto": the fused peer exchange for supersteps that traverse at
            # most n/2 edges (remote combines ~ surviving foreign messages),
            # the dense collective (n slots per rank) for the big ones
            use_peer = peer_ok and (self.exchange == "peer" or 2 * cur.edges <= n)
            self.b.reset_mailbox()
            self.b.scatter_min(dense=(app == "components" and s == 0), peer=use_peer)
            if use_peer:
                self._fence()
                exchange = "peer"
            else:  # with the peer path mapped only big supersteps get here
                exchange = self._exchange_min(op, max_edges, allow_sparse=not peer_ok)
            self.b.exchanged(exchange)
            at_cap = s + 1 == max_steps
            nxt, max_edges = self._gather_counts(self.b.apply_min(app, count_only=at_cap))
            sent = cur.edges if app == "sssp" else cur.broadcasts
            stats.append(dict(index=s, active_count=active,
                              messages_sent=sent, edges=cur.edges,
                              senders=cur.senders, recipients=nxt.recipients,
                              broadcasters=cur.broadcasts,
                              seconds=time.perf_counter() - ts, exchange=exchange))
            active = nxt.recipients
            if nxt.recipients == 0:
                break
            if at_cap:
                hit_cap = True
                break
        return stats, hit_cap, time.perf_counter() - t0

    # ---- PageRank -------------------------------------------------------

    def run_pagerank(self, iterations: int, damping: float, max_steps: int):
        """loop_pagerank, then every rank's ranks gathered (rank order)."""
        stats, hit_cap, wall = self.loop_pagerank(iterations, damping, max_steps)
        return self._gather_values(), stats, hit_cap, wall

    def loop_pagerank(self, iterations: int, damping: float, max_steps: int):
        """The superstep loop of a PageRank run; ranks stay on the rank.
        No host read inside the loop: the dangling mass stays on the device."""
        op = self.dist.ReduceOp.SUM
        n = self.n
        base = (1.0 - damping) / n      # algorithms.py:49
        r0 = 1.0 / n                    # algorithms.py:50
        last = iterations - 1
        ndangling = self.b.init_pagerank(r0)
        t = torch.tensor([ndangling], dtype=torch.int64, device=self._cdev)
        self._coll_sync()
        self.dist.all_reduce(t)
        ndangling = int(t.item())
        nspread = n - ndangling
        # algorithms.py:55: the setup's dangling mass, then each superstep's
        dangling = torch.tensor([r0 * ndangling], dtype=torch.float64, device=self.b.device)
        stats = []
        t0 = time.perf_counter()
        steps = min(max_steps, iterations)
        for s in range(steps):
            ts = time.perf_counter()
            # the fold of superstep s: shares broadcast at s-1 (or the seed)
            self.b.fold_sum()
            self._reduce_slices(op)
            local = self.b.apply_pagerank(base, damping, dangling, s == last)
            d = self._to_coll(local)
            self.dist.all_reduce(d)
            dangling = d.to(self.b.device)
            stats.append(dict(index=s, active_count=n,
                              messages_sent=0 if s == last else nspread,
                              edges=self.m, senders=nspread, recipients=n,
                              broadcasters=0 if s == last else nspread,
                              seconds=time.perf_counter() - ts))
        hit_cap = steps < iterations  # engine.py:299-300
        return stats, hit_cap, time.perf_counter() - t0


# ----------------------------------------------------------------------
# CUDA backend (libpgx phase kernels on this rank's GPU)
# ----------------------------------------------------------------------

class _DeviceArray:
    """``__cuda_array_interface__`` of a raw device allocation (zero-copy
    torch view)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2,
                                         "strides": None}


class PeerMailbox:
    """A rank's full-width min mailbox in a ``cudaMalloc`` block that the
    other ranks map through CUDA IPC (pgx_peer_alloc)."""

    def __init__(self, _lib, lib, n: int, device):
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(_lib.PGX_IPC_HANDLE_BYTES)
        _lib.check(lib.pgx_peer_alloc(4 * max(n, 1), ctypes.byref(ptr), handle),
                   "pgx_peer_alloc")
        self.ptr = int(ptr.value)
        self.n = n
        self.handle = handle.raw
        self.tensor = torch.as_tensor(_DeviceArray(self.ptr, n, "<i4"), device=device)
        # freed with its owner (the backend drops it only after its last run)
        weakref.finalize(self, lib.pgx_peer_free, ctypes.c_void_p(self.ptr))


class CudaBackend:
    """Owns the rank's local CSR, full-width mailbox and owned-block state."""

    def __init__(self, graph, lo: int, hi: int, device, pr_mode: str = "pull",
                 segments: str = "auto"):
        from . import _lib
        self._lib = _lib
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.stream = torch.cuda.current_stream(self.device)
        self.pr_mode = pr_mode
        # CC dense supersteps through K1s (pgx_seg_scatter) unless "off"
        self.segments = segments
        dev = self.device
        # slice where the graph lives and upload only this rank's rows (a
        # pinned host graph stays pinned under slicing: one DMA per array)
        off = graph.out_offsets
        self.n = graph.vertex_count
        self._glob_off = off
        base, end = int(off[lo]), int(off[hi])
        self.row_ptr = (off[lo:hi + 1] - base).to(dev, non_blocking=True) \
            .to(torch.int32).contiguous()
        self.col_global = graph.out_targets[base:end].to(dev, non_blocking=True) \
            .to(torch.int32).contiguous()
        self.col = self.col_global          # padded positions after bind()
        self.len = hi - lo
        self.lo_own, self.hi_own = lo, hi
        self.m_local = int(self.col.numel())
        self.launches = 0
        st = self.stream.cuda_stream
        ws_bytes = _lib.out_size(self.lib.pgx_graph_workspace_bytes, max(self.len, 1),
                                 self.m_local)
        self.gws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        if self.len > 0:
            _lib.check(self.lib.pgx_graph_prepare(self.len, self.m_local,
                                                  self.row_ptr.data_ptr(),
                                                  self.gws.data_ptr(), ws_bytes, st),
                       "pgx_graph_prepare")
        self._g_hdr, self._g_nz_id, self._g_nz_eb, self._g_tile = \
            self._graph_views(self.gws, self.len, self.m_local)
        cb = _lib.out_size(self.lib.pgx_slice_counters_bytes)
        self.ctr = torch.zeros(cb, dtype=torch.uint8, device=dev)
        ntile = (self.m_local + 255) // 256 + 2
        self.f_eb = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_rs = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_msg = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_tile = torch.empty(ntile, dtype=torch.int32, device=dev)
        self.nsrc, self.E = 0, 0
        self._scattered = 0
        self._bound = None
        self._pull = None
        self._last = None
        # fused peer exchange state (PartitionedRun._peer_setup)
        self.peer_active = False
        self._peer_mb = None
        self._peer_sig = None
        self._opened = []
        # peer mappings are closed when the backend goes away
        weakref.finalize(self, CudaBackend._close_all, self.lib, self._opened)

    @staticmethod
    def _graph_views(gws, rows, m):
        """(hdr, nz_id, nz_eb, tile_src) views of a graph workspace
        (pgx_common.cuh graph_ws_layout: 256-byte aligned chunks)."""
        al = lambda x: (x + 255) // 256 * 256
        o_id = al(16)
        o_eb = o_id + al(4 * (rows + 1))
        o_tile = o_eb + al(4 * (rows + 1))
        ntile = (m + 255) // 256 + 2
        return (gws[:16].view(torch.int32), gws[o_id:o_id + 4 * (rows + 1)].view(torch.int32),
                gws[o_eb:o_eb + 4 * (rows + 1)].view(torch.int32),
                gws[o_tile:o_tile + 4 * ntile].view(torch.int32))

    def _k(self, rc, name, kernels=1):
        """Check a libpgx launch and count its kernels (bench gpu_launches)."""
        self.launches += kernels
        self._lib.check(rc, name)

    @staticmethod
    def _close_all(lib, opened):
        for p in opened:
            lib.pgx_peer_close(ctypes.c_void_p(p))
        opened.clear()

    # ---- layout ----
    def bind(self, bounds, rank: int, block: int):
        """Adopt the job's owner-blocked layout: destinations become padded
        mailbox positions (once per bounds)."""
        sig = (tuple(int(x) for x in bounds), rank, block)
        if self._bound == sig:
            return
        self.rank, self.block, self.world = rank, block, len(bounds) - 1
        self.npad = self.world * block
        self.blo = rank * block                       # this rank's block
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.col = padded_positions(self.col_global, bounds, block)
            self.has = torch.zeros(self.npad // 32 + 2, dtype=torch.int32, device=self.device)
            sb = self._lib.out_size(self.lib.pgx_touched_scratch_bytes, self.npad)
            self.tscratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
            self.tcount = torch.zeros(1, dtype=torch.int64, device=self.device)
            self._pbounds = torch.arange(self.world + 1, dtype=torch.int32,
                                         device=self.device) * block
        self._pull = None
        self._seg = None
        self._peer_sig = None
        self._peer_decision = None
        self._bound = sig

    # ---- helpers ----
    def _nnz(self) -> int:
        """Senders with out-degree > 0 (graph workspace header; read once)."""
        if getattr(self, "_nnz_cache", None) is None:
            self._nnz_cache = int(self._g_hdr[0]) if self.len > 0 else 0
        return self._nnz_cache

    def global_out_degree(self, v: int) -> int:
        return int(self._glob_off[v + 1]) - int(self._glob_off[v])

    def global_nonzero_degree(self) -> int:
        if getattr(self, "_nnz_global", None) is None:
            self._nnz_global = int((torch.diff(self._glob_off) > 0).sum())
        return self._nnz_global

    # ---- fused peer exchange ----
    def peer_handle(self):
        """This rank's mappable mailbox and has-bitmap (allocated once: the
        min exchange and the unit-weight SSSP bitmap exchange), or None."""
        try:
            if self._peer_mb is None or self._peer_mb.n != self.npad:
                self._peer_mb = PeerMailbox(self._lib, self.lib, self.npad, self.device)
                self._peer_has = PeerMailbox(self._lib, self.lib, self.npad // 32 + 2,
                                             self.device)
        except Exception:
            return None
        return {"pid": os.getpid(), "device": self.device.index, "ptr": self._peer_mb.ptr,
                "handle": self._peer_mb.handle, "has_ptr": self._peer_has.ptr,
                "has_handle": self._peer_has.handle}

    def close_peers(self):
        CudaBackend._close_all(self.lib, self._opened)  # in place: the finalizer's list
        self._peer_sig = None

    def _map(self, h, ptr_key, handle_key) -> int:
        if h["pid"] == os.getpid():
            if h["device"] != self.device.index:
                with torch.cuda.device(self.device):
                    self._lib.check(self.lib.pgx_peer_enable(h["device"]), "pgx_peer_enable")
            return h[ptr_key]
        p = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self._lib.check(self.lib.pgx_peer_open(h[handle_key], ctypes.byref(p)),
                            "pgx_peer_open")
        self._opened.append(int(p.value))
        return int(p.value)

    def open_peers(self, handles) -> bool:
        """Device arrays of every rank's mailbox and has-bitmap bases:
        IPC-mapped, or the raw pointers for ranks that are threads of this
        process (peer access enabled when they sit on another GPU)."""
        sig = tuple((h["pid"], h["ptr"]) for h in handles)
        if sig == self._peer_sig:
            return True
        self.close_peers()
        try:
            ptrs = [self._map(h, "ptr", "handle") for h in handles]
            has_ptrs = [self._map(h, "has_ptr", "has_handle") for h in handles]
        except Exception:
            self.close_peers()
            return False
        self._peer_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        self._peer_has_ptrs = torch.tensor(has_ptrs, dtype=torch.int64, device=self.device)
        self._peer_sig = sig
        return True

    # ---- K1s on the slice (CC dense supersteps) ----
    def _ensure_seg(self):
        """The rank's rectangular segmented index (rows = its sources,
        destinations = padded mailbox positions), built once per layout."""
        if self._seg is not None:
            return self._seg
        L, lib, dev, st = self._lib.PGX_SEG_LOG2_DEFAULT, self.lib, self.device, self.stream
        n_r, nd, m = self.len, self.npad, self.m_local
        with torch.cuda.device(dev), torch.cuda.stream(st):
            sp = st.cuda_stream
            ws = torch.empty(self._lib.out_size(lib.pgx_seg_workspace_bytes, nd, m, -1, L),
                             dtype=torch.uint8, device=dev)
            nent = ctypes.c_int64(0)
            self._lib.check(lib.pgx_seg_count_ex(n_r, nd, m, self.row_ptr.data_ptr(),
                                                 self.col.data_ptr(), self.gws.data_ptr(), L,
                                                 ws.data_ptr(), ws.numel(), ctypes.byref(nent), sp),
                            "pgx_seg_count_ex")
            ne = int(nent.value)
            ws = torch.empty(self._lib.out_size(lib.pgx_seg_workspace_bytes, nd, m, ne, L),
                             dtype=torch.uint8, device=dev)
            cap = ctypes.c_int32(0)
            self._lib.check(lib.pgx_seg_max_items(nd, m, L, ctypes.byref(cap)), "pgx_seg_max_items")
            arrays = (torch.zeros(ne + 4, dtype=torch.int32, device=dev),       # ent_src
                      torch.empty(ne + 1, dtype=torch.int32, device=dev),       # ent_eb
                      torch.empty(m + 256, dtype=torch.int16, device=dev),      # col16
                      torch.empty((m + 255) // 256 + 1, dtype=torch.int32, device=dev),
                      torch.empty(4 * int(cap.value), dtype=torch.int32, device=dev))
            nitems = ctypes.c_int32(0)
            self._lib.check(lib.pgx_seg_build_ex(n_r, nd, m, self.row_ptr.data_ptr(),
                                                 self.col.data_ptr(), self.gws.data_ptr(), L, ne,
                                                 ws.data_ptr(), ws.numel(),
                                                 *(a.data_ptr() for a in arrays),
                                                 ctypes.byref(nitems), 0, sp), "pgx_seg_build_ex")
        # ent_eb (arrays[1]) is a build output the scatter never reads: freed
        ent_src, _, col16, tile_ent, items = arrays
        arrays = (ent_src, col16, tile_ent, items)
        self._seg = (self._lib.PgxSegIndex(L, ne, int(nitems.value), 0, ent_src.data_ptr(), None,
                                           col16.data_ptr(), tile_ent.data_ptr(),
                                           items.data_ptr()),
                     arrays, torch.zeros(1, dtype=torch.int32, device=dev))
        return self._seg

    def _use_seg(self, dense: bool) -> bool:
        return (self.segments != "off" and self.app == "components" and self.m_local > 0
                and (dense or 4 * self.E >= self.m_local))

    # ---- min programs ----
    def init_min(self, app):
        self.app = app
        if self.peer_active:
            self.mailbox = self._peer_mb.tensor
            self.has = self._peer_has.tensor   # peers set bits in it (SSSP)
        else:
            self.mailbox = torch.empty(self.npad, dtype=torch.int32, device=self.device)
        self.mailbox.fill_(EXCHANGE_NEUTRAL)
        self.has.zero_()
        self._level = 0  # supersteps scattered (unit-weight SSSP: the next level)
        self.val = torch.empty(max(self.len, 1), dtype=torch.int32, device=self.device)
        # CC send values (K1s): the label a sender sends, -1 (UINT32_MAX) otherwise
        self.sv = torch.full((max(self.len, 1),), -1, dtype=torch.int32, device=self.device) \
            if app == "components" and self.segments != "off" else None
        app_id = self._lib.PGX_APP_CC if app == "components" else self._lib.PGX_APP_SSSP
        self._k(self.lib.pgx_slice_init(app_id, self.len, self.lo_own, self.val.data_ptr(),
                                        self.row_ptr.data_ptr(), None, 0.0,
                                        self.stream.cuda_stream), "pgx_slice_init")
        self.nsrc, self.E = 0, 0
        self._last = None  # exchange of the previous superstep

    def seed_source(self, local_v: int):
        rs = int(self.row_ptr[local_v])
        deg = int(self.row_ptr[local_v + 1]) - rs
        self.val[local_v] = 0
        if deg > 0:
            self.f_eb[0] = 0
            self.f_rs[0] = rs
            self.f_msg[0] = 1
            ntiles = (deg + 255) // 256
            self.f_tile[:ntiles] = 0
            self.nsrc, self.E = 1, deg

    def reset_mailbox(self):
        """Undo what the previous superstep's exchange left behind.  The
        owned block is always neutral here (the apply consumed it), and it
        is never written: a peer may already be combining into it."""
        if self._last == "peer":  # foreign filter copies back to neutral, bits cleared
            self._k(self.lib.pgx_reset_touched(
                self.npad, self.blo, self.blo + self.block, self.has.data_ptr(),
                self.mailbox.data_ptr(), EXCHANGE_NEUTRAL, self.stream.cuda_stream),
                "pgx_reset_touched")
            return
        if self._last == "dense":  # every foreign slot holds a stale partial
            self.mailbox[:self.blo].fill_(EXCHANGE_NEUTRAL)
            self.mailbox[self.blo + self.block:].fill_(EXCHANGE_NEUTRAL)
        # sparse: the compaction reset the foreign touched slots.  Foreign
        # has-words only: the owned words were consumed by the apply, and a
        # peer may already be setting next-superstep bits in them (SSSP)
        if self._last is not None:
            self.has[:self.blo // 32].zero_()
            self.has[(self.blo + self.block) // 32:].zero_()

    def exchanged(self, kind: str):
        self._last = kind

    def compact_touched(self):
        """(slot << 32 | value) pairs of the touched foreign slots, in slot
        order (grouped by owner), and the per-owner counts (one host read).
        Touched foreign slots never outnumber the edges just scattered."""
        cap = max(min(self._scattered, self.npad), 1)
        pairs = torch.empty(cap, dtype=torch.int64, device=self.device)
        self._k(self.lib.pgx_touched(
            self.npad, self.blo, self.blo + self.block, self.has.data_ptr(),
            self.mailbox.data_ptr(), EXCHANGE_NEUTRAL, pairs.data_ptr(),
            self.tcount.data_ptr(), self.tscratch.data_ptr(), self.stream.cuda_stream),
            "pgx_touched", 3)
        # per-owner counts of the valid prefix; the unused tail is binned
        # past the last owner
        idx = torch.arange(cap, device=self.device)
        owner = torch.where(idx < self.tcount, (pairs >> 32) // self.block,
                            torch.full_like(pairs, self.world))
        counts = torch.bincount(owner, minlength=self.world + 1).tolist()
        splits = counts[:self.world]
        return pairs[:sum(splits)], splits

    def scatter_pairs(self, pairs):
        self._k(self.lib.pgx_scatter_pairs(pairs.data_ptr(), pairs.numel(),
                                           self.mailbox.data_ptr(),
                                           self.stream.cuda_stream), "pgx_scatter_pairs")

    def scatter_min(self, dense: bool, peer: bool = False):
        L, st = self.lib, self.stream.cuda_stream
        op = self._lib.PGX_OP_MIN_U32
        if not peer and self._use_seg(dense):
            # the dense CC supersteps: K1s into the full-width mailbox
            ix, _, ctr = self._ensure_seg()
            self._scattered = self.m_local if dense else self.E
            self._k(L.pgx_seg_scatter(0 if dense else 1, ctypes.byref(ix), self.m_local, self.npad,
                                      self.lo_own, None if dense else self.sv.data_ptr(),
                                      self.mailbox.data_ptr(), self.has.data_ptr(),
                                      EXCHANGE_NEUTRAL, ctr.data_ptr(), st), "pgx_seg_scatter")
            return
        if dense:
            src = (self._g_nz_eb.data_ptr(), None, self._g_nz_id.data_ptr(), self.lo_own, None,
                   self._g_tile.data_ptr(), self._nnz(), self.m_local)
            self._scattered = self.m_local
        else:
            src = (self.f_eb.data_ptr(), self.f_rs.data_ptr(), None, 0,
                   self.f_msg.data_ptr(), self.f_tile.data_ptr(), self.nsrc, self.E)
            self._scattered = self.E
        self._level += 1
        if peer and self.app == "sssp":
            # unit-weight SSSP: the exchange is the owners' has-bits
            rc = L.pgx_scatter_peer_bfs(self.col.data_ptr(), self.f_eb.data_ptr(),
                                        self.f_rs.data_ptr(), self.f_msg.data_ptr(),
                                        self.f_tile.data_ptr(), self.nsrc, self.E,
                                        self.has.data_ptr(), self._peer_has_ptrs.data_ptr(),
                                        self._pbounds.data_ptr(), self.world, self.blo,
                                        self.blo + self.block, st)
            self._k(rc, "pgx_scatter_peer_bfs")
            return
        if peer:
            rc = L.pgx_scatter_peer(int(dense), self.col.data_ptr(), *src,
                                    self.mailbox.data_ptr(), self.has.data_ptr(),
                                    EXCHANGE_NEUTRAL, self._peer_ptrs.data_ptr(),
                                    self._pbounds.data_ptr(), self.world, self.blo,
                                    self.blo + self.len, st)
            self._k(rc, "pgx_scatter_peer")
            return
        rc = L.pgx_scatter(op, int(dense), self.col.data_ptr(), *src,
                           self.mailbox.data_ptr(), self.has.data_ptr(), EXCHANGE_NEUTRAL, st)
        self._k(rc, "pgx_scatter")

    def apply_min(self, app, count_only: bool) -> torch.Tensor:
        """K2 on the owned block; returns the raw device counter block
        (decode_counts) -- no host synchronisation."""
        self.ctr.zero_()
        app_id = self._lib.PGX_APP_CC if app == "components" else self._lib.PGX_APP_SSSP
        own = self.has[self.blo // 32:(self.blo + self.block) // 32]
        if app == "sssp" and self._last == "peer":
            # the bitmap exchange: the owned block's bits are the recipients
            self._k(self.lib.pgx_apply_slice_bfs(
                self.len, self.row_ptr.data_ptr(), self.val.data_ptr(), own.data_ptr(),
                self.f_eb.data_ptr(), self.f_rs.data_ptr(), self.f_msg.data_ptr(),
                self.f_tile.data_ptr(), self.ctr.data_ptr(), int(count_only), self._level,
                self.stream.cuda_stream), "pgx_apply_slice_bfs", 1 if count_only else 2)
            return self.ctr[:24].view(torch.int64)
        sl = self.mailbox[self.blo:self.blo + self.len]
        sv = None
        if self.sv is not None:
            self.sv.fill_(-1)
            sv = self.sv.data_ptr()
        self._k(self.lib.pgx_apply_slice(
            app_id, self.len, self.row_ptr.data_ptr(), self.val.data_ptr(), sl.data_ptr(),
            self.f_eb.data_ptr(), self.f_rs.data_ptr(), self.f_msg.data_ptr(),
            self.f_tile.data_ptr(), self.ctr.data_ptr(), int(count_only), EXCHANGE_NEUTRAL,
            sv, self.stream.cuda_stream), "pgx_apply_slice")
        # the owned has-words (set by this rank's own scatter) are consumed
        # here, before the counters' all-gather lets any peer start the next
        # superstep
        own.zero_()
        return self.ctr[:24].view(torch.int64)  # the raw block: packed, recip, bcast

    @staticmethod
    def decode_counts(row):
        """(recipients, broadcasts, senders, edges) of a raw counter block."""
        packed = row[0] & 0xFFFFFFFFFFFFFFFF
        return row[1], row[2], packed >> 32, packed & 0xFFFFFFFF

    def set_frontier(self, senders: int, edges: int):
        self.nsrc, self.E = int(senders), int(edges)

    # ---- PageRank ----
    def _ensure_pull(self):
        """The rank's local in-CSR (rows = padded positions, entries = local
        sources in ascending order), its tile map and the rows that span
        tiles -- built once per layout (graph preparation)."""
        if self._pull is not None:
            return self._pull
        dev, st = self.device, self.stream
        with torch.cuda.device(dev), torch.cuda.stream(st):
            src = torch.repeat_interleave(
                torch.arange(self.len, dtype=torch.int32, device=dev),
                torch.diff(self.row_ptr).to(torch.int64))
            dst = self.col
            order = torch.sort(dst, stable=True).indices    # sources stay ascending
            in_col = src[order].contiguous()
            del src, order
            in_deg = torch.bincount(dst.to(torch.int64), minlength=self.npad)
            in_ptr64 = torch.zeros(self.npad + 1, dtype=torch.int64, device=dev)
            in_ptr64[1:] = torch.cumsum(in_deg, 0)
            in_ptr = in_ptr64.to(torch.int32)
            m = self.m_local
            ws_bytes = self._lib.out_size(self.lib.pgx_graph_workspace_bytes, self.npad, m)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            self._lib.check(self.lib.pgx_graph_prepare(self.npad, m, in_ptr.data_ptr(),
                                                       ws.data_ptr(), ws_bytes, st.cuda_stream),
                            "pgx_graph_prepare")
            nz = in_deg > 0
            a = in_ptr64[:-1] // 256
            b = (in_ptr64[1:] - 1) // 256
            rows = torch.nonzero(nz & (a != b)).flatten()
            ntile = (m + 255) // 256 + 2
            self._pull = {
                "in_col": in_col, "in_ptr": in_ptr, "ws": ws, "nsrc": int(nz.sum()),
                "span_rows": rows.to(torch.int32), "span_t0": a[rows].to(torch.int32),
                "span_t1": b[rows].to(torch.int32),
                "head": torch.zeros(ntile, dtype=torch.float64, device=dev),
                "tail": torch.zeros(ntile, dtype=torch.float64, device=dev)}
        return self._pull

    def init_pagerank(self, r0) -> int:
        self.app = "pagerank"
        self.mailbox = torch.zeros(self.npad, dtype=torch.float64, device=self.device)
        self.rank_v = torch.empty(max(self.len, 1), dtype=torch.float64, device=self.device)
        self.share = torch.empty(max(self.len, 1), dtype=torch.float64, device=self.device)
        self._k(self.lib.pgx_slice_init(self._lib.PGX_APP_PAGERANK, self.len, self.lo_own,
                                        self.rank_v.data_ptr(), self.row_ptr.data_ptr(),
                                        self.share.data_ptr(), r0,
                                        self.stream.cuda_stream), "pgx_slice_init")
        self.partials = torch.zeros((self.len + 511) // 512 + 1, dtype=torch.float64,
                                    device=self.device)
        if self.pr_mode == "pull" and self.m_local > 0:
            self._ensure_pull()
        deg = torch.diff(self.row_ptr)
        return int((deg == 0).sum())

    def fold_sum(self):
        """This rank's partial fold of every destination into the full-width
        mailbox: the pull fold (K3) by default, the red.add.f64 scatter for
        pr_mode="push"."""
        st = self.stream.cuda_stream
        self.mailbox.zero_()
        if self.m_local == 0:
            return
        if self.pr_mode == "push":
            self._k(self.lib.pgx_scatter(
                self._lib.PGX_OP_SUM_F64, 1, self.col.data_ptr(), self._g_nz_eb.data_ptr(),
                None, self._g_nz_id.data_ptr(), 0, self.share.data_ptr(),
                self._g_tile.data_ptr(), self._nnz(), self.m_local, self.mailbox.data_ptr(),
                None, 0, st), "pgx_scatter")
            return
        p = self._pull
        self._k(self.lib.pgx_gather_slice(self.npad, self.m_local, p["in_col"].data_ptr(),
                                          p["ws"].data_ptr(), p["nsrc"], self.share.data_ptr(),
                                          self.mailbox.data_ptr(), p["head"].data_ptr(),
                                          p["tail"].data_ptr(), st), "pgx_gather_slice")
        ns = int(p["span_rows"].numel())
        if ns:
            self._k(self.lib.pgx_fold_spanning(ns, p["span_rows"].data_ptr(),
                                               p["span_t0"].data_ptr(), p["span_t1"].data_ptr(),
                                               p["head"].data_ptr(), p["tail"].data_ptr(),
                                               self.mailbox.data_ptr(), st), "pgx_fold_spanning")

    def apply_pagerank(self, base, damping, dangling: torch.Tensor, last: bool) -> torch.Tensor:
        """Apply on the owned block; returns this rank's dangling mass as a
        one-element device tensor (no host read)."""
        sl = self.mailbox[self.blo:self.blo + self.len]
        nb = (self.len + 511) // 512
        self._k(self.lib.pgx_pr_apply_slice(
            self.len, self.row_ptr.data_ptr(), self.rank_v.data_ptr(), sl.data_ptr(),
            self.share.data_ptr(), base, damping, dangling.data_ptr(), float(self.n), int(last),
            self.partials.data_ptr(), self.stream.cuda_stream), "pgx_pr_apply_slice")
        return self.partials[:nb].sum().reshape(1)

    def values(self):
        if self.app == "pagerank":
            return self.rank_v[:self.len]
        return self.val[:self.len]


class PartitionedPlan:
    """A partitioned run prepared on this rank (local CSR slice, tile map,
    padded layout, peer mappings cached on the graph): ``launch()`` runs the
    superstep loop with the result left on the device, ``collect()``
    gathers it."""

    def __init__(self, graph, program, low, config, dist):
        rank, world = dist.get_rank(), dist.get_world_size()
        self.n, self.m = graph.vertex_count, graph.edge_count
        dev = torch.device("cuda", torch.cuda.current_device())
        pr_mode = getattr(config, "pagerank_mode", "pull")
        segments = getattr(config, "segments", "auto")
        key = ("partitioned", world, rank, dev.index, pr_mode, segments)
        cached = graph._device.get(key)
        if cached is None:  # local CSR slice + its tile map, built once per graph
            deg = torch.diff(graph.out_offsets.cpu()).numpy()
            bounds = partition_bounds(deg, world)
            backend = CudaBackend(graph, int(bounds[rank]), int(bounds[rank + 1]), dev,
                                  pr_mode=pr_mode, segments=segments)
            cached = graph._device[key] = (bounds, backend)
        self.bounds, self.backend = cached
        self.runner = PartitionedRun(self.backend, dist, self.bounds, self.n, self.m)
        self.runner.exchange = os.environ.get("PGX_EXCHANGE", "auto")
        self.program, self.low, self.config = program, low, config
        self.app = low["app"]
        self.stream = self.backend.stream
        self._out = None

    def launch(self) -> None:
        """Every superstep of one run (host-driven; values stay on the GPU)."""
        if self.app == "pagerank":
            self._out = self.runner.loop_pagerank(self.low["iterations"], self.low["damping"],
                                                  self.config.max_supersteps)
        else:
            self._out = self.runner.loop_min(self.app, self.low.get("source", 0),
                                             self.config.max_supersteps)

    @property
    def launches(self) -> int:
        """libpgx kernels this rank has launched so far."""
        return self.backend.launches

    def collect(self):
        from .engine import RunReport, SuperstepStats
        stats, cap, wall = self._out
        vals = self.runner._gather_values()
        if self.app == "pagerank":
            values = vals.cpu().numpy()
        else:
            v = vals.cpu().numpy().view(np.uint32)
            values = v.astype(np.int64) if self.app == "components" else v
        steps = [SuperstepStats(**{k: v for k, v in s.items() if k != "exchange"})
                 for s in stats]
        if self.program.extract is not None:
            from types import SimpleNamespace
            values = self.program.extract(SimpleNamespace(state=values,
                                                          halted=np.ones(values.shape[0], bool)))
        return RunReport(values, len(steps), steps, wall, cap, device_values=vals,
                         exchanges=[s.get("exchange", "dense") for s in stats])


def plan_partitioned(graph, program, low, config, dist) -> PartitionedPlan:
    return PartitionedPlan(graph, program, low, config, dist)


def run_partitioned(graph, program, low, config, dist):
    """engine.run() under torchrun: every rank calls run() with the graph."""
    plan = plan_partitioned(graph, program, low, config, dist)
    plan.launch()
    return plan.collect()
