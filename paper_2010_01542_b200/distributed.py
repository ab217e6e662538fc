"""Partitioned multi-GPU superstep, one process per GPU.

The reference has no distributed mode (SPEC.md:420 non-goal); this is the
B200 build's scale-out of the same superstep, with results identical to
one GPU (CC labels / SSSP distances bit-exact, PageRank within 1e-9):

* **partition**: 1-D by source vertex.  Rank r owns the contiguous vertex
  range ``[lo_r, hi_r)`` -- its out-edges (a local CSR with GLOBAL
  destination ids) and that slice of the mailbox.  Ranges follow the
  reference's exact integer edge-balance rule (``edge_balanced_partition``,
  scheduler.py:91-116) over ``out_degree + 1`` (edges + vertex work);
* **per superstep**: every rank scatters its senders into a full-width
  local mailbox (``pgx_scatter``); one reduction per owner delivers the
  combined slice (``min`` for CC/SSSP, ``sum`` for PageRank) -- issued as
  ``len(world)`` ``reduce`` calls, which NCCL runs over NVLink/NVSwitch;
  the owner applies on its slice (``pgx_apply_slice`` /
  ``pgx_pr_apply_slice``); an ``all_reduce`` of the counters (recipients,
  broadcasts, senders, edges, dangling mass) drives the halt test.  No
  all-gather is needed: a sender is always local to its owner.
* has-message after the reduction is ``mailbox != neutral``: CC / SSSP
  messages are < n <= 2^31 and never equal UINT32_MAX, and PageRank needs
  no flag (the paper's neutral-value caveat).
* **fused peer exchange** (min programs, the default when every rank can
  map every other rank's mailbox): the scatter kernel itself combines each
  message that passes its local filter into the OWNER's mailbox slot over
  NVLink peer memory (``pgx_scatter_peer``: one fire-and-forget
  ``red.min`` per surviving foreign message, a system-scope fence at the
  end), so the mailbox is never reduced by a collective: a one-element
  all-reduce after the scatter orders the peers' combines before the
  owners' apply.  Mailboxes are ``cudaMalloc`` blocks shared by CUDA IPC
  (``pgx_peer_alloc`` / ``pgx_peer_open``); ranks that are threads of one
  process use the raw pointers.  The choice is collective: if any rank
  cannot map a peer, every rank falls back to the collective exchanges.
* **sparse exchange** (SURVEY 8(f) row 3): late supersteps touch few
  mailbox slots, yet the dense reduction always moves n slots.  Every rank
  counts the slots it touched outside its own range (has-bits of the
  scatter); when the largest count makes 8-byte (slot, value) pairs cheaper
  than half the dense volume, the ranks compact their touched slots in
  vertex order (grouped by owner) and exchange them with one variable-size
  ``all_to_all_single``; owners min-combine what they receive.  The choice
  is collective (an all-reduce of the counts) and recorded per superstep.

The orchestration below is backend-agnostic: ``CudaBackend`` drives
libpgx.so on the rank's GPU (NCCL process group); tests/ drive the same
``PartitionedRun`` with a CPU test backend over a gloo process group.
"""

from __future__ import annotations

import ctypes
import os
import time
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from .scheduler import edge_balanced_partition

#: min neutral of the exchanged mailbox: INT32_MAX, so that the signed
#: int32 MIN reduction of NCCL / gloo is exact (messages are < n < 2^31 - 1)
EXCHANGE_NEUTRAL = 2 ** 31 - 1


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
    """Owner ranges ``bounds[r]..bounds[r+1]`` (edge + vertex balanced)."""
    deg = np.asarray(out_degrees, dtype=np.int64)
    return edge_balanced_partition(deg + 1, world).boundaries.astype(np.int64)


@dataclass
class StepCounts:
    recipients: int
    broadcasts: int
    senders: int
    edges: int
    dangling: float = 0.0


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
        # min-program exchange: "auto" (peer if every rank maps every peer,
        # else hybrid), "peer", "hybrid" (dense / sparse per superstep),
        # "dense" (A/B switches)
        self.exchange = "auto"
        self._coalesced = None  # NCCL uneven reduce_scatter available?
        be = str(getattr(dist, "get_backend", lambda: "")())
        # gloo has no CUDA all_gather: small collectives go through the host
        self._host_coll = be == "gloo" and self.b.device.type == "cuda"
        self._cdev = torch.device("cpu") if self._host_coll else self.b.device

    @property
    def sparse_ok(self) -> bool:
        return self.exchange != "dense"

    @sparse_ok.setter
    def sparse_ok(self, ok: bool):
        self.exchange = "auto" if ok else "dense"

    def _coll_sync(self):
        """Before a host-side collective: the rank's kernels have finished."""
        if self._host_coll:
            torch.cuda.current_stream(self.b.device).synchronize()

    def _peer_setup(self) -> bool:
        """Map every rank's mailbox on every rank (collective decision).

        The outcome is cached on the rank's backend (cached per graph, so
        every rank of a job holds the same cache state): later runs on the
        same backend skip the handle exchange."""
        cached = getattr(self.b, "_peer_decision", None)
        if cached is not None and cached[0] == self.exchange:
            self.b.peer_active = cached[1]
            return cached[1]
        if self.exchange not in ("auto", "peer") or not hasattr(self.b, "peer_handle"):
            want = False
        else:
            want = True
        h = self.b.peer_handle() if want else None
        handles = [None] * self.world
        self.dist.all_gather_object(handles, h)
        ok = all(x is not None for x in handles) and self.b.open_peers(handles, self.bounds)
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
        """Deliver every owner the reduction of its mailbox slice."""
        if self._host_coll:  # gloo: stage the mailbox through the host
            self._coll_sync()
            full = self.b.mailbox.cpu()
            for r in range(self.world):
                part = full[int(self.bounds[r]):int(self.bounds[r + 1])]
                if part.numel():
                    self.dist.reduce(part, dst=r, op=op)
            self.b.mailbox[self.lo:self.hi].copy_(full[self.lo:self.hi])
            return
        full = self.b.mailbox
        parts = [full[int(self.bounds[r]):int(self.bounds[r + 1])] for r in range(self.world)]
        backend = getattr(self.dist, "get_backend", lambda: None)()
        if self._coalesced is not False and str(backend) == "nccl":
            # one uneven reduce_scatter: NCCL coalesces the per-owner reduces
            try:
                self.dist.reduce_scatter(parts[self.rank], parts, op=op)
                self._coalesced = True
                return
            except Exception:  # pragma: no cover - torch without uneven support
                self._coalesced = False
        for r, part in enumerate(parts):
            if part.numel():
                self.dist.reduce(part, dst=r, op=op)

    def _exchange_min(self, op, allow_sparse: bool = True) -> str:
        """Dense per-owner reduction or sparse pair exchange (collective choice)."""
        if not allow_sparse:  # a big superstep: dense, no count, no host sync
            self._reduce_slices(op)
            self.b.dense_exchanged()
            return "dense"
        touched = self.b.touched_count()
        t = torch.tensor([touched], dtype=torch.int64, device=self._cdev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        if self.exchange != "dense" and 8 * int(t.item()) * 2 < 4 * self.n:
            pairs, splits = self.b.compact_touched(self.bounds)
            pairs = pairs.to(self._cdev)
            sc = torch.tensor(splits, dtype=torch.int64, device=self._cdev)
            rc = torch.empty_like(sc)
            self.dist.all_to_all_single(rc, sc)
            recv_splits = rc.tolist()
            recv = torch.empty(sum(recv_splits), dtype=torch.int64, device=self._cdev)
            self.dist.all_to_all_single(recv, pairs, recv_splits, list(splits))
            self.b.scatter_pairs(recv.to(self.b.device))
            return "sparse"
        self._reduce_slices(op)
        self.b.dense_exchanged()
        return "dense"

    def _gather_counts(self, local: torch.Tensor) -> StepCounts:
        """Every rank's (recipients, broadcasts, senders, edges) in ONE
        all-gather and one host read: the sums drive the halt test and the
        statistics, the rank's own senders / edges size its next scatter."""
        local = local.to(device=self._cdev, dtype=torch.int64)
        parts = [torch.empty_like(local) for _ in range(self.world)]
        self._coll_sync()
        self.dist.all_gather(parts, local)
        rows = [self.b.decode_counts(r) for r in torch.stack(parts).tolist()]
        self.b.set_frontier(rows[self.rank][2], rows[self.rank][3])
        tot = [sum(r[i] for r in rows) for i in range(4)]
        return StepCounts(*tot)

    def _allreduce_counts(self, c: StepCounts) -> StepCounts:
        t = torch.tensor([c.recipients, c.broadcasts, c.senders, c.edges],
                         dtype=torch.int64, device=self._cdev)
        self._coll_sync()
        self.dist.all_reduce(t)
        d = torch.tensor([c.dangling], dtype=torch.float64, device=self._cdev)
        self.dist.all_reduce(d)
        v = t.tolist()
        return StepCounts(v[0], v[1], v[2], v[3], float(d.item()))

    def _gather_values(self):
        local = self.b.values().to(self._cdev)
        sizes = np.diff(self.bounds)
        mx = int(sizes.max())
        pad = torch.zeros(mx, dtype=local.dtype, device=local.device)
        pad[:local.numel()] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad)
        return torch.cat([parts[r][:int(sizes[r])] for r in range(self.world)])

    # ---- min programs: CC / SSSP -------------------------------------

    def run_min(self, app: str, source: int, max_steps: int):
        op = self.dist.ReduceOp.MIN
        n = self.n
        peer_ok = self._peer_setup()
        self.b.init_min(app, self.lo, self.hi)
        if peer_ok:  # every mailbox is neutral before any peer combines into it
            self._fence()
        stats = []
        if app == "sssp":
            own = self.lo <= source < self.hi
            deg = self.b.global_out_degree(source)
            if own:
                self.b.seed_source(source - self.lo)
            nxt = StepCounts(0, 1, 1 if deg > 0 else 0, deg)
        else:
            nxt = StepCounts(0, n, self.b.global_nonzero_degree(), self.m)
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
            self.b.scatter_min(dense=(app == "components" and s == 0),
                               id_offset=self.lo, peer=use_peer)
            if use_peer:
                self._fence()
                exchange = "peer"
            else:  # auto with the peer path mapped: only big supersteps get here
                exchange = self._exchange_min(op, allow_sparse=not peer_ok)
            self.b.exchanged(exchange)
            at_cap = s + 1 == max_steps
            nxt = self._gather_counts(self.b.apply_min(app, count_only=at_cap))
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
        values = self._gather_values()
        return values, stats, hit_cap, time.perf_counter() - t0

    # ---- PageRank -------------------------------------------------------

    def run_pagerank(self, iterations: int, damping: float, max_steps: int):
        op = self.dist.ReduceOp.SUM
        n = self.n
        base = (1.0 - damping) / n      # algorithms.py:49
        r0 = 1.0 / n                    # algorithms.py:50
        last = iterations - 1
        ndangling = self.b.init_pagerank(self.lo, self.hi, r0)
        t = torch.tensor([ndangling], dtype=torch.int64, device=self._cdev)
        self.dist.all_reduce(t)
        ndangling = int(t.item())
        dangling = r0 * ndangling       # algorithms.py:55
        nspread = n - ndangling
        stats = []
        t0 = time.perf_counter()
        steps = min(max_steps, iterations)
        for s in range(steps):
            ts = time.perf_counter()
            # the fold of superstep s: shares broadcast at s-1 (or the seed)
            self.b.reset_mailbox()
            self.b.scatter_sum()
            self._reduce_slices(op)
            local_d = self.b.apply_pagerank(base, damping, dangling / n, s == last)
            d = torch.tensor([local_d], dtype=torch.float64, device=self._cdev)
            self.dist.all_reduce(d)
            dangling = float(d.item())
            stats.append(dict(index=s, active_count=n,
                              messages_sent=0 if s == last else nspread,
                              edges=self.m, senders=nspread, recipients=n,
                              broadcasters=0 if s == last else nspread,
                              seconds=time.perf_counter() - ts))
        hit_cap = steps < iterations  # engine.py:299-300
        values = self._gather_values()
        return values, stats, hit_cap, time.perf_counter() - t0


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
        self.handle = handle.raw
        self.tensor = torch.as_tensor(_DeviceArray(self.ptr, n, "<i4"), device=device)
        # freed with its owner (the backend drops it only after its last run)
        weakref.finalize(self, lib.pgx_peer_free, ctypes.c_void_p(self.ptr))


class CudaBackend:
    """Owns the rank's local CSR, full-width mailbox and owned-slice state."""

    def __init__(self, graph, lo: int, hi: int, device):
        from . import _lib
        self._lib = _lib
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.stream = torch.cuda.current_stream(self.device)
        dev = self.device
        # slice where the graph lives and upload only this rank's rows (a
        # pinned host graph stays pinned under slicing: one DMA per array)
        off = graph.out_offsets
        self.n = graph.vertex_count
        self._glob_off = off
        base, end = int(off[lo]), int(off[hi])
        self.row_ptr = (off[lo:hi + 1] - base).to(dev, non_blocking=True) \
            .to(torch.int32).contiguous()
        self.col = graph.out_targets[base:end].to(dev, non_blocking=True) \
            .to(torch.int32).contiguous()
        self.len = hi - lo
        self.m_local = int(self.col.numel())
        st = self.stream.cuda_stream
        ws_bytes = _lib.out_size(self.lib.pgx_graph_workspace_bytes, max(self.len, 1),
                                 self.m_local)
        self.gws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        if self.len > 0:
            _lib.check(self.lib.pgx_graph_prepare(self.len, self.m_local,
                                                  self.row_ptr.data_ptr(),
                                                  self.gws.data_ptr(), ws_bytes, st),
                       "pgx_graph_prepare")
        # graph workspace layout (pgx_engine.cu graph_ws_layout): hdr, nz_id,
        # nz_eb, tile_src, blk -- 256-byte aligned chunks
        al = lambda x: (x + 255) // 256 * 256
        o_id = al(16)
        o_eb = o_id + al(4 * (self.len + 1))
        o_tile = o_eb + al(4 * (self.len + 1))
        self._g_hdr = self.gws[:16].view(torch.int32)
        self._g_nz_id = self.gws[o_id:o_id + 4 * (self.len + 1)].view(torch.int32)
        self._g_nz_eb = self.gws[o_eb:o_eb + 4 * (self.len + 1)].view(torch.int32)
        ntile = (self.m_local + 255) // 256 + 2
        self._g_tile = self.gws[o_tile:o_tile + 4 * ntile].view(torch.int32)
        cb = _lib.out_size(self.lib.pgx_slice_counters_bytes)
        self.ctr = torch.zeros(cb, dtype=torch.uint8, device=dev)
        self.f_eb = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_rs = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_msg = torch.empty(self.len + 1, dtype=torch.int32, device=dev)
        self.f_tile = torch.empty(ntile, dtype=torch.int32, device=dev)
        self.nsrc, self.E = 0, 0
        self.lo_own, self.hi_own = lo, hi
        self.has = torch.zeros(self.n // 32 + 2, dtype=torch.int32, device=dev)
        sb = _lib.out_size(self.lib.pgx_touched_scratch_bytes, self.n)
        self.tscratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        self.tcount = torch.zeros(1, dtype=torch.int64, device=dev)
        self._last = None
        # fused peer exchange state (PartitionedRun._peer_setup)
        self.peer_active = False
        self._peer_mb = None
        self._peer_sig = None
        self._opened = []
        # peer mappings are closed when the backend goes away
        weakref.finalize(self, CudaBackend._close_all, self.lib, self._opened)

    @staticmethod
    def _close_all(lib, opened):
        for p in opened:
            lib.pgx_peer_close(ctypes.c_void_p(p))
        opened.clear()

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

    def _counters(self):
        c = self.ctr[:32].view(torch.int64).tolist()
        d = float(self.ctr[24:32].view(torch.float64).item())
        return c, d

    # ---- min programs ----
    # ---- fused peer exchange ----
    def peer_handle(self):
        """This rank's mappable mailbox (allocated once), or None."""
        try:
            if self._peer_mb is None:
                self._peer_mb = PeerMailbox(self._lib, self.lib, self.n, self.device)
        except Exception:
            return None
        return {"pid": os.getpid(), "ptr": self._peer_mb.ptr, "handle": self._peer_mb.handle}

    def close_peers(self):
        CudaBackend._close_all(self.lib, self._opened)  # in place: the finalizer's list
        self._peer_sig = None

    def open_peers(self, handles, bounds) -> bool:
        """Device array of every rank's mailbox base (IPC-mapped, or the raw
        pointer for ranks that are threads of this process)."""
        sig = tuple((h["pid"], h["ptr"]) for h in handles)
        if sig == self._peer_sig:
            return True
        self.close_peers()
        ptrs = []
        try:
            for h in handles:
                if h["pid"] == os.getpid():
                    ptrs.append(h["ptr"])
                    continue
                p = ctypes.c_void_p()
                self._lib.check(self.lib.pgx_peer_open(h["handle"], ctypes.byref(p)),
                                "pgx_peer_open")
                self._opened.append(int(p.value))
                ptrs.append(int(p.value))
        except Exception:
            self.close_peers()
            return False
        self._peer_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        self._bounds32 = torch.tensor(np.asarray(bounds), dtype=torch.int32, device=self.device)
        self._world = len(handles)
        self._peer_sig = sig
        return True

    def init_min(self, app, lo, hi):
        self.app = app
        self.lo = lo
        if self.peer_active:
            self.mailbox = self._peer_mb.tensor
        else:
            self.mailbox = torch.empty(self.n, dtype=torch.int32, device=self.device)
        self.mailbox.fill_(EXCHANGE_NEUTRAL)
        self.has.zero_()
        self.val = torch.empty(max(self.len, 1), dtype=torch.int32, device=self.device)
        app_id = self._lib.PGX_APP_CC if app == "components" else self._lib.PGX_APP_SSSP
        self._lib.check(self.lib.pgx_slice_init(app_id, self.len, lo, self.val.data_ptr(),
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
        owned slice is always neutral here (the apply consumed it), and it
        is never written: a peer may already be combining into it."""
        if self.app == "pagerank":
            self.mailbox.zero_()
            return
        if self._last == "peer":  # foreign filter copies back to neutral, bits cleared
            self._lib.check(self.lib.pgx_reset_touched(
                self.n, self.lo_own, self.hi_own, self.has.data_ptr(), self.mailbox.data_ptr(),
                EXCHANGE_NEUTRAL, self.stream.cuda_stream), "pgx_reset_touched")
            return
        if self._last == "dense":  # every foreign slot holds a stale partial
            self.mailbox[:self.lo_own].fill_(EXCHANGE_NEUTRAL)
            self.mailbox[self.hi_own:].fill_(EXCHANGE_NEUTRAL)
        # sparse: the compaction reset the foreign touched slots
        if self._last is not None:
            self.has.zero_()

    def exchanged(self, kind: str):
        self._last = kind

    def dense_exchanged(self):
        pass  # recorded by exchanged("dense")

    def touched_count(self) -> int:
        self._lib.check(self.lib.pgx_touched(
            self.n, self.lo_own, self.hi_own, self.has.data_ptr(), None, EXCHANGE_NEUTRAL,
            None, self.tcount.data_ptr(), self.tscratch.data_ptr(), self.stream.cuda_stream),
            "pgx_touched")
        return int(self.tcount.item())

    def compact_touched(self, bounds):
        cnt = int(self.tcount.item())
        pairs = torch.empty(max(cnt, 1), dtype=torch.int64, device=self.device)
        self._lib.check(self.lib.pgx_touched(
            self.n, self.lo_own, self.hi_own, self.has.data_ptr(), self.mailbox.data_ptr(),
            EXCHANGE_NEUTRAL, pairs.data_ptr(), self.tcount.data_ptr(),
            self.tscratch.data_ptr(), self.stream.cuda_stream), "pgx_touched")
        pairs = pairs[:cnt]
        slots = pairs >> 32
        b = torch.as_tensor(bounds[1:-1], dtype=torch.int64, device=self.device)
        owner = torch.searchsorted(b, slots, right=True)
        splits = torch.bincount(owner, minlength=len(bounds) - 1).tolist()
        return pairs, splits

    def scatter_pairs(self, pairs):
        self._lib.check(self.lib.pgx_scatter_pairs(pairs.data_ptr(), pairs.numel(),
                                                   self.mailbox.data_ptr(),
                                                   self.stream.cuda_stream), "pgx_scatter_pairs")

    def scatter_min(self, dense: bool, id_offset: int, peer: bool = False):
        L, st = self.lib, self.stream.cuda_stream
        op = self._lib.PGX_OP_MIN_U32
        if peer:
            if dense:
                src = (self._g_nz_eb.data_ptr(), None, self._g_nz_id.data_ptr(), id_offset, None,
                       self._g_tile.data_ptr(), self._nnz(), self.m_local)
            else:
                src = (self.f_eb.data_ptr(), self.f_rs.data_ptr(), None, 0,
                       self.f_msg.data_ptr(), self.f_tile.data_ptr(), self.nsrc, self.E)
            rc = L.pgx_scatter_peer(int(dense), self.col.data_ptr(), *src,
                                    self.mailbox.data_ptr(), self.has.data_ptr(),
                                    EXCHANGE_NEUTRAL, self._peer_ptrs.data_ptr(),
                                    self._bounds32.data_ptr(), self._world, self.lo_own,
                                    self.hi_own, st)
            self._lib.check(rc, "pgx_scatter_peer")
            return
        if dense:
            nnz = self._nnz()
            rc = L.pgx_scatter(op, 1, self.col.data_ptr(), self._g_nz_eb.data_ptr(), None,
                               self._g_nz_id.data_ptr(), id_offset, None,
                               self._g_tile.data_ptr(), nnz, self.m_local,
                               self.mailbox.data_ptr(), self.has.data_ptr(),
                               EXCHANGE_NEUTRAL, st)
        else:
            rc = L.pgx_scatter(op, 0, self.col.data_ptr(), self.f_eb.data_ptr(),
                               self.f_rs.data_ptr(), None, 0, self.f_msg.data_ptr(),
                               self.f_tile.data_ptr(), self.nsrc, self.E,
                               self.mailbox.data_ptr(), self.has.data_ptr(),
                               EXCHANGE_NEUTRAL, st)
        self._lib.check(rc, "pgx_scatter")

    def apply_min(self, app, count_only: bool) -> torch.Tensor:
        """K2 on the owned slice; returns the raw device counter block
        (decode_counts) -- no host synchronisation, no extra kernels."""
        self.ctr.zero_()
        app_id = self._lib.PGX_APP_CC if app == "components" else self._lib.PGX_APP_SSSP
        sl = self.mailbox[self.lo:self.lo + self.len]
        self._lib.check(self.lib.pgx_apply_slice(
            app_id, self.len, self.row_ptr.data_ptr(), self.val.data_ptr(), sl.data_ptr(),
            self.f_eb.data_ptr(), self.f_rs.data_ptr(), self.f_msg.data_ptr(),
            self.f_tile.data_ptr(), self.ctr.data_ptr(), int(count_only), EXCHANGE_NEUTRAL,
            self.stream.cuda_stream), "pgx_apply_slice")
        return self.ctr[:24].view(torch.int64)  # the raw block: packed, recip, bcast

    @staticmethod
    def decode_counts(row):
        """(recipients, broadcasts, senders, edges) of a raw counter block."""
        packed = row[0] & 0xFFFFFFFFFFFFFFFF
        return row[1], row[2], packed >> 32, packed & 0xFFFFFFFF

    def set_frontier(self, senders: int, edges: int):
        self.nsrc, self.E = int(senders), int(edges)

    # ---- PageRank ----
    def init_pagerank(self, lo, hi, r0) -> int:
        self.app = "pagerank"
        self.lo = lo
        self.mailbox = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        self.rank = torch.empty(max(self.len, 1), dtype=torch.float64, device=self.device)
        self.share = torch.empty(max(self.len, 1), dtype=torch.float64, device=self.device)
        self._lib.check(self.lib.pgx_slice_init(self._lib.PGX_APP_PAGERANK, self.len, lo,
                                                self.rank.data_ptr(), self.row_ptr.data_ptr(),
                                                self.share.data_ptr(), r0,
                                                self.stream.cuda_stream), "pgx_slice_init")
        self.partials = torch.zeros((self.len + 511) // 512 + 1, dtype=torch.float64,
                                    device=self.device)
        deg = torch.diff(self.row_ptr)
        return int((deg == 0).sum())

    def scatter_sum(self):
        nnz = self._nnz()
        self._lib.check(self.lib.pgx_scatter(
            self._lib.PGX_OP_SUM_F64, 1, self.col.data_ptr(), self._g_nz_eb.data_ptr(), None,
            self._g_nz_id.data_ptr(), 0, self.share.data_ptr(), self._g_tile.data_ptr(), nnz,
            self.m_local, self.mailbox.data_ptr(), None, 0, self.stream.cuda_stream),
            "pgx_scatter")

    def apply_pagerank(self, base, damping, dn, last: bool) -> float:
        sl = self.mailbox[self.lo:self.lo + self.len]
        self._lib.check(self.lib.pgx_pr_apply_slice(
            self.len, self.row_ptr.data_ptr(), self.rank.data_ptr(), sl.data_ptr(),
            self.share.data_ptr(), base, damping, dn, int(last), self.partials.data_ptr(),
            self.stream.cuda_stream), "pgx_pr_apply_slice")
        return float(self.partials[:(self.len + 511) // 512].sum().item())

    def values(self):
        if self.app == "pagerank":
            return self.rank[:self.len]
        return self.val[:self.len]


def run_partitioned(graph, program, low, config, dist):
    """engine.run() under torchrun: every rank calls run() with the graph."""
    from .engine import RunReport, SuperstepStats
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = graph.vertex_count, graph.edge_count
    dev = torch.device("cuda", torch.cuda.current_device())
    key = ("partitioned", world, rank, dev.index)
    cached = graph._device.get(key)
    if cached is None:  # local CSR slice + its tile map, built once per graph
        deg = torch.diff(graph.out_offsets.cpu()).numpy()
        bounds = partition_bounds(deg, world)
        backend = CudaBackend(graph, int(bounds[rank]), int(bounds[rank + 1]), dev)
        cached = graph._device[key] = (bounds, backend)
    bounds, backend = cached
    runner = PartitionedRun(backend, dist, bounds, n, m)
    runner.exchange = os.environ.get("PGX_EXCHANGE", "auto")
    app = low["app"]
    if app == "pagerank":
        vals, stats, cap, wall = runner.run_pagerank(low["iterations"], low["damping"],
                                                     config.max_supersteps)
        values = vals.cpu().numpy()
    else:
        vals, stats, cap, wall = runner.run_min(app, low.get("source", 0),
                                                config.max_supersteps)
        v = vals.cpu().numpy().view(np.uint32)
        values = v.astype(np.int64) if app == "components" else v
    steps = [SuperstepStats(**{k: v for k, v in s.items() if k != "exchange"}) for s in stats]
    if program.extract is not None:
        from types import SimpleNamespace
        values = program.extract(SimpleNamespace(state=values,
                                                 halted=np.ones(values.shape[0], bool)))
    return RunReport(values, len(steps), steps, wall, cap, device_values=vals,
                     exchanges=[s.get("exchange", "dense") for s in stats])
