"""CPU stand-in for CudaBackend -- TEST INFRASTRUCTURE ONLY.

Mirrors the semantics of libpgx's phase kernels (pgx_scatter,
pgx_scatter_peer, pgx_reset_touched, pgx_touched, pgx_apply_slice,
pgx_gather_slice + pgx_fold_spanning, pgx_pr_apply_slice) with numpy on CPU
torch tensors and the same owner-blocked padded mailbox layout, so that
the partitioned driver (paper_2010_01542_b200.distributed.PartitionedRun:
partitioning, block reduce_scatter, sparse pairs, peer exchange, counter
all-gather, halt test, value gather) runs over a gloo process group
without a GPU.  The peer exchange maps the ranks' mailboxes as
shared-memory files (the stand-in for CUDA IPC); an flock per owner
serialises the read-modify-write of its block (the GPU's red.min is atomic).
"""

from __future__ import annotations

import fcntl
import os
import tempfile

import numpy as np
import torch

from paper_2010_01542_b200.distributed import EXCHANGE_NEUTRAL, padded_positions


class CpuBackend:
    def __init__(self, off, tgt, lo, hi):
        self.device = torch.device("cpu")
        off = np.asarray(off, np.int64)
        self.n = off.size - 1
        self.glob_deg = np.diff(off)
        self.lo, self.hi, self.len = lo, hi, hi - lo
        base = off[lo]
        self.row_ptr = off[lo:hi + 1] - base
        self.col_global = np.asarray(tgt[base:off[hi]], np.int64)
        self.deg = np.diff(self.row_ptr)
        self.front = (np.empty(0, np.int64), np.empty(0, np.int64))  # (local ids, msgs)
        self._last = None
        self.peer_active = False
        self._shm = None
        self._peers = None

    def bind(self, bounds, rank, block):
        self.rank, self.block, self.world = rank, block, len(bounds) - 1
        self.npad = self.world * block
        self.blo = rank * block
        self.col = padded_positions(torch.from_numpy(self.col_global), bounds,
                                    block).numpy().astype(np.int64)
        self.has = np.zeros(self.npad, bool)

    # ---- peer exchange (shared-memory stand-in for CUDA IPC) ----
    def peer_handle(self):
        if self._shm is None:
            fd, path = tempfile.mkstemp(prefix="pgx_peer_", dir="/dev/shm"
                                        if os.path.isdir("/dev/shm") else None)
            os.close(fd)
            self._shm = (path, np.memmap(path, dtype=np.int32, mode="w+",
                                         shape=(max(self.npad, 1),)))
        return {"pid": os.getpid(), "path": self._shm[0]}

    def open_peers(self, handles):
        self._peers = [np.memmap(h["path"], dtype=np.int32, mode="r+", shape=(max(self.npad, 1),))
                       for h in handles]
        self._locks = [open(h["path"], "rb") for h in handles]
        self._me = [h["path"] for h in handles].index(self._shm[0])
        return True

    def _locked_min(self, owner, dst, m):
        fcntl.flock(self._locks[owner], fcntl.LOCK_EX)
        try:
            np.minimum.at(self._peers[owner], dst, m)
        finally:
            fcntl.flock(self._locks[owner], fcntl.LOCK_UN)

    def close(self):
        if self._shm is not None:
            os.unlink(self._shm[0])
            self._shm = None

    def global_out_degree(self, v):
        return int(self.glob_deg[v])

    def global_nonzero_degree(self):
        return int((self.glob_deg > 0).sum())

    def _edges_of(self, lv, msg):
        if lv.size == 0:
            return np.empty(0, np.int64), np.empty(0, msg.dtype)
        reps = self.deg[lv]
        starts = self.row_ptr[lv]
        flat = np.repeat(starts - np.cumsum(reps) + reps, reps) + np.arange(reps.sum())
        return self.col[flat], np.repeat(msg, reps)

    # ---- min programs ----
    def init_min(self, app):
        self.app = app
        if self.peer_active:
            self.mailbox = torch.from_numpy(self._shm[1][:self.npad])
            self.mailbox.fill_(EXCHANGE_NEUTRAL)
        else:
            self.mailbox = torch.full((self.npad,), EXCHANGE_NEUTRAL, dtype=torch.int32)
        self.has[:] = False
        self._last = None
        if app == "components":
            self.val = np.arange(self.lo, self.hi, dtype=np.int64)
        else:
            self.val = np.full(self.len, 0xFFFFFFFF, np.int64)
        self.front = (np.empty(0, np.int64), np.empty(0, np.int64))

    def seed_source(self, lv):
        self.val[lv] = 0
        if self.deg[lv] > 0:
            self.front = (np.array([lv]), np.array([1]))

    def _own(self, idx):
        return (idx >= self.blo) & (idx < self.blo + self.block)

    def reset_mailbox(self):
        mb = self.mailbox.numpy()
        if self._last == "peer":  # pgx_reset_touched
            mb[self._foreign()] = EXCHANGE_NEUTRAL
        elif self._last == "dense":  # foreign blocks only: the owned block is neutral
            mb[:self.blo] = EXCHANGE_NEUTRAL
            mb[self.blo + self.block:] = EXCHANGE_NEUTRAL
        self.has[:] = False

    def exchanged(self, kind):
        self._last = kind

    def _foreign(self):
        idx = np.flatnonzero(self.has)
        return idx[~self._own(idx)]

    def compact_touched(self):
        idx = self._foreign()
        mb = self.mailbox.numpy()
        vals = mb[idx].astype(np.int64)
        mb[idx] = EXCHANGE_NEUTRAL
        pairs = torch.from_numpy((idx.astype(np.int64) << 32) | vals)
        owner = idx // self.block
        return pairs, np.bincount(owner, minlength=self.world).tolist()

    def scatter_pairs(self, pairs):
        p = pairs.numpy()
        np.minimum.at(self.mailbox.numpy(), (p >> 32).astype(np.int64),
                      (p & 0xFFFFFFFF).astype(np.int32))

    def scatter_min(self, dense, peer=False):
        if dense:
            lv = np.flatnonzero(self.deg > 0)
            msg = lv + self.lo
        else:
            lv, msg = self.front
        dst, m = self._edges_of(lv, msg)
        m = m.astype(np.int32)
        mb = self.mailbox.numpy()
        if not peer:
            np.minimum.at(mb, dst, m)
            self.has[dst] = True
            return
        # pgx_scatter_peer: own slots and every owner's slot under its lock,
        # the local copies of foreign slots (this rank's filter) unlocked
        foreign = ~self._own(dst)
        np.minimum.at(mb, dst[foreign], m[foreign])
        self._locked_min(self._me, dst[~foreign], m[~foreign])
        owner = dst[foreign] // self.block
        for o in np.unique(owner):
            sel = owner == o
            self._locked_min(int(o), dst[foreign][sel], m[foreign][sel])
        self.has[dst] = True

    def apply_min(self, app, count_only):
        blk = slice(self.blo, self.blo + self.len)
        sl = self.mailbox.numpy()[blk].astype(np.int64)
        has = sl != EXCHANGE_NEUTRAL
        rec = int(has.sum())
        if count_only:
            return torch.tensor([rec, 0, 0, 0], dtype=torch.int64)
        self.mailbox.numpy()[blk] = EXCHANGE_NEUTRAL
        imp = has & (sl < self.val)
        self.val[imp] = sl[imp]
        lv = np.flatnonzero(imp & (self.deg > 0))
        msg = sl[lv] + (1 if app == "sssp" else 0)
        self.front = (lv, msg)
        return torch.tensor([rec, int(imp.sum()), int(lv.size), int(self.deg[lv].sum())],
                            dtype=torch.int64)

    @staticmethod
    def decode_counts(row):
        return tuple(row)

    def set_frontier(self, senders, edges):
        pass  # the CPU stand-in keeps its frontier as arrays

    # ---- PageRank ----
    def init_pagerank(self, r0):
        self.app = "pagerank"
        self.mailbox = torch.zeros(self.npad, dtype=torch.float64)
        self.rank = np.full(self.len, r0)
        self.share = np.where(self.deg > 0, r0 / np.maximum(self.deg, 1), 0.0)
        return int((self.deg == 0).sum())

    def fold_sum(self):
        self.mailbox.zero_()
        lv = np.flatnonzero(self.deg > 0)
        dst, m = self._edges_of(lv, self.share[lv])
        np.add.at(self.mailbox.numpy(), dst, m)

    def apply_pagerank(self, base, damping, dangling, last):
        dn = float(dangling.reshape(-1)[0]) / self.n
        folded = self.mailbox.numpy()[self.blo:self.blo + self.len].copy()
        r = base + damping * (folded + dn)
        self.rank = r
        if not last:
            sp = self.deg > 0
            self.share = np.where(sp, r / np.maximum(self.deg, 1), 0.0)
        return torch.tensor([float(r[self.deg == 0].sum())], dtype=torch.float64)

    def values(self):
        if self.app == "pagerank":
            return torch.from_numpy(self.rank.copy())
        return torch.from_numpy(self.val.astype(np.int64))
