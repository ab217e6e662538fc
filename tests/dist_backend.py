"""CPU stand-in for CudaBackend -- TEST INFRASTRUCTURE ONLY.

Mirrors the semantics of libpgx's phase kernels (pgx_scatter,
pgx_apply_slice, pgx_pr_apply_slice) with numpy on CPU torch tensors, so
that the partitioned driver (paper_2010_01542_b200.distributed.
PartitionedRun: partitioning, per-owner reductions, counter all-reduce,
halt test, value gather) runs over a gloo process group without a GPU.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2010_01542_b200.distributed import EXCHANGE_NEUTRAL, StepCounts


class CpuBackend:
    def __init__(self, off, tgt, lo, hi):
        self.device = torch.device("cpu")
        off = np.asarray(off, np.int64)
        self.n = off.size - 1
        self.glob_deg = np.diff(off)
        self.lo, self.hi, self.len = lo, hi, hi - lo
        base = off[lo]
        self.row_ptr = off[lo:hi + 1] - base
        self.col = np.asarray(tgt[base:off[hi]], np.int64)
        self.deg = np.diff(self.row_ptr)
        self.front = (np.empty(0, np.int64), np.empty(0, np.int64))  # (local ids, msgs)
        self.has = np.zeros(self.n, bool)
        self._full_reset = True

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
    def init_min(self, app, lo, hi):
        self.app = app
        self.mailbox = torch.full((self.n,), EXCHANGE_NEUTRAL, dtype=torch.int32)
        if app == "components":
            self.val = np.arange(lo, hi, dtype=np.int64)
        else:
            self.val = np.full(self.len, 0xFFFFFFFF, np.int64)
        self.front = (np.empty(0, np.int64), np.empty(0, np.int64))

    def seed_source(self, lv):
        self.val[lv] = 0
        if self.deg[lv] > 0:
            self.front = (np.array([lv]), np.array([1]))

    def reset_mailbox(self):
        if self.app == "pagerank":
            self.mailbox.zero_()
            return
        if self._full_reset:
            self.mailbox.fill_(EXCHANGE_NEUTRAL)
        self.has[:] = False
        self._full_reset = False

    def dense_exchanged(self):
        self._full_reset = True

    def _foreign(self):
        idx = np.flatnonzero(self.has)
        return idx[(idx < self.lo) | (idx >= self.hi)]

    def touched_count(self):
        return int(self._foreign().size)

    def compact_touched(self, bounds):
        idx = self._foreign()
        mb = self.mailbox.numpy()
        vals = mb[idx].astype(np.int64)
        mb[idx] = EXCHANGE_NEUTRAL
        pairs = torch.from_numpy((idx.astype(np.int64) << 32) | vals)
        owner = np.searchsorted(np.asarray(bounds[1:-1]), idx, side="right")
        return pairs, np.bincount(owner, minlength=len(bounds) - 1).tolist()

    def scatter_pairs(self, pairs):
        p = pairs.numpy()
        np.minimum.at(self.mailbox.numpy(), (p >> 32).astype(np.int64),
                      (p & 0xFFFFFFFF).astype(np.int32))

    def scatter_min(self, dense, id_offset):
        if dense:
            lv = np.flatnonzero(self.deg > 0)
            msg = lv + id_offset
        else:
            lv, msg = self.front
        dst, m = self._edges_of(lv, msg)
        mb = self.mailbox.numpy()
        np.minimum.at(mb, dst, m.astype(np.int32))
        self.has[dst] = True

    def apply_min(self, app, count_only):
        sl = self.mailbox.numpy()[self.lo:self.hi].astype(np.int64)
        has = sl != EXCHANGE_NEUTRAL
        rec = int(has.sum())
        if count_only:
            return StepCounts(rec, 0, 0, 0)
        self.mailbox.numpy()[self.lo:self.hi] = EXCHANGE_NEUTRAL
        imp = has & (sl < self.val)
        self.val[imp] = sl[imp]
        lv = np.flatnonzero(imp & (self.deg > 0))
        msg = sl[lv] + (1 if app == "sssp" else 0)
        self.front = (lv, msg)
        return StepCounts(rec, int(imp.sum()), int(lv.size), int(self.deg[lv].sum()))

    # ---- PageRank ----
    def init_pagerank(self, lo, hi, r0):
        self.app = "pagerank"
        self.mailbox = torch.zeros(self.n, dtype=torch.float64)
        self.rank = np.full(self.len, r0)
        self.share = np.where(self.deg > 0, r0 / np.maximum(self.deg, 1), 0.0)
        return int((self.deg == 0).sum())

    def scatter_sum(self):
        lv = np.flatnonzero(self.deg > 0)
        dst, m = self._edges_of(lv, self.share[lv])
        np.add.at(self.mailbox.numpy(), dst, m)

    def apply_pagerank(self, base, damping, dn, last):
        folded = self.mailbox.numpy()[self.lo:self.hi].copy()
        r = base + damping * (folded + dn)
        self.rank = r
        if not last:
            sp = self.deg > 0
            self.share = np.where(sp, r / np.maximum(self.deg, 1), 0.0)
        return float(r[self.deg == 0].sum())

    def values(self):
        if self.app == "pagerank":
            return torch.from_numpy(self.rank.copy())
        return torch.from_numpy(self.val.astype(np.int64))
