"""Thread-based stand-in for torch.distributed -- TEST INFRASTRUCTURE ONLY.

Runs W "ranks" as threads of one process so the partitioned driver and the
CUDA phase kernels (pgx_scatter / pgx_apply_slice / pgx_pr_apply_slice)
can be exercised on ONE GPU.  Collectives are implemented with a barrier
and torch ops on the participants' tensors; no kernel waits on another
rank, so nothing spins on the device.
"""

from __future__ import annotations

import threading

import torch
import torch.distributed as _d


class ThreadDist:
    ReduceOp = _d.ReduceOp

    def __init__(self, world: int):
        self.world = world
        self.calls = {}  # collective name -> calls (rank 0), for the tests
        self._bar = threading.Barrier(world)
        self._slots = [None] * world
        self._tls = threading.local()

    def bind(self, rank: int):
        self._tls.rank = rank

    def get_rank(self):
        return self._tls.rank

    def get_world_size(self):
        return self.world

    def _combine(self, op):
        ts = self._slots
        out = ts[0].clone()
        for t in ts[1:]:
            if op == _d.ReduceOp.MIN:
                out = torch.minimum(out, t)
            elif op == _d.ReduceOp.MAX:
                out = torch.maximum(out, t)
            else:
                out = out + t
        return out

    def reduce(self, tensor, dst, op=_d.ReduceOp.SUM):
        r = self.get_rank()
        torch.cuda.synchronize() if tensor.is_cuda else None
        self._slots[r] = tensor
        self._bar.wait()
        if r == dst:
            res = self._combine(op)
        self._bar.wait()
        if r == dst:
            tensor.copy_(res)
            torch.cuda.synchronize() if tensor.is_cuda else None
        self._bar.wait()

    def all_reduce(self, tensor, op=_d.ReduceOp.SUM):
        r = self.get_rank()
        torch.cuda.synchronize() if tensor.is_cuda else None
        self._slots[r] = tensor
        self._bar.wait()
        res = self._combine(op)
        self._bar.wait()
        tensor.copy_(res)
        torch.cuda.synchronize() if tensor.is_cuda else None
        self._bar.wait()

    def get_backend(self):
        """The production branch of the driver (CUDA tensors, no host
        staging): the collectives below take device tensors like NCCL's."""
        return "nccl"

    def _count(self, name):
        if self.get_rank() == 0:
            self.calls[name] = self.calls.get(name, 0) + 1

    def reduce_scatter_tensor(self, out, inp, op=_d.ReduceOp.SUM):
        """Equal blocks; `out` may alias this rank's block of `inp` (the
        driver's in-place call): every rank reduces its block from every
        input before anyone writes."""
        self._count("reduce_scatter_tensor")
        r = self.get_rank()
        torch.cuda.synchronize() if inp.is_cuda else None
        blk = out.numel()
        assert inp.numel() == blk * self.world, "reduce_scatter_tensor: unequal blocks"
        self._slots[r] = inp
        self._bar.wait()
        parts = [t[r * blk:(r + 1) * blk] for t in self._slots]
        res = parts[0].clone()
        for t in parts[1:]:
            if op == _d.ReduceOp.MIN:
                res = torch.minimum(res, t)
            elif op == _d.ReduceOp.MAX:
                res = torch.maximum(res, t)
            else:
                res = res + t
        torch.cuda.synchronize() if inp.is_cuda else None
        self._bar.wait()
        out.copy_(res)
        torch.cuda.synchronize() if out.is_cuda else None
        self._bar.wait()

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None):
        self._count("all_to_all_single")
        r = self.get_rank()
        torch.cuda.synchronize() if inp.is_cuda else None
        w = self.world
        ins = in_splits if in_splits is not None else [inp.numel() // w] * w
        self._slots[r] = (inp, list(ins))
        self._bar.wait()
        chunks = []
        for src in range(w):
            t, sp = self._slots[src]
            off = sum(sp[:r])
            chunks.append(t[off:off + sp[r]])
        self._bar.wait()
        if chunks:
            out.copy_(torch.cat(chunks))
        torch.cuda.synchronize() if out.is_cuda else None
        self._bar.wait()

    def all_gather(self, parts, tensor):
        r = self.get_rank()
        torch.cuda.synchronize() if tensor.is_cuda else None
        self._slots[r] = tensor
        self._bar.wait()
        for i in range(self.world):
            parts[i].copy_(self._slots[i])
        self._bar.wait()


    def all_gather_object(self, out, obj):
        r = self.get_rank()
        self._slots[r] = obj
        self._bar.wait()
        for i in range(self.world):
            out[i] = self._slots[i]
        self._bar.wait()

    def barrier(self):
        self._bar.wait()


def run_ranks(world, fn, d=None):
    """Run fn(rank, dist) on `world` threads; returns the per-rank results."""
    d = ThreadDist(world) if d is None else d
    out = [None] * world
    err = []

    def body(r):
        d.bind(r)
        try:
            out[r] = fn(r, d)
        except BaseException as e:  # pragma: no cover
            err.append(e)
            d._bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out
