"""Multi-GPU superstep (placeholder until the partitioned path lands)."""

from __future__ import annotations

import os


def distributed_context():
    """Active torch.distributed world with >1 rank, else None."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    if dist.get_world_size() <= 1:
        return None
    return dist


def run_partitioned(graph, program, low, config, ctx):  # pragma: no cover
    raise NotImplementedError
