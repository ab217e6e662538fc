"""R-MAT inputs built on the GPU (input construction only).

The reference ships no R-MAT (generate.py); BASELINE.json's configs need
one.  Draws come from ``pgx_rmat_keys`` (counter-based SplitMix64, the
same text as oracle/pregel_oracle.c), then ``torch.sort`` +
``unique_consecutive`` dedup and a ``bincount`` row pointer -- CSR rows
sorted ascending exactly like graph.py:185.  BASELINE.md section 3's
SHA-256 values pin the output (tests/test_gpu.py).
"""

from __future__ import annotations

import torch

from . import _lib
from .graph import Graph

#: BASELINE.json configs: (scale, edge_factor, a, b, c, seed, symmetric)
CONFIGS = {
    "C1": (16, 16, 0.57, 0.19, 0.19, 1, False),
    "C2": (22, 8, 0.57, 0.19, 0.19, 2, True),
    "C3": (22, 16, 0.57, 0.19, 0.19, 3, False),
    "C4": (22, 28, 0.45, 0.22, 0.22, 4, False),
    "C5": (26, 14, 0.57, 0.19, 0.19, 5, True),
    # test-only: C5's shape (symmetrised, a/b/c, edge factor, seed) at scale 16
    "C5S": (16, 14, 0.57, 0.19, 0.19, 5, True),
}


def rmat_keys(scale, edge_factor, a, b, c, seed, symmetric, device=None,
              src_lo: int = 0, src_hi: int | None = None) -> torch.Tensor:
    """Sorted, deduplicated ``src << 32 | dst`` keys (int64) on the device."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    n = 1 << scale
    src_hi = n if src_hi is None else src_hi
    draws = edge_factor * n
    cap = draws * (2 if symmetric else 1)
    lib = _lib.load()
    with torch.cuda.device(dev):
        keys = torch.empty(cap, dtype=torch.int64, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(lib.pgx_rmat_keys(scale, 0, draws, a, b, c, seed, int(symmetric),
                                     src_lo, src_hi, keys.data_ptr(), cap,
                                     count.data_ptr(), st), "pgx_rmat_keys")
        kept = int(count.item())
        keys = keys[:kept]
        keys, _ = torch.sort(keys)
        keys = torch.unique_consecutive(keys)
    return keys


def rmat_graph(name_or_spec, device=None) -> Graph:
    """Build the R-MAT graph of a BASELINE config ("C1".."C5") on a GPU."""
    spec = CONFIGS[name_or_spec] if isinstance(name_or_spec, str) else name_or_spec
    scale = spec[0]
    keys = rmat_keys(*spec, device=device)
    n = 1 << scale
    src = keys >> 32
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=keys.device)
    offsets[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    del src
    targets = (keys & 0xFFFFFFFF).to(torch.int32)
    del keys
    return Graph(n, offsets, targets)
