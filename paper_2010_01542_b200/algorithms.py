"""Built-in vertex programs with device lowerings (reference: algorithms.py).

Each factory validates its arguments exactly like the reference
(algorithms.py:37-40, 126-133) and returns a ``VertexProgram`` whose
``compute`` carries the lowering the engine dispatches on.  The semantics
the kernels reproduce:

* ``pagerank`` (algorithms.py:27-84): fp64; setup seeds r0/outdeg shares;
  rank = (1-d)/n + d*(folded + dangling/n); broadcast rank/outdeg except on
  the last superstep; dangling mass re-summed after every superstep;
  exactly ``iterations`` supersteps.  The reference's pull fold is
  realised as a push scatter with ``red.add.f64`` -- the same sum, a
  different addition order (<= 1e-9 relative, see tests).
* ``connected_components`` (algorithms.py:87-113): Hashmin; superstep 0
  broadcasts every id; later a vertex adopts a smaller label and
  rebroadcasts; push-form realisation of the pull program.
  Labels are returned as int64 like the reference state dtype.
* ``sssp`` (algorithms.py:116-152): push, min, uint32 hops,
  ``UNREACHED = 2**32 - 1``.

The compute callables are markers: calling one on the host raises, since
computes run inside the kernel.
"""

from __future__ import annotations

import numpy as np

from .engine import LOWERING_ATTR, CommMode, VertexProgram
from .errors import ConfigError
from .mailbox import min_combine, sum_combine

#: distance value of vertices no path reaches (algorithms.py:21)
UNREACHED = int(np.iinfo(np.uint32).max)

DEFAULT_DAMPING = 0.85
DEFAULT_ITERATIONS = 10


def _device_only(name):
    def compute(ctx):
        raise ConfigError(f"{name}: compute runs inside the B200 kernel only")
    return compute


def _marker(name):
    def fn(*args, **kwargs):
        raise ConfigError(f"{name}: runs inside the B200 kernel only")
    return fn


def _program(app, comm_mode, msg_dtype, state_dtype, combine, track_active,
             name, setup=None, hook=None, **params):
    compute = _device_only(name)
    parts = dict(setup=setup, on_superstep_end=hook, combine=combine,
                 comm_mode=comm_mode, track_active=track_active)
    setattr(compute, LOWERING_ATTR, dict(app=app, parts=parts, **params))
    return VertexProgram(compute=compute, comm_mode=comm_mode,
                         message_dtype=msg_dtype, state_dtype=state_dtype,
                         combine=combine, setup=setup, on_superstep_end=hook,
                         track_active=track_active, name=name)


def pagerank(iterations: int = DEFAULT_ITERATIONS,
             damping: float = DEFAULT_DAMPING) -> VertexProgram:
    """Power-iteration PageRank over a fixed superstep budget."""
    if iterations < 1:
        raise ConfigError(f"iterations must be >= 1, got {iterations}")
    if not 0.0 <= damping <= 1.0:
        raise ConfigError(f"damping must be in [0, 1], got {damping}")
    return _program("pagerank", CommMode.PULL, np.float64, np.float64,
                    sum_combine(np.float64), False, "pagerank",
                    setup=_marker("pagerank.setup"),
                    hook=_marker("pagerank.on_superstep_end"),
                    iterations=int(iterations), damping=float(damping))


def connected_components() -> VertexProgram:
    """Label propagation toward the minimum vertex id of each component."""
    return _program("components", CommMode.PULL, np.int64, np.int64,
                    min_combine(np.int64), True, "components",
                    setup=_marker("components.setup"))


def sssp(source: int) -> VertexProgram:
    """Unweighted single-source shortest paths (hop counts)."""
    if source < 0:
        raise ConfigError(f"source must be a vertex id >= 0, got {source}")
    return _program("sssp", CommMode.PUSH, np.uint32, np.uint32,
                    min_combine(np.uint32), True, "sssp",
                    setup=_marker("sssp.setup"), source=int(source))
