"""Superstep executor host side (reference: engine.py).

``run(graph, program, config)`` keeps the reference signature and return
type (engine.py:201-204, 94-108).  The reference body -- ``_Executor.run``
with W worker threads, two barriers per superstep and per-vertex Python
callbacks (engine.py:255-474) -- is replaced by ONE call into libpgx.so:
a persistent cooperative kernel that runs every superstep (scatter with
the hybrid combiner, apply, frontier build, halt test) on the B200 and
writes per-superstep statistics to device memory.  The host reads the
statistics back once, after the run.

Only the three built-in programs have a device lowering (their factories
tag the compute callable).  A program whose compute has no lowering, or
whose setup / hook / combine were swapped for other callables, raises
``ConfigError``: there is no CPU fallback.  ``extract`` overrides are
honoured (applied to the final state on the host, engine.py:310-311).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from enum import Enum
from types import SimpleNamespace
from typing import Any, Callable

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, ExecutionError
from .graph import Graph
from .layout import LayoutMode
from .mailbox import CombineFn, CombinerKind
from .scheduler import SchedulerMode

DEFAULT_MAX_SUPERSTEPS = 10_000


class CommMode(Enum):
    PUSH = "push"
    PULL = "pull"


@dataclass(frozen=True)
class VertexProgram:
    """engine.py:59-81.  ``compute`` must carry a device lowering."""

    compute: Callable[["VertexContext"], None]
    comm_mode: CommMode
    message_dtype: Any
    state_dtype: Any
    combine: CombineFn | None = None
    setup: Callable | None = None
    on_superstep_end: Callable | None = None
    extract: Callable | None = None
    track_active: bool = True
    name: str = ""


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:84-91.  ``workers``/``scheduler``/``layout``/``combiner``/
    ``validate_phases`` are validated and inert on the device; ``device``
    selects the CUDA device (default: the current one)."""

    workers: int = 1
    scheduler: SchedulerMode = field(default_factory=SchedulerMode.static)
    layout: LayoutMode = LayoutMode.INTERLEAVED
    combiner: CombinerKind = CombinerKind.HYBRID
    max_supersteps: int = DEFAULT_MAX_SUPERSTEPS
    validate_phases: bool = False
    device: int | None = None
    #: PageRank lowering: "pull" (the reference's comm mode, algorithms.py:80;
    #: in-neighbour fold, no atomics) or "push" (scatter with red.add.f64)
    pagerank_mode: str = "pull"
    #: pull PageRank: the highest out-degree sources' shares kept in each
    #: CTA's shared memory (pgx_pagerank_pull_hubs_run; bit-identical
    #: results; the in-CSR's hub edges are encoded once per graph): "auto"
    #: for graphs that live on the GPU with >= 2^24 edges (C4 5.76 -> 5.29
    #: ms; on C1 the table's staging costs more than it saves: 0.133 ->
    #: 0.154 ms), "on" always, "off" never
    pagerank_hubs: str = "auto"
    #: shared-memory combiner for hub recipients (CC / SSSP, ablation arm;
    #: measured slower on B200): "auto" builds
    #: the hub encoding from the second run on a device CSR (amortised graph
    #: preprocessing), "on" always, "off" never
    hub_cache: str = "off"
    #: destination-segmented index for the dense supersteps of CC / SSSP
    #: (shared-memory combine of every message, pgx_seg.cuh): "auto" builds
    #: it for graphs that live on the GPU (graph preprocessing amortised
    #: over runs; host graphs uploaded for one run use K1 throughout),
    #: "on" always, "off" never.  Results and statistics are identical.
    segments: str = "auto"
    #: unit-weight SSSP direction-optimising supersteps (pgx_pull.cuh): a
    #: superstep whose senders hold >= m/8 edges runs bottom-up over the
    #: in-CSR.  "auto" builds the transpose for graphs that live on the GPU
    #: (graph preprocessing, amortised like the segmented index), "on"
    #: always, "off" never (push only).  Results and statistics are identical.
    direction: str = "auto"
    #: connected components of a graph in host memory: superstep 0 (every
    #: vertex sends its id) is combined chunk by chunk while the targets
    #: upload (pgx_cc_source_scatter), the run starts at its apply.  "auto"
    #: on, "off" uploads first.  Results and statistics are identical.
    overlap_upload: str = "auto"


@dataclass(frozen=True)
class SuperstepStats:
    """engine.py:94-99 plus the device counters behind GTEPS / bytes."""

    index: int
    active_count: int
    messages_sent: int
    seconds: float
    edges: int = 0          # edges traversed by this superstep's senders
    senders: int = 0        # senders with out-degree > 0 (#F_s)
    recipients: int = 0     # distinct recipients of its messages (R_s)
    broadcasters: int = 0   # vertices that sent (out-degree 0 included)


@dataclass(frozen=True)
class RunReport:
    """engine.py:102-108 plus the device view of the result."""

    values: np.ndarray
    superstep_count: int
    supersteps: list
    wall_seconds: float
    hit_superstep_cap: bool
    device_values: Any = None      # torch tensor on the device (u32 / f64)
    device_seconds: float = 0.0    # kernel time from the device timer
    ctas: int = 0                  # persistent CTAs of the run kernel
    exchanges: Any = None          # partitioned runs: mailbox exchange per superstep


class VertexContext:
    """Present for API compatibility (engine.py:115-194).  Device programs
    never see a Python context: computes run inside the kernel."""

    def __init__(self, *args, **kwargs):
        raise ConfigError("VertexContext exists only inside device kernels; "
                          "use pagerank / connected_components / sssp")


# ----------------------------------------------------------------------
# lowering
# ----------------------------------------------------------------------

LOWERING_ATTR = "_pgx_lowering"


def lowering_of(program: VertexProgram) -> dict:
    """Return the device lowering of ``program`` or raise ConfigError."""
    low = getattr(program.compute, LOWERING_ATTR, None)
    if low is None:
        raise ConfigError(
            f"program {program.name or program.compute!r} has no device lowering: "
            f"the B200 engine runs pagerank / connected_components / sssp "
            f"(there is no CPU fallback for Python compute callbacks)")
    for attr in ("setup", "on_superstep_end", "combine"):
        if getattr(program, attr) is not low["parts"][attr]:
            raise ConfigError(
                f"{low['app']}: a replaced `{attr}` cannot be lowered to the device")
    if program.comm_mode is not low["parts"]["comm_mode"] or \
            program.track_active != low["parts"]["track_active"]:
        raise ConfigError(f"{low['app']}: comm_mode/track_active were changed")
    return low


def _validate(program: VertexProgram, config: EngineConfig) -> None:
    """engine.py:477-490."""
    if config.workers < 1:
        raise ConfigError(f"worker count must be >= 1, got {config.workers}")
    if config.max_supersteps < 1:
        raise ConfigError(f"superstep cap must be >= 1, got {config.max_supersteps}")
    if config.max_supersteps > 2 ** 31 - 2:
        raise ConfigError("superstep cap must fit in int32")
    if not isinstance(config.scheduler, SchedulerMode):
        raise ConfigError(f"bad scheduler mode: {config.scheduler!r}")
    if not isinstance(config.layout, LayoutMode):
        raise ConfigError(f"bad layout mode: {config.layout!r}")
    if not isinstance(config.combiner, CombinerKind):
        raise ConfigError(f"bad combiner kind: {config.combiner!r}")
    if config.pagerank_mode not in ("pull", "push"):
        raise ConfigError(f"bad pagerank_mode: {config.pagerank_mode!r}")
    if config.pagerank_hubs not in ("auto", "on", "off"):
        raise ConfigError(f"bad pagerank_hubs: {config.pagerank_hubs!r}")
    if config.hub_cache not in ("auto", "on", "off"):
        raise ConfigError(f"bad hub_cache: {config.hub_cache!r}")
    if config.segments not in ("auto", "on", "off"):
        raise ConfigError(f"bad segments: {config.segments!r}")
    if config.overlap_upload not in ("auto", "off"):
        raise ConfigError(f"bad overlap_upload: {config.overlap_upload!r}")
    if config.direction not in ("auto", "on", "off"):
        raise ConfigError(f"bad direction: {config.direction!r}")
    if program.comm_mode is CommMode.PUSH and program.combine is None:
        raise ConfigError("push-mode programs must declare a combine function")
    if config.combiner is CombinerKind.CAS and program.comm_mode is CommMode.PUSH \
            and (program.combine is None or program.combine.neutral is None):
        raise ConfigError("the CAS combiner strategy needs a combine function "
                          "with a neutral element to pre-fill slots with")


# ----------------------------------------------------------------------
# run
# ----------------------------------------------------------------------

def run(graph: Graph, program: VertexProgram,
        config: EngineConfig | None = None) -> RunReport:
    """Execute ``program`` on ``graph`` until quiescence or the cap."""
    config = config or EngineConfig()
    _validate(program, config)
    low = lowering_of(program)
    app = low["app"]
    n = graph.vertex_count
    if app == "sssp" and not 0 <= low["source"] < n:
        raise ConfigError(f"source vertex {low['source']} out of range [0, {n})")
    if n == 0:
        return _empty_run(program, low)
    if not torch.cuda.is_available():
        raise ExecutionError("no CUDA device: the B200 engine has no CPU fallback")
    from .distributed import distributed_context  # multi-GPU under torchrun
    ctx = distributed_context()
    if ctx is not None:
        from .distributed import run_partitioned
        return run_partitioned(graph, program, low, config, ctx)
    return _run_device(graph, program, low, config)


def _empty_run(program, low) -> RunReport:
    """An empty graph runs one empty superstep (engine.py:271-296)."""
    dtype = {"pagerank": np.float64, "components": np.int64,
             "sssp": np.uint32}[low["app"]]
    values = np.empty(0, dtype=dtype)
    stats = [SuperstepStats(0, 0, 0, 0.0)]
    if program.extract is not None:
        values = program.extract(SimpleNamespace(state=values,
                                                 halted=np.ones(0, bool)))
    return RunReport(values, 1, stats, 0.0, False)


@dataclass
class LaunchPlan:
    """Everything one device run needs, allocated up front (re-usable)."""

    app: str
    csr: Any
    values: torch.Tensor
    stats: torch.Tensor
    ws: torch.Tensor
    ws_bytes: int
    max_steps: int
    low: dict
    stream: Any
    pull: bool = False
    hubs: bool = False
    seg: Any = None          # _lib.PgxSegIndex when the segmented scatter is on
    bottom_up: bool = False  # SSSP: direction-optimising (in-CSR bottom-up supersteps)
    prescattered: bool = False  # CC: superstep 0 combined during the upload (first launch)

    def _hub_args(self):
        c = self.csr
        if self.hubs:
            return c.hub_col.data_ptr(), c.hub_ids.data_ptr(), int(c.hub_ids.numel())
        return c.col_idx.data_ptr(), None, 0

    def launch(self) -> None:
        """Enqueue the persistent run kernel (asynchronous)."""
        lib = _lib.load()
        c = self.csr
        sp = self.stream.cuda_stream
        if self.app == "pagerank" and self.pull:
            it, d = self.low["iterations"], self.low["damping"]
            base = (1.0 - d) / c.n      # algorithms.py:49 (host float math)
            r0 = 1.0 / c.n              # algorithms.py:50
            if self.hubs and c.pr_nhubs > 0:
                rc = lib.pgx_pagerank_pull_hubs_run(
                    c.n, c.m, c.row_ptr.data_ptr(), c.in_row_ptr.data_ptr(),
                    c.pr_hub_col.data_ptr(), c.in_ws.data_ptr(), c.pr_hub_slot.data_ptr(),
                    c.pr_nhubs, it, d, base, r0, self.max_steps, self.values.data_ptr(),
                    self.ws.data_ptr(), self.ws_bytes, self.stats.data_ptr(), sp)
                _lib.check(rc, "pgx_pagerank_pull_hubs_run")
            else:
                rc = lib.pgx_pagerank_pull_run(c.n, c.m, c.row_ptr.data_ptr(),
                                               c.in_row_ptr.data_ptr(), c.in_col.data_ptr(),
                                               c.in_ws.data_ptr(), it, d, base, r0,
                                               self.max_steps, self.values.data_ptr(),
                                               self.ws.data_ptr(), self.ws_bytes,
                                               self.stats.data_ptr(), sp)
                _lib.check(rc, "pgx_pagerank_pull_run")
        elif self.app == "pagerank":
            it, d = self.low["iterations"], self.low["damping"]
            base = (1.0 - d) / c.n      # algorithms.py:49 (host float math)
            r0 = 1.0 / c.n              # algorithms.py:50
            rc = lib.pgx_pagerank_run(c.n, c.m, c.row_ptr.data_ptr(),
                                      c.col_idx.data_ptr(), c.ws.data_ptr(),
                                      it, d, base, r0, self.max_steps,
                                      self.values.data_ptr(), self.ws.data_ptr(),
                                      self.ws_bytes, self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_pagerank_run")
        elif self.app == "sssp" and self.bottom_up:
            rc = lib.pgx_sssp_run_dir(c.n, c.m, c.row_ptr.data_ptr(), c.col_idx.data_ptr(),
                                      c.ws.data_ptr(),
                                      ctypes.byref(self.seg) if self.seg is not None else None,
                                      c.in_row_ptr.data_ptr(), c.in_col.data_ptr(),
                                      self.low["source"], self.max_steps,
                                      self.values.data_ptr(), self.ws.data_ptr(),
                                      self.ws_bytes, self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_sssp_run_dir")
        elif self.app == "components" and self.prescattered:
            # the first launch after the upload pipeline (plan_run); a later
            # launch of the same plan runs superstep 0 itself
            self.prescattered = False
            rc = lib.pgx_cc_run_prescattered(c.n, c.m, c.row_ptr.data_ptr(),
                                             c.col_idx.data_ptr(), c.ws.data_ptr(),
                                             self.max_steps, self.values.data_ptr(),
                                             self.ws.data_ptr(), self.ws_bytes,
                                             self.stats.data_ptr(), sp)
            if rc == _lib.PGX_EINVAL:  # ablation options set: the plain run
                self.launch()
                return
            _lib.check(rc, "pgx_cc_run_prescattered")
        elif self.app == "components" and self.seg is not None:
            rc = lib.pgx_cc_run_ex(c.n, c.m, c.row_ptr.data_ptr(), c.col_idx.data_ptr(),
                                   c.ws.data_ptr(), ctypes.byref(self.seg), self.max_steps,
                                   self.values.data_ptr(), self.ws.data_ptr(), self.ws_bytes,
                                   self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_cc_run_ex")
        elif self.app == "sssp" and self.seg is not None:
            rc = lib.pgx_sssp_run_ex(c.n, c.m, c.row_ptr.data_ptr(), c.col_idx.data_ptr(),
                                     c.ws.data_ptr(), ctypes.byref(self.seg), self.low["source"],
                                     self.max_steps, self.values.data_ptr(), self.ws.data_ptr(),
                                     self.ws_bytes, self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_sssp_run_ex")
        elif self.app == "components":
            col, hub_ids, nh = self._hub_args()
            rc = lib.pgx_cc_run(c.n, c.m, c.row_ptr.data_ptr(), col, c.ws.data_ptr(),
                                hub_ids, nh, self.max_steps,
                                self.values.data_ptr(), self.ws.data_ptr(),
                                self.ws_bytes, self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_cc_run")
        else:
            col, hub_ids, nh = self._hub_args()
            rc = lib.pgx_sssp_run(c.n, c.m, c.row_ptr.data_ptr(), col, c.ws.data_ptr(),
                                  hub_ids, nh, self.low["source"], self.max_steps,
                                  self.values.data_ptr(), self.ws.data_ptr(),
                                  self.ws_bytes, self.stats.data_ptr(), sp)
            _lib.check(rc, "pgx_sssp_run")


_APP_ID = {"pagerank": _lib.PGX_APP_PAGERANK, "components": _lib.PGX_APP_CC,
           "sssp": _lib.PGX_APP_SSSP}


def plan_run(graph: Graph, program: VertexProgram,
             config: EngineConfig | None = None, device=None) -> LaunchPlan:
    """Upload/prepare the graph and allocate a run's buffers (no launch)."""
    config = config or EngineConfig()
    _validate(program, config)
    low = lowering_of(program)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None
                       and config.device is None else
                       (device if device is not None else config.device))
    stream = torch.cuda.current_stream(dev)
    app = low["app"]
    # CC from host memory: superstep 0 under the upload (_upload_overlapped)
    overlap = (app == "components" and config.overlap_upload == "auto"
               and graph.device.type != "cuda" and graph.out_targets.dtype == torch.int32
               and graph.edge_count > 0 and config.hub_cache == "off"
               and config.segments != "on" and graph._device.get(dev.index) is None)
    csr = graph.device_csr(dev, stream, defer_targets=overlap)
    n, m = csr.n, csr.m
    lib = _lib.load()
    max_steps = int(config.max_supersteps)
    pull = app == "pagerank" and config.pagerank_mode == "pull"
    if app == "pagerank":
        max_steps = min(max_steps, int(low["iterations"]))
    else:
        # CC / SSSP quiesce within n + 1 supersteps, so a larger cap is never
        # reached: size the per-superstep buffers for n + 2 at most
        max_steps = min(max_steps, n + 2)
    if pull:
        csr.ensure_transpose(stream)
    hubs = app != "pagerank" and (config.hub_cache == "on" or
                                  (config.hub_cache == "auto" and csr.runs >= 1))
    if hubs:
        csr.ensure_hubs(stream)
    # "auto": graphs that live on the GPU (the encoding is graph preparation
    # amortised over runs, like the segmented index) with >= 2^24 edges
    if pull and csr.m > 0 and (config.pagerank_hubs == "on" or
                               (config.pagerank_hubs == "auto" and csr.m >= 1 << 24
                                and graph.device.type == "cuda")):
        csr.ensure_pr_hubs(stream)
        hubs = True
    seg = None
    # "auto": CC on device-resident graphs (the index is graph preparation,
    # amortised over runs; a host graph uploaded for one run keeps K1
    # throughout).  Unit-weight SSSP keeps K1 with its has-bitmap filter,
    # which hits L1 (C3 0.421 vs 0.448 ms segmented)
    if app != "pagerank" and not hubs and csr.m > 0 and (
            config.segments == "on" or
            (config.segments == "auto" and app == "components"
             and graph.device.type == "cuda")):
        csr.ensure_segments(stream)
        seg = csr.seg
    # direction-optimising SSSP (bottom-up supersteps need the in-CSR; the
    # hub-cache ablation arm runs push only)
    bottom_up = app == "sssp" and not hubs and csr.m > 0 and (
        config.direction == "on" or
        (config.direction == "auto" and graph.device.type == "cuda"))
    if bottom_up:
        csr.ensure_transpose(stream)
    csr.runs += 1
    app_id = _lib.PGX_APP_PAGERANK_PULL if pull else _APP_ID[app]
    ws_bytes = _lib.out_size(lib.pgx_run_workspace_bytes, app_id, n, m, max_steps)
    with torch.cuda.device(dev):
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        stats = torch.zeros(_lib.PGX_STAT_HDR + _lib.PGX_STAT_FIELDS * max_steps,
                            dtype=torch.int64, device=dev)
        vdt = torch.float64 if app == "pagerank" else torch.int32
        values = torch.empty(n, dtype=vdt, device=dev)
    if overlap:
        _upload_overlapped(graph, csr, ws, ws_bytes, max_steps, stream, lib)
    return LaunchPlan(app, csr, values, stats, ws, ws_bytes, max_steps, low, stream, pull, hubs,
                      seg, bottom_up, overlap)


#: edges per chunk of the CC upload pipeline (256 MB of targets)
_OVERLAP_CHUNK = 1 << 26


def _upload_overlapped(graph, csr, ws, ws_bytes, max_steps, stream, lib) -> None:
    """Copy the targets of a host graph in chunks on a copy stream and
    combine each landed chunk's superstep-0 messages (source ids) into the
    run's mailbox on ``stream`` (pgx_cc_source_scatter): the PCIe copy,
    the longest part of a run from host memory, hides superstep 0.  The
    offsets and the tile map are on the device already (device_csr)."""
    host = graph.out_targets
    n, m = csr.n, csr.m
    dev = csr.col_idx.device
    sp = stream.cuda_stream
    _lib.check(lib.pgx_cc_prescatter_init(n, m, max_steps, ws.data_ptr(), ws_bytes, sp),
               "pgx_cc_prescatter_init")
    copy = torch.cuda.Stream(device=dev)
    ready = torch.cuda.Event()
    ready.record(stream)            # offsets, tile map, cleared mailbox first
    copy.wait_event(ready)
    for lo in range(0, m, _OVERLAP_CHUNK):
        hi = min(m, lo + _OVERLAP_CHUNK)
        with torch.cuda.stream(copy):
            csr.col_idx[lo:hi].copy_(host[lo:hi], non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(copy)
        stream.wait_event(landed)
        _lib.check(lib.pgx_cc_source_scatter(n, m, csr.row_ptr.data_ptr(),
                                             csr.col_idx.data_ptr(), csr.ws.data_ptr(), lo, hi,
                                             max_steps, ws.data_ptr(), ws_bytes, sp),
                   "pgx_cc_source_scatter")
    csr.col_idx.record_stream(copy)
    csr.h2d_bytes += m * host.element_size()


def collect(plan: LaunchPlan, program: VertexProgram, wall: float | None = None) -> RunReport:
    """Read the device statistics and values back into a RunReport."""
    hdr = plan.stats[:_lib.PGX_STAT_HDR].cpu().tolist()
    k, hit_cap, ctas, t0 = int(hdr[0]), bool(hdr[1]), int(hdr[2]), int(hdr[3])
    if k < 1:
        raise ExecutionError("device run did not report a superstep count")
    rows = plan.stats[_lib.PGX_STAT_HDR:_lib.PGX_STAT_HDR + k * _lib.PGX_STAT_FIELDS]
    rows = rows.view(k, _lib.PGX_STAT_FIELDS).cpu().numpy()
    steps = []
    prev = t0
    for s in range(k):
        a, sent, e, f, r, t, bc = (int(x) for x in rows[s, :7])
        steps.append(SuperstepStats(s, a, sent, max(t - prev, 0) * 1e-9, e, f, r, bc))
        prev = t
    dev_seconds = max(int(rows[k - 1, 5]) - t0, 0) * 1e-9
    app = plan.app
    dv = plan.values
    if app == "components":
        dv = dv.to(torch.int64)                          # algorithms.py:111 int64
    # read back through page-locked memory (torch's caching host allocator):
    # a pageable .cpu() of a C2-sized result costs ~20x more
    host = torch.empty(dv.shape, dtype=dv.dtype, pin_memory=True)
    host.copy_(dv, non_blocking=True)
    plan.stream.synchronize()
    values = host.numpy()
    if app == "sssp":
        values = values.view(np.uint32)                  # algorithms.py:150 uint32
    if program.extract is not None:
        values = program.extract(SimpleNamespace(state=values,
                                                 halted=np.ones(values.shape[0], bool)))
    return RunReport(values, k, steps, dev_seconds if wall is None else wall, hit_cap,
                     device_values=dv, device_seconds=dev_seconds, ctas=ctas)


def _run_device(graph, program, low, config) -> RunReport:
    plan = plan_run(graph, program, config)
    t = time.perf_counter()
    plan.launch()
    plan.stream.synchronize()
    wall = time.perf_counter() - t
    return collect(plan, program, wall)
