"""CSR graph container with PyTorch tensors (reference: graph.py).

Same contract as the reference ``Graph`` (graph.py:39-106): a directed
multigraph in CSR form with each row's targets sorted ascending, duplicate
edges and self-loops kept verbatim, ``undirected=True`` storing every input
edge in both directions (graph.py:141-187).  Differences are placement
only:

* arrays are ``torch`` tensors (CPU or CUDA); offsets int64 like the
  reference (graph.py:28), targets of the id dtype (int32 by default);
* the in-CSR (transpose) is built lazily on first use -- the push superstep
  never needs it;
* ``device_csr()`` returns the device-resident form the B200 engine walks:
  int32 ``row_ptr``/``col_idx`` plus the per-graph tile map built by
  ``pgx_graph_prepare`` -- cached per device, so a graph already in HBM is
  never re-uploaded.

Ingestion (``load_edge_list``) and the binary cache are kept host-side and
byte-compatible with the reference (``PGLCSR1`` format, graph.py:298-373).
"""

from __future__ import annotations

import ctypes
import io
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import GraphLoadError

_CACHE_MAGIC = b"PGLCSR1\n"
_LITTLE = np.little_endian
_TORCH_OF = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
             np.dtype(np.int16): torch.int16}


def _as_tensor(a, dtype=torch.int64, device=None) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a.to(dtype)
    else:
        t = torch.as_tensor(np.asarray(a), dtype=dtype)
    if device is not None:
        t = t.to(device)
    return t.reshape(-1).contiguous()


@dataclass
class DeviceCSR:
    """Device-resident CSR the engine walks (int32, n < 2^31, m < 2^31)."""

    n: int
    m: int
    row_ptr: torch.Tensor   # int32 [n+1]
    col_idx: torch.Tensor   # int32 [m]
    ws: torch.Tensor        # uint8 per-graph workspace (tile map, nz list)
    h2d_bytes: int          # bytes copied host->device to build it
    in_row_ptr: torch.Tensor | None = None   # int32 [n+1] transpose (pull mode)
    in_col: torch.Tensor | None = None       # int32 [m], rows sorted by source
    in_ws: torch.Tensor | None = None        # tile map of the transpose
    hub_col: torch.Tensor | None = None      # col_idx with hub edges encoded
    hub_ids: torch.Tensor | None = None      # hub slot -> vertex
    pr_hub_col: torch.Tensor | None = None   # in_col with hub-source edges encoded
    pr_hub_slot: torch.Tensor | None = None  # vertex -> hub slot (or -1)
    pr_nhubs: int = 0
    runs: int = 0                            # device runs on this CSR
    seg: object = None                       # _lib.PgxSegIndex (segmented scatter)
    seg_arrays: tuple = ()                   # the tensors seg points into

    def ensure_segments(self, stream=None, seg_log2: int | None = None) -> None:
        """Build the destination-segmented index (pgx_seg_count /
        pgx_seg_build: run detection, stable radix sort by segment, 16-bit
        destinations, tile map, work items) once per graph and device.
        Graph preprocessing, like the tile map and the in-CSR."""
        if self.seg is not None or self.m == 0:
            return
        dev = self.row_ptr.device
        st = torch.cuda.current_stream(dev) if stream is None else stream
        lib = _lib.load()
        L = _lib.PGX_SEG_LOG2_DEFAULT if seg_log2 is None else int(seg_log2)
        n, m = self.n, self.m
        with torch.cuda.device(dev), torch.cuda.stream(st):
            sp = st.cuda_stream
            ws = torch.empty(_lib.out_size(lib.pgx_seg_workspace_bytes, n, m, -1, L),
                             dtype=torch.uint8, device=dev)
            nent = ctypes.c_int64(0)
            _lib.check(lib.pgx_seg_count(n, m, self.row_ptr.data_ptr(), self.col_idx.data_ptr(),
                                         self.ws.data_ptr(), L, ws.data_ptr(), ws.numel(),
                                         ctypes.byref(nent), sp), "pgx_seg_count")
            ne = int(nent.value)
            del ws
            ws = torch.empty(_lib.out_size(lib.pgx_seg_workspace_bytes, n, m, ne, L),
                             dtype=torch.uint8, device=dev)
            cap = ctypes.c_int32(0)
            _lib.check(lib.pgx_seg_max_items(n, m, L, ctypes.byref(cap)), "pgx_seg_max_items")
            # + 4: the scatter stages entries in 16-byte chunks
            ent_src = torch.zeros(ne + 4, dtype=torch.int32, device=dev)
            ent_eb = torch.empty(ne + 1, dtype=torch.int32, device=dev)
            col16 = torch.empty(m + 256, dtype=torch.int16, device=dev)
            tile_ent = torch.empty((m + 255) // 256 + 1, dtype=torch.int32, device=dev)
            items = torch.empty(4 * int(cap.value), dtype=torch.int32, device=dev)
            nitems = ctypes.c_int32(0)
            _lib.check(lib.pgx_seg_build(n, m, self.row_ptr.data_ptr(), self.col_idx.data_ptr(),
                                         self.ws.data_ptr(), L, ne, ws.data_ptr(), ws.numel(),
                                         ent_src.data_ptr(), ent_eb.data_ptr(), col16.data_ptr(),
                                         tile_ent.data_ptr(), items.data_ptr(),
                                         ctypes.byref(nitems), 0, sp), "pgx_seg_build")
            del ws
        # ent_eb (4 B per entry, 3.5 GB on C5) is a build output the scatter
        # never reads (entry boundaries are col16's flags): freed here
        del ent_eb
        self.seg_arrays = (ent_src, col16, tile_ent, items)
        self.seg = _lib.PgxSegIndex(L, ne, int(nitems.value), 0, ent_src.data_ptr(),
                                    None, col16.data_ptr(), tile_ent.data_ptr(),
                                    items.data_ptr())

    def ensure_hubs(self, stream=None) -> None:
        """Encode the hub recipients for the scatter's shared-memory combiner.

        Hubs are the (at most pgx_hub_capacity) highest in-degree vertices;
        an edge into hub h is stored as (0x80000000 | slot(h)).  Graph
        preprocessing, amortised over repeated runs (engine: from the
        second run on a device CSR when ``hub_cache="auto"``).
        """
        if self.hub_col is not None:
            return
        dev = self.row_ptr.device
        st = torch.cuda.current_stream(dev) if stream is None else stream
        lib = _lib.load()
        cap = ctypes.c_int32(0)
        _lib.check(lib.pgx_hub_capacity(ctypes.byref(cap)), "pgx_hub_capacity")
        with torch.cuda.device(dev), torch.cuda.stream(st):
            col = self.col_idx.to(torch.int64)
            indeg = torch.bincount(col, minlength=self.n)
            h = min(int(cap.value), self.n, int(os.environ.get("PGX_HUBS", cap.value)))
            vals, idx = torch.topk(indeg, h, sorted=True)
            idx = idx[vals >= 2]          # a hub must receive >= 2 edges
            slot = torch.full((self.n,), -1, dtype=torch.int32, device=dev)
            slot[idx] = torch.arange(idx.numel(), dtype=torch.int32, device=dev)
            s = slot[col]
            del col
            enc = torch.where(s >= 0, s | torch.tensor(-2 ** 31, dtype=torch.int32, device=dev),
                              self.col_idx)
            self.hub_col, self.hub_ids = enc.contiguous(), idx.to(torch.int32).contiguous()

    def ensure_pr_hubs(self, stream=None) -> None:
        """Encode the hub SOURCES of the pull fold (pgx_pagerank_pull_hubs_run).

        Hubs are the (at most pgx_pr_hub_capacity) highest out-degree
        vertices; an in-CSR edge from hub h is stored as (0x80000000 |
        slot(h)) and its share is read from each CTA's shared-memory table.
        Needs the transpose; one pass over in_col, once per graph.
        """
        if self.pr_hub_col is not None:
            return
        self.ensure_transpose(stream)
        dev = self.row_ptr.device
        st = torch.cuda.current_stream(dev) if stream is None else stream
        lib = _lib.load()
        cap = ctypes.c_int32(0)
        _lib.check(lib.pgx_pr_hub_capacity(ctypes.byref(cap)), "pgx_pr_hub_capacity")
        h = min(int(cap.value), int(os.environ.get("PGX_PR_HUBS", cap.value)))
        with torch.cuda.device(dev), torch.cuda.stream(st):
            enc, slot, nh = encode_hub_sources(self.row_ptr, self.in_col, h)
            self.pr_hub_col, self.pr_hub_slot, self.pr_nhubs = enc, slot, nh

    def ensure_transpose(self, stream=None) -> None:
        """Build the in-CSR on the device (sort by (dst, src)), once."""
        if self.in_row_ptr is not None:
            return
        dev = self.row_ptr.device
        st = torch.cuda.current_stream(dev) if stream is None else stream
        lib = _lib.load()
        with torch.cuda.device(dev), torch.cuda.stream(st):
            n, m = self.n, self.m
            deg = torch.diff(self.row_ptr.to(torch.int64))
            src = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int64),
                                          deg, output_size=m)
            key = (self.col_idx.to(torch.int64) << 32) | src
            del src
            key, _ = torch.sort(key)
            dst = key >> 32
            in_row_ptr = torch.zeros(n + 1, dtype=torch.int32, device=dev)
            in_row_ptr[1:] = torch.cumsum(torch.bincount(dst, minlength=n), 0).to(torch.int32)
            del dst
            in_col = (key & 0xFFFFFFFF).to(torch.int32)
            del key
            ws_bytes = _lib.out_size(lib.pgx_graph_workspace_bytes, n, m)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            _lib.check(lib.pgx_graph_prepare(n, m, in_row_ptr.data_ptr(), ws.data_ptr(),
                                             ws_bytes, st.cuda_stream), "pgx_graph_prepare")
        self.in_row_ptr, self.in_col, self.in_ws = in_row_ptr, in_col, ws


def encode_hub_sources(row_ptr: torch.Tensor, in_col: torch.Tensor, capacity: int):
    """The pull fold's hub-source encoding (pgx_pagerank_pull_hubs_run):
    hubs are the (at most ``capacity``) highest out-degree vertices that
    send >= 2 edges, in descending out-degree order; an in-CSR edge from
    hub h becomes (0x80000000 | slot(h)).  Returns (encoded in_col, the
    vertex -> slot map with -1 for non-hubs, the hub count)."""
    n = int(row_ptr.numel()) - 1
    dev = in_col.device
    outdeg = torch.diff(row_ptr.to(torch.int64))
    vals, idx = torch.topk(outdeg, min(int(capacity), n), sorted=True)
    idx = idx[vals >= 2]
    slot = torch.full((n,), -1, dtype=torch.int32, device=dev)
    slot[idx] = torch.arange(idx.numel(), dtype=torch.int32, device=dev)
    s = slot[in_col.long()]
    enc = torch.where(s >= 0, s | torch.tensor(-2 ** 31, dtype=torch.int32, device=dev), in_col)
    return enc.contiguous(), slot, int(idx.numel())


class Graph:
    """A directed multigraph in CSR form, with its (lazy) transpose."""

    def __init__(self, vertex_count: int, out_offsets: torch.Tensor,
                 out_targets: torch.Tensor, in_offsets: torch.Tensor | None = None,
                 in_targets: torch.Tensor | None = None, id_map=None,
                 source_path: str | None = None):
        self.vertex_count = int(vertex_count)
        self.out_offsets = out_offsets
        self.out_targets = out_targets
        self._in = None if in_offsets is None else (in_offsets, in_targets)
        self.id_map = id_map
        self.source_path = source_path
        self._device: dict = {}

    # ---- reference surface (graph.py:56-106) --------------------------

    @property
    def edge_count(self) -> int:
        return int(self.out_targets.shape[0])

    @property
    def id_dtype(self):
        return self.out_targets.dtype

    @property
    def in_offsets(self) -> torch.Tensor:
        return self._transpose()[0]

    @property
    def in_targets(self) -> torch.Tensor:
        return self._transpose()[1]

    def _transpose(self):
        if self._in is None:
            self._in = _csr(self.out_targets.to(torch.int64),
                            _expand_sources(self.out_offsets, self.edge_count),
                            self.vertex_count, self.out_targets.dtype)
        return self._in

    def out_neighbors(self, v: int) -> torch.Tensor:
        self._check_vertex(v)
        return self.out_targets[int(self.out_offsets[v]):int(self.out_offsets[v + 1])]

    def in_neighbors(self, v: int) -> torch.Tensor:
        self._check_vertex(v)
        return self.in_targets[int(self.in_offsets[v]):int(self.in_offsets[v + 1])]

    def out_degree(self, v: int) -> int:
        self._check_vertex(v)
        return int(self.out_offsets[v + 1] - self.out_offsets[v])

    def in_degree(self, v: int) -> int:
        self._check_vertex(v)
        return int(self.in_offsets[v + 1] - self.in_offsets[v])

    @property
    def out_degrees(self) -> torch.Tensor:
        return torch.diff(self.out_offsets)

    @property
    def in_degrees(self) -> torch.Tensor:
        return torch.diff(self.in_offsets)

    def original_ids(self, dense):
        if self.id_map is None:
            return np.asarray(dense)
        return np.asarray(self.id_map)[np.asarray(dense)]

    def _check_vertex(self, v: int) -> None:
        if not 0 <= v < self.vertex_count:
            raise IndexError(f"vertex id {v} out of range [0, {self.vertex_count})")

    def __repr__(self) -> str:
        return (f"Graph(vertex_count={self.vertex_count}, "
                f"edge_count={self.edge_count}, id_dtype={self.id_dtype})")

    # ---- placement ----------------------------------------------------

    @property
    def device(self) -> torch.device:
        return self.out_targets.device

    def pin_memory(self) -> "Graph":
        """Host graph with page-locked CSR (fast, async H2D)."""
        g = Graph(self.vertex_count, self.out_offsets.cpu().pin_memory(),
                  self.out_targets.cpu().pin_memory(), id_map=self.id_map,
                  source_path=self.source_path)
        return g

    def drop_device_cache(self) -> None:
        self._device.clear()

    def device_csr(self, device=None, stream=None, defer_targets: bool = False) -> DeviceCSR:
        """The int32 device CSR + tile map, built once per device.

        ``defer_targets`` (host graphs with int32 targets): the targets are
        only allocated on the device; the caller copies them (the CC upload
        pipeline of engine.plan_run) and counts their bytes."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        key = dev.index
        hit = self._device.get(key)
        if hit is not None:
            return hit
        n, m = self.vertex_count, self.edge_count
        if n >= 2 ** 31 - 1 or m >= 2 ** 31:
            raise GraphLoadError("device CSR needs n < 2^31 and m < 2^31 (int32)")
        lib = _lib.load()
        st = torch.cuda.current_stream(dev) if stream is None else stream
        h2d = 0
        with torch.cuda.device(dev), torch.cuda.stream(st):
            off = self.out_offsets
            if off.device != dev:
                h2d += off.numel() * off.element_size()
                off = off.to(dev, non_blocking=True)
            tgt = self.out_targets
            if defer_targets and tgt.device != dev and tgt.dtype == torch.int32:
                col = torch.empty(m, dtype=torch.int32, device=dev)
            else:
                if tgt.device != dev:
                    h2d += tgt.numel() * tgt.element_size()
                    tgt = tgt.to(dev, non_blocking=True)
                col = tgt if tgt.dtype == torch.int32 else tgt.to(torch.int32)
            row_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
            _lib.check(lib.pgx_offsets_to_i32(off.to(torch.int64).data_ptr(),
                                              row_ptr.data_ptr(), n + 1,
                                              st.cuda_stream), "pgx_offsets_to_i32")
            ws_bytes = _lib.out_size(lib.pgx_graph_workspace_bytes, n, m)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            if n > 0:
                _lib.check(lib.pgx_graph_prepare(n, m, row_ptr.data_ptr(),
                                                 ws.data_ptr(), ws_bytes,
                                                 st.cuda_stream),
                           "pgx_graph_prepare")
        d = DeviceCSR(n, m, row_ptr, col, ws, h2d)
        self._device[key] = d
        return d


@dataclass(frozen=True)
class DegreeStats:
    """graph.py:109-123: degree summary used by the edge-balanced split."""

    degrees: torch.Tensor
    prefix: torch.Tensor
    min_degree: int
    max_degree: int
    mean_degree: float


def degree_prefix_sums(graph: Graph, *, incoming: bool = False) -> DegreeStats:
    degrees = graph.in_degrees if incoming else graph.out_degrees
    prefix = torch.cumsum(degrees, 0, dtype=torch.int64)
    if degrees.numel() == 0:
        return DegreeStats(degrees, prefix, 0, 0, 0.0)
    return DegreeStats(degrees, prefix, int(degrees.min()), int(degrees.max()),
                       float(degrees.double().mean()))


# ----------------------------------------------------------------------
# construction
# ----------------------------------------------------------------------

def _expand_sources(offsets: torch.Tensor, m: int) -> torch.Tensor:
    n = offsets.numel() - 1
    deg = torch.diff(offsets)
    return torch.repeat_interleave(torch.arange(n, dtype=torch.int64,
                                                device=offsets.device), deg,
                                   output_size=m)


def _csr(key: torch.Tensor, val: torch.Tensor, n: int, id_dtype):
    """graph.py:179-187: group by key, targets ascending within a row."""
    dev = key.device
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    if key.numel():
        offsets[1:] = torch.cumsum(torch.bincount(key, minlength=n), 0)
        order = torch.argsort(key * max(n, 1) + val)
        targets = val[order].to(id_dtype)
    else:
        targets = torch.empty(0, dtype=id_dtype, device=dev)
    return offsets, targets


def from_edges(src, dst, vertex_count: int, *, undirected: bool = False,
               id_dtype=np.int32, device=None) -> Graph:
    """Build a graph from parallel dense-id edge arrays (graph.py:141-176).

    Every id must be in ``[0, vertex_count)``.  Duplicate edges and
    self-loops are kept; with ``undirected=True`` each input edge (self-loops
    included) is stored in both directions.  ``device`` places the CSR
    (default: where ``src`` lives).
    """
    dev = device
    if dev is None and isinstance(src, torch.Tensor):
        dev = src.device
    src = _as_tensor(src, torch.int64, dev)
    dst = _as_tensor(dst, torch.int64, dev)
    if src.shape != dst.shape:
        raise GraphLoadError("src/dst must be 1-d arrays of equal length")
    if vertex_count < 0:
        raise GraphLoadError(f"vertex_count must be >= 0, got {vertex_count}")
    np_id = np.dtype(id_dtype)
    if not np.issubdtype(np_id, np.integer):
        raise GraphLoadError(f"id dtype must be an integer type, got {np_id}")
    if vertex_count > 0 and vertex_count - 1 > np.iinfo(np_id).max:
        raise GraphLoadError(
            f"vertex count {vertex_count} does not fit id dtype {np_id}")
    tdt = {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
           np.dtype(np.int16): torch.int16}.get(np_id)
    if tdt is None:
        raise GraphLoadError(f"unsupported id dtype {np_id}")
    if src.numel():
        lo = int(torch.minimum(src.min(), dst.min()))
        hi = int(torch.maximum(src.max(), dst.max()))
        if lo < 0 or hi >= vertex_count:
            raise GraphLoadError(
                f"edge endpoint {lo if lo < 0 else hi} outside [0, {vertex_count})")
    if undirected and src.numel():
        src, dst = torch.cat([src, dst]), torch.cat([dst, src])
    out_offsets, out_targets = _csr(src, dst, vertex_count, tdt)
    return Graph(vertex_count, out_offsets, out_targets)


def from_csr(offsets, targets, vertex_count: int | None = None) -> Graph:
    """Wrap an existing row-sorted CSR (e.g. a generator's output)."""
    off = _as_tensor(offsets, torch.int64)
    tgt = targets if isinstance(targets, torch.Tensor) else \
        torch.as_tensor(np.asarray(targets))
    n = off.numel() - 1 if vertex_count is None else int(vertex_count)
    if off.numel() != n + 1 or n < 0:
        raise GraphLoadError("offsets must have vertex_count + 1 entries")
    tgt = tgt.reshape(-1).contiguous()
    m = tgt.numel()
    # the checks load_cache runs (graph.py:325-373): the kernels index the
    # mailbox with these values unchecked
    if int(off[0]) != 0 or int(off[-1]) != m or bool((torch.diff(off) < 0).any()):
        raise GraphLoadError("offsets must start at 0, end at len(targets) and never decrease")
    if m and (int(tgt.min()) < 0 or int(tgt.max()) >= n):
        raise GraphLoadError(f"target id out of range [0, {n})")
    return Graph(n, off, tgt)


def gather_adjacency(offsets, targets, ids):
    """graph.py:380-397: concatenated adjacency slices of ``ids``."""
    offsets = _as_tensor(offsets, torch.int64)
    ids = _as_tensor(ids, torch.int64, offsets.device)
    targets = targets if isinstance(targets, torch.Tensor) else torch.as_tensor(targets)
    starts = offsets[ids]
    lengths = offsets[ids + 1] - starts
    total = int(lengths.sum()) if lengths.numel() else 0
    if total == 0:
        return targets[:0], lengths
    row_ends = torch.cumsum(lengths, 0)
    flat = torch.arange(total, dtype=torch.int64, device=offsets.device)
    flat += torch.repeat_interleave(starts - (row_ends - lengths), lengths)
    return targets[flat], lengths


def densify_ids(src, dst):
    """graph.py:196-211: raw ids -> 0..n-1 in first-appearance order."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    raw = np.empty(src.size * 2, dtype=np.int64)
    raw[0::2] = src
    raw[1::2] = dst
    sorted_ids, first_pos, inverse = np.unique(raw, return_index=True,
                                               return_inverse=True)
    appearance = np.argsort(first_pos, kind="stable")
    rank = np.empty(appearance.size, dtype=np.int64)
    rank[appearance] = np.arange(appearance.size)
    dense = rank[inverse]
    return dense[0::2], dense[1::2], sorted_ids[appearance]


def load_edge_list(path, *, undirected: bool = False, id_dtype=np.int32) -> Graph:
    """Whitespace edge list -> Graph (graph.py:218-291; host-side ingestion)."""
    path = os.fspath(path)
    src, dst = [], []
    try:
        fh = open(path, "rt", encoding="utf-8", errors="replace")
    except OSError as e:
        raise GraphLoadError(f"{path}: {e.strerror}") from e
    with fh:
        for lineno, line in enumerate(fh, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            tok = s.split()
            if len(tok) < 2:
                raise GraphLoadError(f"{path}:{lineno}: expected at least two "
                                     f"vertex ids, got {len(tok)} token(s)")
            try:
                a, b = int(tok[0]), int(tok[1])
            except ValueError:
                raise GraphLoadError(f"{path}:{lineno}: non-integer vertex id "
                                     f"{tok[0]!r} {tok[1]!r}") from None
            if a < 0 or b < 0:
                raise GraphLoadError(f"{path}:{lineno}: negative vertex id")
            src.append(a)
            dst.append(b)
    if not src:
        g = from_edges(np.empty(0, np.int64), np.empty(0, np.int64), 0,
                       id_dtype=id_dtype)
    else:
        s, d, id_map = densify_ids(np.asarray(src), np.asarray(dst))
        g = from_edges(s, d, int(id_map.size), undirected=undirected,
                       id_dtype=id_dtype)
        g.id_map = id_map
    g.source_path = path
    return g


def save_cache(graph: Graph, path) -> None:
    """graph.py:298-322: little-endian PGLCSR1 snapshot."""
    tgt = graph.out_targets.cpu().numpy()
    id_dt = tgt.dtype.newbyteorder("<")
    header = io.BytesIO()
    header.write(_CACHE_MAGIC)
    header.write(id_dt.str.encode("ascii").ljust(8, b"\x00"))
    header.write(np.asarray([graph.vertex_count, graph.edge_count], "<u8").tobytes())
    header.write(bytes([1 if graph.id_map is not None else 0]) + b"\x00" * 7)
    tmp = os.fspath(path) + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(header.getvalue())
        fh.write(np.ascontiguousarray(graph.out_offsets.cpu().numpy(), "<i8").tobytes())
        fh.write(np.ascontiguousarray(tgt, id_dt).tobytes())
        fh.write(np.ascontiguousarray(graph.in_offsets.cpu().numpy(), "<i8").tobytes())
        fh.write(np.ascontiguousarray(graph.in_targets.cpu().numpy(), id_dt).tobytes())
        if graph.id_map is not None:
            fh.write(np.ascontiguousarray(graph.id_map, "<i8").tobytes())
    os.replace(tmp, path)


def load_cache(path, *, device=None, pin_memory: bool = False) -> Graph:
    """graph.py:325-373: read and validate a PGLCSR1 snapshot.

    The reference reads the whole file into one blob and copies every array
    out of it.  Here each array is read straight into its own host tensor
    (``readinto``, no intermediate copy) -- page-locked when ``pin_memory``
    is set or a CUDA ``device`` is given, in which case the arrays are then
    uploaded asynchronously and the CSR is validated on the device.  The
    checks and their error messages are the reference's.
    """
    path = os.fspath(path)
    try:
        fh = open(path, "rb")
    except OSError as e:
        raise GraphLoadError(f"{path}: {e.strerror}") from e
    with fh:
        head = fh.read(40)
        size = os.fstat(fh.fileno()).st_size
        if len(head) < 32 or head[:8] != _CACHE_MAGIC:
            raise GraphLoadError(f"{path}: not a graph cache (bad magic/version)")
        if len(head) < 40:
            raise GraphLoadError(f"{path}: truncated graph cache")
        try:
            id_dt = np.dtype(head[8:16].rstrip(b"\x00").decode("ascii"))
        except (TypeError, UnicodeDecodeError) as e:
            raise GraphLoadError(f"{path}: unreadable id dtype tag") from e
        if id_dt.newbyteorder("=") not in _TORCH_OF:
            raise GraphLoadError(f"{path}: unsupported id dtype {id_dt}")
        n, m = (int(x) for x in np.frombuffer(head[16:32], dtype="<u8"))
        has_id_map = head[32] == 1
        dev = torch.device(device) if device is not None else None
        pin = pin_memory or (dev is not None and dev.type == "cuda")
        i8 = np.dtype("<i8")
        parts = [(n + 1, i8), (m, id_dt), (n + 1, i8), (m, id_dt)]
        if has_id_map:
            parts.append((n, i8))
        need = 40 + sum(c * d.itemsize for c, d in parts)
        if size < need:
            raise GraphLoadError(f"{path}: truncated graph cache")
        if size > need:
            raise GraphLoadError(f"{path}: trailing bytes in graph cache")
        arrays = []
        for count, dt in parts:
            t = torch.empty(count, dtype=_TORCH_OF[dt.newbyteorder("=")], pin_memory=pin)
            buf = memoryview(t.numpy()).cast("B")
            if fh.readinto(buf) != len(buf):
                raise GraphLoadError(f"{path}: truncated graph cache")
            if dt.byteorder == ">" or (dt.byteorder == "=" and not _LITTLE):
                t = t.numpy().byteswap().view(dt.newbyteorder("="))
                t = torch.from_numpy(t)
            arrays.append(t)
    out_off, out_tgt, in_off, in_tgt = arrays[:4]
    id_map = arrays[4].numpy() if has_id_map else None
    if dev is not None:
        out_off, out_tgt, in_off, in_tgt = (a.to(dev, non_blocking=True)
                                            for a in (out_off, out_tgt, in_off, in_tgt))
    for offs in (out_off, in_off):
        if int(offs[0]) != 0 or int(offs[-1]) != m or bool((torch.diff(offs) < 0).any()):
            raise GraphLoadError(f"{path}: corrupt offsets in graph cache")
    if m and (int(out_tgt.max()) >= n or int(in_tgt.max()) >= n
              or int(out_tgt.min()) < 0 or int(in_tgt.min()) < 0):
        raise GraphLoadError(f"{path}: target id out of range in graph cache")
    return Graph(n, out_off, out_tgt, in_off, in_tgt, id_map=id_map, source_path=path)
