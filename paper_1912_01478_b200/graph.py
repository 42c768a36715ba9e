"""Graph types and device graph construction.

Mirrors the reference's graph core (pkg/src/hybridcolor/graph.py):
  * `EdgeList`  -- graph.py:28-46 (declared node count + int64 (src, dst) pairs)
  * `CsrGraph`  -- graph.py:49-93 (host int64 CSR, the reference's own layout)
  * `build_csr` -- graph.py:184-201, executed on the GPU (hc_build_csr)
plus the device-resident `DeviceCsr` (int64 row offsets, int32 column ids:
SURVEY.md §8(a) a12) that the solver consumes, and the on-device synthetic
generators of SURVEY.md Appendix C (hc_gen_grid / hc_gen_er / hc_gen_rmat).

MatrixMarket ingestion (device parser), the .npz cache and degree_stats
live in ingest.py (graph.py:96-254).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import torch

from . import _lib

ID_DTYPE = np.int64


@dataclass
class EdgeList:
    """Declared node count plus zero-based (src, dst) pairs (graph.py:28-46)."""

    num_nodes_declared: int
    edges: np.ndarray

    def __post_init__(self):
        self.edges = np.asarray(self.edges, dtype=ID_DTYPE).reshape(-1, 2)
        if self.num_nodes_declared < 0:
            raise ValueError("declared node count must be non-negative")
        if self.edges.size and (self.edges.min() < 0 or self.edges.max() >= self.num_nodes_declared):
            raise ValueError("edge endpoint outside declared node range")

    @property
    def num_edges(self) -> int:
        return self.edges.shape[0]


@dataclass
class CsrGraph:
    """Host CSR in the reference layout (graph.py:49-93): int64 arrays,
    num_edges = directed half-edges."""

    num_nodes: int
    num_edges: int
    row_offsets: np.ndarray
    col_indices: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=ID_DTYPE)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=ID_DTYPE)
        self.row_offsets.flags.writeable = False
        self.col_indices.flags.writeable = False

    @cached_property
    def degrees(self) -> np.ndarray:
        d = np.diff(self.row_offsets)
        d.flags.writeable = False
        return d

    @cached_property
    def max_degree(self) -> int:
        return int(self.degrees.max()) if self.num_nodes else 0

    @property
    def num_undirected_edges(self) -> int:
        return self.num_edges // 2

    def neighbors(self, u: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[u] : self.row_offsets[u + 1]]

    def to_edge_list(self) -> EdgeList:
        """One (u, v) pair per undirected edge, u < v side (graph.py:86-93)."""
        src = np.repeat(np.arange(self.num_nodes, dtype=ID_DTYPE), self.degrees)
        keep = src < self.col_indices
        return EdgeList(self.num_nodes, np.column_stack((src[keep], self.col_indices[keep])))

    @classmethod
    def pinned(cls, g: "CsrGraph") -> "CsrGraph":
        """Copy of `g` whose arrays live in page-locked host memory, so uploads
        are straight DMA (no staging copy)."""
        ro = torch.from_numpy(np.array(g.row_offsets)).pin_memory()
        ci = torch.from_numpy(np.array(g.col_indices)).pin_memory()
        out = cls(g.num_nodes, g.num_edges, ro.numpy(), ci.numpy())
        out._pinned = (ro, ci)
        out._lower_first = getattr(g, "_lower_first", None)
        return out

    def _host_tensors(self):
        pinned = getattr(self, "_pinned", None)
        if pinned is not None:
            return pinned
        ro = torch.from_numpy(np.array(self.row_offsets)).pin_memory()
        ci = torch.from_numpy(np.array(self.col_indices)).pin_memory()
        return ro, ci

    def to_device(self, dev: torch.device | None = None) -> "DeviceCsr":
        """Upload (pinned host memory) and narrow the column ids to int32 on the GPU."""
        dev = dev or _lib.device()
        n, m = self.num_nodes, self.num_edges
        h_ro, h_ci = self._host_tensors()
        ro = h_ro.to(dev, non_blocking=True)
        ci32 = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
        if m:
            ci64 = h_ci[:m].to(dev, non_blocking=True)
            _lib.check(_lib.load().hc_narrow_i64_i32(ci64.data_ptr(), ci32.data_ptr(), m,
                                                      _lib.stream_handle()))
            del ci64
        return DeviceCsr(n, m, ro, ci32, host=self, lower_first=getattr(self, "_lower_first", None))


@dataclass
class DeviceCsr:
    """GPU-resident CSR: row_offsets int64[n+1], col_indices int32[m]."""

    num_nodes: int
    num_edges: int
    row_offsets: torch.Tensor
    col_indices: torch.Tensor
    host: CsrGraph | None = field(default=None, repr=False)
    _ci64: torch.Tensor | None = field(default=None, repr=False)
    # True when every row lists its lower-id neighbours first (build_csr output
    # is sorted, graph.py:193-197); None = unknown (caller-supplied CSR), checked
    # on the device by ensure_lower_first() before a solve.
    lower_first: bool | None = field(default=None, repr=False)

    def ensure_lower_first(self) -> "DeviceCsr":
        """Make each row's lower-id neighbours a prefix of the row (the fused
        solve's early-exit precondition, include/hcb.h).  A caller CSR with
        unsorted rows gets a stable-partitioned copy of its columns on the
        device; solve outputs depend only on the row sets, so the result is
        the reference's (which scans whole rows, _kernels.pyx:106-113)."""
        if self.lower_first or self.num_edges == 0:
            self.lower_first = True
            return self
        L = _lib.load()
        acc = torch.zeros(1, dtype=torch.int64, device=self.device)
        bad = ctypes.c_int64(0)
        _lib.check(L.hc_csr_check_lower_first(self.row_offsets.data_ptr(), _lib.ptr(self.col_indices),
                                              self.num_nodes, acc.data_ptr(), ctypes.byref(bad),
                                              _lib.stream_handle()))
        if bad.value:
            out = torch.empty_like(self.col_indices)
            _lib.check(L.hc_csr_partition_lower_first(self.row_offsets.data_ptr(), _lib.ptr(self.col_indices),
                                                      _lib.ptr(out), self.num_nodes, _lib.stream_handle()))
            self.col_indices = out
            self._ci64 = None
        self.lower_first = True
        return self

    @property
    def num_undirected_edges(self) -> int:
        return self.num_edges // 2

    @property
    def device(self) -> torch.device:
        return self.row_offsets.device

    @cached_property
    def max_degree(self) -> int:
        if self.host is not None:
            return self.host.max_degree
        if self.num_nodes == 0:
            return 0
        L = _lib.load()  # device reduction (hc_degree_stats), no host copy of the offsets
        ws = _lib.workspace(L.hc_degree_stats_workspace_bytes(), self.device)
        lo, med, hi = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(L.hc_degree_stats(self.row_offsets.data_ptr(), self.num_nodes, ctypes.byref(lo),
                                     ctypes.byref(med), ctypes.byref(hi), ws.data_ptr(), ws.numel(),
                                     _lib.stream_handle()))
        return int(hi.value)

    @property
    def col_indices_i64(self) -> torch.Tensor:
        """int64 column ids for the reference-layout plugin kernels (_kernels.pyx)."""
        if self._ci64 is None:
            self._ci64 = self.col_indices.to(torch.int64)
        return self._ci64

    def to_host(self) -> CsrGraph:
        if self.host is None:
            self.host = CsrGraph(self.num_nodes, self.num_edges,
                                 self.row_offsets.cpu().numpy(),
                                 self.col_indices.cpu().numpy().astype(np.int64))
            if self.lower_first:
                self.host._lower_first = True
        return self.host


def _edges_to_device(edge_list: EdgeList, dev) -> torch.Tensor:
    e = np.ascontiguousarray(edge_list.edges, dtype=np.int64)
    return torch.from_numpy(e).to(dev)


def build_csr_device(d_edges: torch.Tensor, num_nodes: int) -> DeviceCsr:
    """build_csr (graph.py:184-201) over a device int64[m, 2] edge tensor."""
    L = _lib.load()
    dev = d_edges.device
    m = int(d_edges.shape[0]) if d_edges.numel() else 0
    n = int(num_nodes)
    ro = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
    ws = _lib.workspace(L.hc_build_csr_workspace_bytes(n, m), dev)
    mdir = ctypes.c_int64(0)
    _lib.check(L.hc_build_csr(_lib.ptr(d_edges), m, n, ro.data_ptr(), ci.data_ptr(),
                              ctypes.byref(mdir), ws.data_ptr(), ws.numel(), _lib.stream_handle()))
    del ws
    md = int(mdir.value)
    ci = ci[:md].clone() if md else ci[:0]
    return DeviceCsr(n, md, ro, ci, lower_first=True)  # rows sorted ascending


def build_csr(edge_list: EdgeList) -> CsrGraph:
    """Reference-compatible build_csr: runs on the GPU, returns the host CsrGraph."""
    n = edge_list.num_nodes_declared
    if n == 0 or edge_list.edges.size == 0:  # graph.py:188-189
        return CsrGraph(n, 0, np.zeros(n + 1, dtype=ID_DTYPE), np.empty(0, dtype=ID_DTYPE))
    dev = _lib.device()
    d = build_csr_device(_edges_to_device(edge_list, dev), n)
    g = d.to_host()
    return g


# --------------------------------------------------------------------------
# synthetic generators, all on device
# --------------------------------------------------------------------------
def grid_num_pairs(rows: int, cols: int) -> int:
    if rows <= 0 or cols <= 0:
        return 0
    return rows * (cols - 1) + (rows - 1) * cols


def gen_grid_edges(rows: int, cols: int, dev=None) -> torch.Tensor:
    """4-neighbour grid, ids i*cols+j, conftest.grid_graph edge order."""
    dev = dev or _lib.device()
    m = grid_num_pairs(rows, cols)
    e = torch.empty((m, 2), dtype=torch.int64, device=dev)
    if m:
        _lib.check(_lib.load().hc_gen_grid(rows, cols, e.data_ptr(), _lib.stream_handle()))
    return e


def gen_er_edges(n: int, m: int, seed: int = 0, dev=None) -> torch.Tensor:
    dev = dev or _lib.device()
    e = torch.empty((m, 2), dtype=torch.int64, device=dev)
    if m:
        _lib.check(_lib.load().hc_gen_er(n, m, seed, e.data_ptr(), _lib.stream_handle()))
    return e


def gen_rmat_edges(scale: int, edgefactor: int = 16, seed: int = 0, dev=None) -> torch.Tensor:
    dev = dev or _lib.device()
    m = edgefactor << scale
    e = torch.empty((m, 2), dtype=torch.int64, device=dev)
    if m:
        _lib.check(_lib.load().hc_gen_rmat(scale, m, seed, e.data_ptr(), _lib.stream_handle()))
    return e


def grid_graph(rows: int, cols: int) -> DeviceCsr:
    return build_csr_device(gen_grid_edges(rows, cols), rows * cols)


def er_graph(n: int, avg_degree: int = 32, seed: int = 0) -> DeviceCsr:
    """n nodes, m = n*avg_degree/2 uniform endpoint pairs."""
    return build_csr_device(gen_er_edges(n, n * avg_degree // 2, seed), n)


def rmat_graph(scale: int, edgefactor: int = 16, seed: int = 0) -> DeviceCsr:
    return build_csr_device(gen_rmat_edges(scale, edgefactor, seed), 1 << scale)


def synthetic(kind: str, **kw) -> DeviceCsr:
    """Named synthetic workload: kind in {grid, er, rmat}."""
    if kind == "grid":
        return grid_graph(kw["rows"], kw["cols"])
    if kind == "er":
        return er_graph(kw["n"], kw.get("avg_degree", 32), kw.get("seed", 0))
    if kind == "rmat":
        return rmat_graph(kw["scale"], kw.get("edgefactor", 16), kw.get("seed", 0))
    raise ValueError(f"unknown synthetic graph kind {kind!r}")

