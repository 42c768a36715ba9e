"""Graph ingestion and degree statistics.

Same surface and error behaviour as the reference's graph I/O
(pkg/src/hybridcolor/graph.py): `MatrixMarketError` (23-24),
`parse_matrix_market` (105-181), `DegreeStats` / `degree_stats` (96-102,
204-217), `save_csr_cache` / `load_csr_cache` (220-244), `load_graph`
(247-254).  What moves to the GPU is the O(file) work:

  * the banner and the size line are parsed here, on the host, exactly as the
    reference does (graph.py:119-150) -- a few bytes;
  * the entry section is uploaded as raw bytes and parsed by hc_mtx_parse
    (hcb_ingest.cu): line split, comment / blank filtering, int() parsing,
    bounds and count checks, first-bad-line error ranking;
  * `load_graph_device` keeps the edges in HBM and builds the CSR there
    (hc_build_csr), so a .mtx file goes to a DeviceCsr without any host pass
    over the entries;
  * `degree_stats` is a device radix select (hc_degree_stats).

The .npz cache is the reference's own host file format (np.savez / np.load),
kept byte-compatible.

Deviation (documented): the device parser reads ASCII.  Files with a byte
>= 0x80 raise UnicodeDecodeError like the reference's ascii-mode open; str /
text inputs with non-ASCII characters are rejected with MatrixMarketError
instead of being split on Unicode whitespace.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, TextIO

import numpy as np
import torch

from . import _lib
from .graph import ID_DTYPE, CsrGraph, DeviceCsr, EdgeList, build_csr_device

CACHE_FORMAT_VERSION = 1  # graph.py:21

HC_MTX_FEW_FIELDS = 1
HC_MTX_NON_INTEGER = 2
HC_MTX_BOUNDS = 3
HC_MTX_TOO_MANY = 4


class MatrixMarketError(ValueError):
    """Malformed or out-of-contract Matrix Market input (graph.py:23-24)."""


@dataclass
class DegreeStats:
    min_degree: int
    median_degree: int
    max_degree: int
    num_nodes: int
    num_undirected_edges: int


# --------------------------------------------------------------------------
# host: banner + size line (graph.py:119-150)
# --------------------------------------------------------------------------
def _next_line(data: bytes, pos: int, universal: bool):
    """(line, next_pos) of the text line starting at pos, or (None, pos) at
    the end.  universal: '\\r', '\\r\\n' also end a line (text-mode files)."""
    if pos >= len(data):
        return None, pos
    j = data.find(b"\n", pos)
    if universal:
        k = data.find(b"\r", pos)
        if k >= 0 and (j < 0 or k < j):
            nxt = k + 2 if data[k + 1:k + 2] == b"\n" else k + 1
            return data[pos:k + 1], nxt
    if j < 0:
        return data[pos:], len(data)
    return data[pos:j + 1], j + 1


def _header(data: bytes, universal: bool):
    """(rows, cols, nnz, offset of the entry section)."""
    banner, pos = _next_line(data, 0, universal)
    if banner is None:
        raise MatrixMarketError("empty input: missing MatrixMarket banner")
    banner = banner.decode("ascii")
    tokens = banner.split()
    if (len(tokens) < 3 or tokens[0].lower() != "%%matrixmarket" or tokens[1].lower() != "matrix"
            or tokens[2].lower() != "coordinate"):
        raise MatrixMarketError(
            f"malformed banner (expected '%%MatrixMarket matrix coordinate ...'): {banner.strip()!r}")
    size_line = None
    while True:
        line, pos = _next_line(data, pos, universal)
        if line is None:
            break
        stripped = line.decode("ascii").strip()
        if not stripped or stripped.startswith("%"):
            continue
        size_line = stripped
        break
    if size_line is None:
        raise MatrixMarketError("missing size line")
    parts = size_line.split()
    if len(parts) != 3:
        raise MatrixMarketError(f"size line must be 'rows cols nnz': {size_line!r}")
    try:
        rows, cols, nnz = (int(p) for p in parts)
    except ValueError:
        raise MatrixMarketError(f"non-integer size line: {size_line!r}") from None
    if rows < 0 or cols < 0 or nnz < 0:
        raise MatrixMarketError(f"negative size entry: {size_line!r}")
    return rows, cols, nnz, pos


def _line_message(code: int, line: str, rows: int, cols: int, nnz: int) -> str:
    """The reference's message for the bad line the device found (graph.py:158-176)."""
    stripped = line.strip()
    if code == HC_MTX_FEW_FIELDS:
        return f"entry needs at least two coordinates: {stripped!r}"
    if code == HC_MTX_NON_INTEGER:
        return f"non-integer coordinate: {stripped!r}"
    if code == HC_MTX_BOUNDS:
        fields = stripped.split()
        return f"coordinate ({int(fields[0])}, {int(fields[1])}) outside declared bounds {rows}x{cols}"
    return f"more than the declared {nnz} entries"


# --------------------------------------------------------------------------
# device: entry section
# --------------------------------------------------------------------------
def _parse_device(data: bytes, universal: bool, dev=None) -> tuple[int, torch.Tensor]:
    """(num_nodes, device int64[nnz, 2] edges) of a whole MatrixMarket text."""
    rows, cols, nnz, off = _header(data, universal)
    dev = dev or _lib.device()
    L = _lib.load()
    body = np.frombuffer(data, dtype=np.uint8)[off:]
    nb = int(body.size)
    d_body = torch.from_numpy(body.copy()).pin_memory().to(dev, non_blocking=True) if nb else \
        torch.empty(1, dtype=torch.uint8, device=dev)
    edges = torch.empty((max(nnz, 1), 2), dtype=torch.int64, device=dev)
    ws = _lib.workspace(L.hc_mtx_workspace_bytes(nb), dev)
    nent, eline, ecode = ctypes.c_int64(0), ctypes.c_int64(-1), ctypes.c_int(0)
    span = (ctypes.c_int64 * 2)()
    nonascii = ctypes.c_int64(-1)
    _lib.check(L.hc_mtx_parse(d_body.data_ptr(), nb, int(universal), rows, cols, nnz, edges.data_ptr(),
                              ctypes.byref(nent), ctypes.byref(eline), ctypes.byref(ecode), span,
                              ctypes.byref(nonascii), ws.data_ptr(), ws.numel(), _lib.stream_handle()))
    del ws
    if nonascii.value >= 0:
        pos = off + int(nonascii.value)
        raise UnicodeDecodeError("ascii", data, pos, pos + 1, "ordinal not in range(128)")
    if eline.value >= 0:
        line = bytes(body[span[0]:span[1]]).decode("ascii")
        raise MatrixMarketError(_line_message(ecode.value, line, rows, cols, nnz))
    if nent.value != nnz:
        raise MatrixMarketError(f"declared {nnz} entries but found {nent.value}")
    return max(rows, cols), edges[:nnz]


def _source_bytes(source) -> tuple[bytes, bool]:
    if isinstance(source, (bytes, bytearray)):
        data = bytes(source)
    elif isinstance(source, str):
        data = source.encode("utf-8")
    elif hasattr(source, "read"):
        text = source.read()
        data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    else:  # an iterable of lines
        data = "".join(ln if ln.endswith("\n") else ln + "\n" for ln in source).encode("utf-8")
    if not data.isascii():
        raise MatrixMarketError("non-ASCII MatrixMarket text is not supported by the device parser")
    return data, False


def parse_matrix_market(source: TextIO | Iterable[str] | str) -> EdgeList:
    """graph.py:105-181 with the entry section parsed on the GPU.  Returns the
    reference's EdgeList (host int64 pairs)."""
    data, universal = _source_bytes(source)
    n, edges = _parse_device(data, universal)
    return EdgeList(n, edges.cpu().numpy())


def load_graph_device(path: str | Path) -> DeviceCsr:
    """.mtx -> device parse -> device build_csr, or an .npz cache uploaded."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"graph file not found: {path}")
    if path.suffix == ".npz":
        return load_csr_cache(path).to_device()
    n, edges = _parse_device(path.read_bytes(), True)
    if n == 0 or edges.shape[0] == 0:  # graph.py:188-189
        return CsrGraph(n, 0, np.zeros(n + 1, dtype=ID_DTYPE), np.empty(0, dtype=ID_DTYPE)).to_device()
    return build_csr_device(edges, n)


def load_graph(path: str | Path) -> CsrGraph:
    """graph.py:247-254: a .mtx file or a .npz CSR cache -> host CsrGraph."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"graph file not found: {path}")
    if path.suffix == ".npz":
        return load_csr_cache(path)
    return load_graph_device(path).to_host()


def save_csr_cache(graph, path: str | Path) -> None:
    """graph.py:220-228 (same .npz layout)."""
    if isinstance(graph, DeviceCsr):
        graph = graph.to_host()
    np.savez(path, format_version=np.array([CACHE_FORMAT_VERSION], dtype=ID_DTYPE),
             num_nodes=np.array([graph.num_nodes], dtype=ID_DTYPE),
             row_offsets=graph.row_offsets, col_indices=graph.col_indices)


def load_csr_cache(path: str | Path) -> CsrGraph:
    """graph.py:231-244 (format-version check, same messages)."""
    with np.load(path) as data:
        if "format_version" not in data:
            raise ValueError(f"{path}: not a CSR cache (missing format_version)")
        version = int(data["format_version"][0])
        if version != CACHE_FORMAT_VERSION:
            raise ValueError(f"{path}: cache format version {version} unsupported "
                             f"(expected {CACHE_FORMAT_VERSION})")
        row_offsets = data["row_offsets"]
        col_indices = data["col_indices"]
        return CsrGraph(int(data["num_nodes"][0]), col_indices.shape[0], row_offsets, col_indices)


def degree_stats(graph) -> DegreeStats:
    """graph.py:204-217 on the device: min / median (sorted element n//2) / max."""
    n = graph.num_nodes
    if n == 0:
        raise ValueError("degree statistics are undefined for an empty graph")
    dg = graph if isinstance(graph, DeviceCsr) else CsrGraph(
        graph.num_nodes, graph.num_edges, graph.row_offsets, graph.col_indices).to_device()
    L = _lib.load()
    ws = _lib.workspace(L.hc_degree_stats_workspace_bytes(), dg.device)
    lo, med, hi = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(L.hc_degree_stats(dg.row_offsets.data_ptr(), n, ctypes.byref(lo), ctypes.byref(med),
                                 ctypes.byref(hi), ws.data_ptr(), ws.numel(), _lib.stream_handle()))
    return DegreeStats(min_degree=int(lo.value), median_degree=int(med.value), max_degree=int(hi.value),
                       num_nodes=n, num_undirected_edges=graph.num_edges // 2)
