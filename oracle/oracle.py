"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module; the product package never does.  It wraps
`liboracle.so` (ipgc_oracle.c, a C restatement of the reference hot path, see
that file's header for the per-function citations) with ctypes and carries a
pure-numpy twin of the synthetic generators so the C generators are pinned by a
second, independent implementation.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB = None

MODE_CODES = {"data": 0, "topo": 1, "hybrid": 2}


def lib():
    global _LIB
    if _LIB is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            import subprocess

            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = ctypes.CDLL(str(path))
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.orc_hash.restype = ctypes.c_uint64
        L.orc_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_grid_num_edges.restype = i64
        L.orc_grid_num_edges.argtypes = [i64, i64]
        L.orc_gen_grid.argtypes = [i64, i64, p]
        L.orc_gen_er.argtypes = [i64, i64, ctypes.c_uint64, p]
        L.orc_gen_rmat.argtypes = [ctypes.c_int, i64, ctypes.c_uint64, p]
        L.orc_build_csr.restype = i64
        L.orc_build_csr.argtypes = [i64, i64, p, p, p]
        L.orc_color.restype = i64
        L.orc_color.argtypes = [i64, p, p, ctypes.c_int, i64, p, p, i64]
        L.orc_verify.restype = i64
        L.orc_verify.argtypes = [i64, p, p, p]
        L.orc_colors_used.restype = i64
        L.orc_colors_used.argtypes = [i64, p]
        L.orc_num_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# generators (C) -- SURVEY.md Appendix C
# --------------------------------------------------------------------------
def grid_num_edges(rows: int, cols: int) -> int:
    return int(lib().orc_grid_num_edges(rows, cols))


def gen_grid(rows: int, cols: int) -> np.ndarray:
    m = lib().orc_grid_num_edges(rows, cols)
    e = np.empty((m, 2), dtype=np.int64)
    if m:
        lib().orc_gen_grid(rows, cols, _ptr(e))
    return e


def gen_er(n: int, m: int, seed: int = 0) -> np.ndarray:
    e = np.empty((m, 2), dtype=np.int64)
    if m:
        lib().orc_gen_er(n, m, seed, _ptr(e))
    return e


def gen_rmat(scale: int, edgefactor: int = 16, seed: int = 0) -> np.ndarray:
    m = edgefactor << scale
    e = np.empty((m, 2), dtype=np.int64)
    if m:
        lib().orc_gen_rmat(scale, m, seed, _ptr(e))
    return e


# --------------------------------------------------------------------------
# numpy twin of the generators (independent second implementation)
# --------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def np_splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def np_hash(seed: int, k: np.ndarray, l: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) << np.uint64(40)) + (k.astype(np.uint64) << np.uint64(6)) + np.uint64(l)
    return np_splitmix64(key)


def np_gen_grid(rows: int, cols: int) -> np.ndarray:
    """conftest.grid_graph edge order (pkg/tests/conftest.py:30-41)."""
    edges = []
    for i in range(rows):
        for j in range(cols):
            u = i * cols + j
            if i + 1 < rows:
                edges.append((u, u + cols))
            if j + 1 < cols:
                edges.append((u, u + 1))
    return np.array(edges, dtype=np.int64).reshape(-1, 2)


def np_gen_er(n: int, m: int, seed: int = 0) -> np.ndarray:
    k = np.arange(m, dtype=np.uint64)
    src = (np_hash(seed, k, 0) % np.uint64(n)).astype(np.int64)
    dst = (np_hash(seed, k, 1) % np.uint64(n)).astype(np.int64)
    return np.column_stack([src, dst])


RMAT_THRESHOLDS = (
    round(0.57 * 2**32),
    round(0.57 * 2**32) + round(0.19 * 2**32),
    round(0.57 * 2**32) + 2 * round(0.19 * 2**32),
)


def np_gen_rmat(scale: int, edgefactor: int = 16, seed: int = 0) -> np.ndarray:
    m = edgefactor << scale
    k = np.arange(m, dtype=np.uint64)
    ta, tb, tc = (np.uint64(t) for t in RMAT_THRESHOLDS)
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    for l in range(scale):
        r = np_hash(seed, k, l) >> np.uint64(32)
        sb = r >= tb
        db = ((r >= ta) & (r < tb)) | (r >= tc)
        src |= sb.astype(np.int64) << l
        dst |= db.astype(np.int64) << l
    return np.column_stack([src, dst])


# --------------------------------------------------------------------------
# CSR + solve
# --------------------------------------------------------------------------
def build_csr(n: int, edges: np.ndarray):
    """graph.py:184-201 restated in C; returns (row_offsets, col_indices) int64."""
    edges = np.ascontiguousarray(edges, dtype=np.int64).reshape(-1, 2)
    m = edges.shape[0]
    ro = np.zeros(n + 1, dtype=np.int64)
    ci = np.empty(max(2 * m, 1), dtype=np.int64)
    mdir = lib().orc_build_csr(n, m, _ptr(edges), _ptr(ro), _ptr(ci))
    return ro, ci[:mdir].copy()


def color(ro: np.ndarray, ci: np.ndarray, mode: str = "hybrid", threshold_fraction: float = 0.6,
          max_rec: int | None = None):
    """driver.py:122-176 restated in C.

    Returns (colors int64[n], records int64[rounds, 4]) with record columns
    (topo flag, wl_in, wl_out, conflicts)."""
    ro = np.ascontiguousarray(ro, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    n = ro.shape[0] - 1
    thr = math.ceil(threshold_fraction * n)  # driver.py:138
    if max_rec is None:
        max_rec = max(n, 1)
    colors = np.zeros(max(n, 1), dtype=np.int64)
    rec = np.zeros((max_rec, 4), dtype=np.int64)
    rounds = lib().orc_color(n, _ptr(ro), _ptr(ci if ci.size else np.zeros(1, np.int64)),
                             MODE_CODES[mode], thr, _ptr(colors), _ptr(rec), max_rec)
    return colors[:n].copy(), rec[: min(rounds, max_rec)].copy()


def verify(ro, ci, colors) -> int:
    ro = np.ascontiguousarray(ro, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    colors = np.ascontiguousarray(colors, dtype=np.int64)
    n = ro.shape[0] - 1
    if ci.size == 0:
        return 0
    return lib().orc_verify(n, _ptr(ro), _ptr(ci), _ptr(colors))


def num_threads() -> int:
    return lib().orc_num_threads()


def reference_module():
    """The reference package compiled into oracle/_ref (oracle/build_ref.sh), or None."""
    ref = HERE / "_ref"
    if not (ref / "hybridcolor").exists():
        return None
    import sys

    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import hybridcolor  # noqa: F401

    return hybridcolor


if __name__ == "__main__":  # pragma: no cover
    print("oracle threads:", num_threads(), "reference:", reference_module())
    os._exit(0)
