"""The `cuda` kernel module: the reference's plugin API on the GPU.

Same module surface as pkg/src/hybridcolor/_kernels.pyx:25-187 (and its numpy
twin _kernels_py.py): `NAME`, `PARALLEL` and the six positional functions,
same argument meaning, same in-place mutation of `colors_write`, `stamp`,
`next_ids`, `cursor` and `active`, same return values.  Each function is one
libhcb entry point (hc_k_*, include/hcb.h).

Arrays may be CUDA tensors (int64, contiguous; used in place, no copies) or
numpy arrays -- the reference's own calling convention (coloring.py:127-139)
-- in which case they are staged to the GPU for the call and the mutated ones
are written back.  `workers` / `chunk_size` are accepted for signature parity
and ignored, as the reference's numpy backend does (_kernels_py.py:5-7).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

NAME = "cuda"
PARALLEL = True


class _Args:
    """Stage numpy / tensor arguments on the device; write back on exit."""

    def __init__(self):
        self.back = []
        self.dev = _lib.device()

    def get(self, a, dtype=torch.int64, mutable=False):
        if isinstance(a, torch.Tensor):
            if a.device.type != "cuda" or a.dtype != dtype or not a.is_contiguous():
                raise ValueError("device arguments must be contiguous CUDA tensors of the reference dtype")
            return a
        arr = np.asarray(a)
        host = torch.from_numpy(np.ascontiguousarray(arr).copy() if not arr.flags.writeable else
                                np.ascontiguousarray(arr))
        if host.dtype != dtype:
            host = host.to(dtype)
        t = host.to(self.dev)
        if mutable:
            self.back.append((arr, t))
        return t

    def acc(self, n=1):
        return torch.zeros(n, dtype=torch.int64, device=self.dev)

    def finish(self):
        for arr, t in self.back:
            arr[...] = t.cpu().numpy().astype(arr.dtype, copy=False).reshape(arr.shape)


def _p(t: torch.Tensor):
    return _lib.ptr(t)


def assign_from_list(row_offsets, col_indices, colors_read, colors_write, stamp, nodes,
                     round_no, max_degree, workers, chunk_size):
    """_kernels.pyx:29-58"""
    A = _Args()
    nodes_t = A.get(nodes)
    if nodes_t.numel() == 0:
        return None
    ro, ci, cr = A.get(row_offsets), A.get(col_indices), A.get(colors_read)
    cw, st = A.get(colors_write, mutable=True), A.get(stamp, mutable=True)
    _lib.check(_lib.load().hc_k_assign_from_list(
        _p(ro), _p(ci), _p(cr), _p(cw), _p(st), _p(nodes_t), nodes_t.numel(), int(round_no),
        int(max_degree), _lib.stream_handle()))
    A.finish()
    return None


def assign_sweep(row_offsets, col_indices, colors_read, colors_write, stamp,
                 round_no, max_degree, workers, chunk_size):
    """_kernels.pyx:61-91; returns the number of processed (colors_read==0) nodes."""
    A = _Args()
    ro, ci, cr = A.get(row_offsets), A.get(col_indices), A.get(colors_read)
    cw, st = A.get(colors_write, mutable=True), A.get(stamp, mutable=True)
    acc = A.acc()
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_k_assign_sweep(
        _p(ro), _p(ci), _p(cr), _p(cw), _p(st), cr.numel(), int(round_no), int(max_degree),
        _p(acc), ctypes.byref(out), _lib.stream_handle()))
    A.finish()
    return int(out.value)


def resolve_from_list(row_offsets, col_indices, colors_read, colors_write, stamp, nodes,
                      round_no, next_ids, cursor, workers, chunk_size):
    """_kernels.pyx:94-120; returns the summed conflict count."""
    A = _Args()
    nodes_t = A.get(nodes)
    ro, ci, cr, st = A.get(row_offsets), A.get(col_indices), A.get(colors_read), A.get(stamp)
    cw = A.get(colors_write, mutable=True)
    nxt, cur = A.get(next_ids, mutable=True), A.get(cursor, mutable=True)
    acc = A.acc()
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_k_resolve_from_list(
        _p(ro), _p(ci), _p(cr), _p(cw), _p(st), _p(nodes_t), nodes_t.numel(), int(round_no),
        _p(nxt), nxt.numel(), _p(cur), _p(acc), ctypes.byref(out), _lib.stream_handle()))
    A.finish()
    return int(out.value)


def resolve_sweep(row_offsets, col_indices, colors_read, colors_write, stamp,
                  round_no, next_ids, cursor, workers, chunk_size):
    """_kernels.pyx:123-149"""
    A = _Args()
    ro, ci, cr, st = A.get(row_offsets), A.get(col_indices), A.get(colors_read), A.get(stamp)
    cw = A.get(colors_write, mutable=True)
    nxt, cur = A.get(next_ids, mutable=True), A.get(cursor, mutable=True)
    acc = A.acc()
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_k_resolve_sweep(
        _p(ro), _p(ci), _p(cr), _p(cw), _p(st), cr.numel(), int(round_no),
        _p(nxt), nxt.numel(), _p(cur), _p(acc), ctypes.byref(out), _lib.stream_handle()))
    A.finish()
    return int(out.value)


def bench_from_list(nodes, active, cutoff, next_ids, cursor, workers, chunk_size):
    """_kernels.pyx:152-168"""
    A = _Args()
    nodes_t = A.get(nodes)
    act = A.get(active, dtype=torch.uint8, mutable=True)
    nxt, cur = A.get(next_ids, mutable=True), A.get(cursor, mutable=True)
    _lib.check(_lib.load().hc_k_bench_from_list(
        _p(nodes_t), nodes_t.numel(), _p(act), int(cutoff), _p(nxt), nxt.numel(), _p(cur),
        _lib.stream_handle()))
    A.finish()


def bench_sweep(active, cutoff, next_ids, cursor, workers, chunk_size):
    """_kernels.pyx:171-187"""
    A = _Args()
    act = A.get(active, dtype=torch.uint8, mutable=True)
    nxt, cur = A.get(next_ids, mutable=True), A.get(cursor, mutable=True)
    _lib.check(_lib.load().hc_k_bench_sweep(
        _p(act), act.numel(), int(cutoff), _p(nxt), nxt.numel(), _p(cur), _lib.stream_handle()))
    A.finish()


def commit_list(colors_read, colors_write, nodes):
    """coloring.py:105-106 (_commit_list) on device tensors."""
    _lib.check(_lib.load().hc_k_commit_list(_p(colors_read), _p(colors_write), _p(nodes),
                                            nodes.numel(), _lib.stream_handle()))


def commit_stamped(colors_read, colors_write, stamp, round_no):
    """coloring.py:109-110 (_commit_stamped) on device tensors."""
    _lib.check(_lib.load().hc_k_commit_stamped(_p(colors_read), _p(colors_write), _p(stamp),
                                               colors_read.numel(), int(round_no),
                                               _lib.stream_handle()))
