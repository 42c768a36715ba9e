"""1D-partitioned multi-GPU hybrid IPGC.

One process per GPU.  The node range is split into P contiguous, edge-balanced
ranges [lo_p, hi_p); rank p processes only its owned nodes but keeps a
replicated copy of the state word X[n] (the single-GPU solver's encoding,
hcb_solve.cu: 0 / T / C|FBIT).  A round (reference coloring.py:113-176):

  1. assign the owned active nodes            (hc_dist_assign)
  2. exchange A: all-gather-v of (u, T) for owned *boundary* nodes, apply
  3. resolve the owned active nodes           (hc_dist_resolve)
  4. exchange B: all-gather-v of boundary winners (u, C|FBIT), apply
  5. all-reduce (|W'|, sum k_u): every rank makes the identical mode decision
     (driver.py:147-152) and termination test (driver.py:145)

Interior nodes are never exchanged -- no other rank reads them.  Because the
round reads only the previous snapshot (assign) and same-round tentatives
(resolve) and ties break by id, every partition gives the bit-identical
coloring, round count and per-round records of the single-GPU solve.

Collectives go through torch.distributed: NCCL over NVLink/NVSwitch on GPUs;
gloo in the CPU tests, where the per-phase kernels are replaced by a CPU
stand-in (`ops=`) so the exchange / partition / termination logic can be
tested without a GPU.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .driver import HybridConfig, RoundRecord, RunReport, threshold_count

FBIT = 0x80000000


def partition_bounds(row_offsets, world: int) -> list[tuple[int, int]]:
    """Edge-balanced contiguous node ranges: cut p sits at the first node whose
    row starts at or after m*p/P half-edges (node-balanced when m == 0)."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n = len(ro) - 1
    m = int(ro[-1]) if n >= 0 else 0
    cuts = [0]
    for p in range(1, world):
        if m > 0:
            c = int(np.searchsorted(ro, (m * p) // world, side="left"))
        else:
            c = (n * p) // world
        cuts.append(min(max(c, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[p], cuts[p + 1]) for p in range(world)]


class Exchange:
    """Variable-size all-gather and all-reduce over a torch.distributed group.
    Pairs travel packed as int64 (id << 32 | value)."""

    def __init__(self, group=None, device: torch.device | None = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        self.host_staged = backend == "gloo"  # gloo collectives run on host tensors
        self.device = device

    def _comm(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host_staged else t

    def allreduce(self, values) -> list[int]:
        t = torch.tensor(list(values), dtype=torch.int64, device=self.device)
        t = self._comm(t)
        dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.tolist()]

    def allgather_pairs(self, ids: torch.Tensor, vals: torch.Tensor, count: int):
        """Every rank's (ids, vals)[:count] concatenated in rank order."""
        cnt = self._comm(torch.tensor([count], dtype=torch.int64, device=ids.device))
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts, cnt, group=self.group)
        counts = [int(c.item()) for c in counts]
        mx = max(counts)
        if mx == 0:
            return ids[:0], vals[:0]
        packed = torch.zeros(mx, dtype=torch.int64, device=ids.device)
        if count:
            packed[:count] = (ids[:count].to(torch.int64) << 32) | (vals[:count].to(torch.int64) & 0xFFFFFFFF)
        packed = self._comm(packed)
        out = torch.empty(self.world * mx, dtype=torch.int64, device=packed.device)
        dist.all_gather_into_tensor(out, packed, group=self.group)
        out = out.view(self.world, mx)
        parts = [out[p, : counts[p]] for p in range(self.world) if counts[p]]
        allp = torch.cat(parts).to(ids.device)
        return (allp >> 32).to(torch.int32), (allp & 0xFFFFFFFF).to(torch.int64)

    def allgather_colors(self, colors: torch.Tensor, bounds) -> torch.Tensor:
        mx = max(hi - lo for lo, hi in bounds)
        buf = torch.zeros(max(mx, 1), dtype=torch.int64, device=colors.device)
        buf[: colors.numel()] = colors
        buf = self._comm(buf)
        out = torch.empty(self.world * buf.numel(), dtype=torch.int64, device=buf.device)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        out = out.view(self.world, -1)
        return torch.cat([out[p, : hi - lo] for p, (lo, hi) in enumerate(bounds)])


class DeviceOps:
    """Per-phase kernels of libhcb (include/hcb.h hc_dist_*) on CUDA tensors."""

    def __init__(self, ro: torch.Tensor, ci: torch.Tensor, n: int):
        self.L = _lib.load()
        self.ro, self.ci, self.n = ro, ci, n
        self.dev = ro.device
        self.cnt = torch.zeros(4, dtype=torch.int64, device=self.dev)  # out, next, conflicts, spare

    def new_state(self):
        return torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)

    def buffers(self, lo, hi):
        k = max(hi - lo, 1)
        self.ids = torch.empty(k, dtype=torch.int32, device=self.dev)
        self.vals = torch.empty(k, dtype=torch.int32, device=self.dev)
        self.nxt = [torch.empty(k, dtype=torch.int32, device=self.dev) for _ in range(2)]

    def boundary(self, lo, hi):
        flags = torch.zeros(max(hi - lo, 1), dtype=torch.uint8, device=self.dev)
        _lib.check(self.L.hc_dist_boundary(self.ro.data_ptr(), _lib.ptr(self.ci), lo, hi, flags.data_ptr(),
                                           _lib.stream_handle()))
        return flags

    def assign(self, X, items, count, lo, boundary):
        self.cnt.zero_()
        _lib.check(self.L.hc_dist_assign(self.ro.data_ptr(), _lib.ptr(self.ci), X.data_ptr(), _lib.ptr(items),
                                         count, lo, boundary.data_ptr(), self.ids.data_ptr(), self.vals.data_ptr(),
                                         self.cnt.data_ptr(), _lib.stream_handle()))
        return self.ids, self.vals, int(self.cnt[0].item())

    def resolve(self, X, items, count, lo, boundary, out_slot):
        self.cnt.zero_()
        nxt = self.nxt[out_slot]
        base = self.cnt.data_ptr()
        _lib.check(self.L.hc_dist_resolve(self.ro.data_ptr(), _lib.ptr(self.ci), X.data_ptr(), _lib.ptr(items),
                                          count, lo, boundary.data_ptr(), nxt.data_ptr(), base + 8,
                                          self.ids.data_ptr(), self.vals.data_ptr(), base, base + 16,
                                          _lib.stream_handle()))
        out, nc, conf = (int(v) for v in self.cnt[:3].tolist())
        return nxt, nc, self.ids, self.vals, out, conf

    def apply(self, X, ids, vals):
        k = int(ids.numel())
        if k:
            v32 = vals.to(torch.int32) if vals.dtype != torch.int32 else vals
            _lib.check(self.L.hc_dist_apply(X.data_ptr(), ids.data_ptr(), v32.contiguous().data_ptr(), k,
                                            _lib.stream_handle()))

    def colors(self, X, lo, hi):
        out = torch.empty(max(hi - lo, 1), dtype=torch.int64, device=self.dev)
        _lib.check(self.L.hc_dist_colors(X.data_ptr(), lo, hi, out.data_ptr(), _lib.stream_handle()))
        return out[: hi - lo]


@dataclass
class DistResult:
    colors: np.ndarray
    report: RunReport
    bounds: list
    exchanged_pairs: int
    seconds: float


def dist_color_graph(row_offsets: torch.Tensor, col_indices: torch.Tensor, num_nodes: int,
                     config: HybridConfig | None = None, *, group=None, ops=None,
                     graph_name: str = "graph", host_row_offsets: np.ndarray | None = None) -> DistResult:
    """Partitioned solve of the whole graph (every rank passes the same CSR;
    each rank processes only its owned range).  Returns the full coloring on
    every rank and, on every rank, the RunReport with the global per-round
    records (driver.py:47-119 semantics)."""
    if config is None:
        config = HybridConfig()
    ex = Exchange(group, row_offsets.device)
    world, rank = ex.world, ex.rank
    n = int(num_nodes)
    ro_host = host_row_offsets if host_row_offsets is not None else row_offsets.cpu().numpy()
    bounds = partition_bounds(ro_host, world)
    lo, hi = bounds[rank]
    if ops is None:
        ops = DeviceOps(row_offsets, col_indices, n)
    ops.buffers(lo, hi)
    X = ops.new_state()
    boundary = ops.boundary(lo, hi)
    thr = threshold_count(config, n)
    report = RunReport(graph_name, n, int(ro_host[-1]) // 2 if n else 0, config)

    exchanged = 0
    items, local_cnt, full = None, hi - lo, True  # round 1: W = all owned nodes
    (s,) = ex.allreduce([local_cnt])
    t = 1
    slot = 0
    t0 = time.perf_counter()
    while s > 0:  # driver.py:145
        tr = time.perf_counter()
        topo = config.mode == "topo" or (config.mode == "hybrid" and s > thr)  # driver.py:147-152
        if topo or full:
            it_items, it_count = None, hi - lo  # sweep of the owned range with the activity test
        else:
            it_items, it_count = items, local_cnt
        ids, vals, c = ops.assign(X, it_items, it_count, lo, boundary)
        gi, gv = ex.allgather_pairs(ids, vals, c)
        exchanged += int(gi.numel())
        ops.apply(X, gi, gv)
        nxt, nc, ids, vals, c, conf = ops.resolve(X, it_items, it_count, lo, boundary, slot)
        gi, gv = ex.allgather_pairs(ids, vals, c)
        exchanged += int(gi.numel())
        ops.apply(X, gi, gv)
        s_next, conflicts = ex.allreduce([nc, conf])
        report.per_round.append(RoundRecord(t, "topo" if topo else "data", s, s_next, conflicts,
                                            time.perf_counter() - tr))
        items, local_cnt, full = nxt, nc, False
        slot ^= 1
        s = s_next
        t += 1
    report.total_seconds = time.perf_counter() - t0
    report.total_rounds = len(report.per_round)
    colors = ex.allgather_colors(ops.colors(X, lo, hi), bounds)
    colors_np = colors.cpu().numpy().astype(np.int64)
    report.colors_used = int(colors_np.max()) if n else 0
    return DistResult(colors_np, report, bounds, exchanged, report.total_seconds)
