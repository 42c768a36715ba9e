"""Hybrid IPGC driver: the drop-in for hybridcolor.color_graph.

Same names, argument meaning and error behaviour as the reference driver
(pkg/src/hybridcolor/driver.py): `HybridConfig` (29-44), `RoundRecord`
(47-54), `RunReport` with its JSON / CSV / table views (57-119),
`color_graph` (122-176), `colors_used` (179-185), `verify_coloring`
(188-204).  The difference is where the round loop lives: `color_graph`
hands the whole loop to ONE device-resident solve (hc_solve, a persistent
cooperative kernel: assign -> grid barrier -> resolve -> grid barrier per
round, hybrid mode switch and worklist on the device), so there is no host
round trip per round.  `total_seconds` is the device time of that solve
(CUDA events on the launching stream), the same boundary as the
reference's loop timer (driver.py:144,170); per-round `wall_seconds` come
from %globaltimer stamps taken by the device at every round boundary.
"""

from __future__ import annotations

import csv
import ctypes
import json
import math
from dataclasses import dataclass, field
from types import SimpleNamespace
from typing import IO

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, DeviceCsr

MODES = ("data", "topo", "hybrid")


@dataclass
class HybridConfig:
    """driver.py:29-44.  `workers` / `chunk_size` are accepted and validated
    for signature parity; like the reference's numpy backend
    (_kernels_py.py:5-7) they do not affect the result."""

    threshold_fraction: float = 0.6
    mode: str = "hybrid"
    workers: int = 1
    chunk_size: int = 1024

    def __post_init__(self):
        if not 0.0 <= self.threshold_fraction <= 1.0:
            raise ValueError(f"threshold_fraction must be in [0, 1], got {self.threshold_fraction}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be >= 1")


@dataclass
class RoundRecord:
    round: int
    mode_used: str
    worklist_size_in: int
    worklist_size_out: int
    conflicts: int
    wall_seconds: float


@dataclass
class RunReport:
    graph_name: str
    num_nodes: int
    num_undirected_edges: int
    config: HybridConfig
    per_round: list[RoundRecord] = field(default_factory=list)
    total_rounds: int = 0
    total_seconds: float = 0.0
    colors_used: int = 0
    valid: bool = False

    def to_dict(self) -> dict:
        """JSON form (driver.py:69-97); timing keys end in 'micros'."""
        return {
            "graph": self.graph_name,
            "num_nodes": self.num_nodes,
            "num_undirected_edges": self.num_undirected_edges,
            "config": {
                "mode": self.config.mode,
                "threshold_fraction": self.config.threshold_fraction,
                "workers": self.config.workers,
                "chunk_size": self.config.chunk_size,
            },
            "colors_used": self.colors_used,
            "valid": self.valid,
            "total_rounds": self.total_rounds,
            "total_micros": self.total_seconds * 1e6,
            "per_round": [
                {
                    "round": r.round,
                    "mode": r.mode_used,
                    "wl_in": r.worklist_size_in,
                    "wl_out": r.worklist_size_out,
                    "conflicts": r.conflicts,
                    "micros": r.wall_seconds * 1e6,
                }
                for r in self.per_round
            ],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True)

    def write_round_csv(self, stream: IO[str]) -> None:
        writer = csv.writer(stream)
        writer.writerow(["round", "mode", "wl_in", "wl_out", "conflicts", "micros"])
        for r in self.per_round:
            writer.writerow([r.round, r.mode_used, r.worklist_size_in, r.worklist_size_out,
                             r.conflicts, f"{r.wall_seconds * 1e6:.3f}"])

    def rows_table(self) -> str:
        header = f"{'round':>5}  {'mode':<5} {'wl_in':>9} {'wl_out':>9} {'conflicts':>9} {'micros':>12}"
        lines = [header]
        for r in self.per_round:
            lines.append(
                f"{r.round:>5}  {r.mode_used:<5} {r.worklist_size_in:>9} "
                f"{r.worklist_size_out:>9} {r.conflicts:>9} {r.wall_seconds * 1e6:>12.1f}"
            )
        return "\n".join(lines)


@dataclass
class DeviceSolve:
    """Raw result of one device solve (colors stay on the GPU)."""

    colors: torch.Tensor          # int64[n] on device
    records: np.ndarray           # int64[rounds, 6] (round, topo, wl_in, wl_out, conflicts, ns)
    rounds: int
    seconds: float                # CUDA-event time of hc_solve


class Solver:
    """Reusable device solve for one graph: workspace, output and record
    buffers are allocated once, so repeated solves (benchmarks) allocate
    nothing.  Thread/stream: uses the current torch CUDA stream."""

    def __init__(self, graph: DeviceCsr, max_rec: int | None = None):
        self.L = _lib.load()
        # the solver keeps the graph's tensors, not the DeviceCsr: color_graph
        # caches the solver on the DeviceCsr, and a graph -> solver -> graph
        # cycle kept a dropped graph's CSR and workspace on the GPU until the
        # cyclic GC ran (later calls then allocated afresh: e2e steps 370 ms
        # one time, 400+ the next)
        lf = graph.ensure_lower_first()
        self.g = SimpleNamespace(num_nodes=lf.num_nodes, num_edges=lf.num_edges, row_offsets=lf.row_offsets,
                                 col_indices=lf.col_indices, device=lf.device)
        dev = graph.device
        n = graph.num_nodes
        self.ws = _lib.workspace(self.L.hc_solve_workspace_bytes(n, graph.num_edges), dev)
        self.colors = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.max_rec = int(max_rec if max_rec is not None else max(1, min(n, 1 << 20)))
        self.rec = torch.empty((self.max_rec, _lib.REC_FIELDS), dtype=torch.int64, device=dev)
        self.start = torch.cuda.Event(enable_timing=True)
        self.stop = torch.cuda.Event(enable_timing=True)

    def _grow_records(self, rounds: int):
        self.max_rec = int(rounds)
        self.rec = torch.empty((self.max_rec, _lib.REC_FIELDS), dtype=torch.int64,
                               device=self.g.device)

    def run(self, mode: str, thr_count: int, *, fetch_records: bool = True, plain: bool = False) -> DeviceSolve:
        """plain=True: the bench-only Plain baseline (hc_solve_plain: unordered,
        atomically pushed worklists); same results."""
        g = self.g
        rounds = ctypes.c_int64(0)
        st = torch.cuda.current_stream()
        self.start.record(st)
        rc = (self.L.hc_solve_plain if plain else self.L.hc_solve)(
            g.row_offsets.data_ptr(), _lib.ptr(g.col_indices), g.num_nodes, g.num_edges,
            _lib.MODE_CODES[mode], int(thr_count), self.colors.data_ptr(), self.rec.data_ptr(),
            self.max_rec, ctypes.byref(rounds), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(st))
        self.stop.record(st)
        if rc == _lib.HC_ERR_RECORDS:  # more rounds than record slots: grow and redo
            self._grow_records(rounds.value)
            return self.run(mode, thr_count, fetch_records=fetch_records, plain=plain)
        _lib.check(rc)
        self.stop.synchronize()
        secs = self.start.elapsed_time(self.stop) / 1e3
        r = int(rounds.value)
        recs = self.rec[:r].cpu().numpy() if fetch_records else np.zeros((0, _lib.REC_FIELDS), np.int64)
        return DeviceSolve(self.colors[: g.num_nodes], recs, r, secs)


class PlannedSolver(Solver):
    """A solve that can be captured into a CUDA graph: the per-graph
    preprocessing runs once (hc_solve_plan_graph, one host sync) and every
    `launch` is stream-ordered work only (hc_solve_launch: state reset, the
    persistent solve kernel, the (rounds, flags) triple copied into the device
    tensor `info`).  `result` synchronises and reads the outcome."""

    def __init__(self, graph: DeviceCsr, max_rec: int | None = None):
        super().__init__(graph, max_rec)
        g = self.g
        self.plan = _lib.SolvePlan()
        self.info = torch.zeros(3, dtype=torch.int64, device=graph.device)
        _lib.check(self.L.hc_solve_plan_graph(
            g.row_offsets.data_ptr(), _lib.ptr(g.col_indices), g.num_nodes, g.num_edges,
            self.ws.data_ptr(), self.ws.numel(), ctypes.byref(self.plan), _lib.stream_handle()))

    def launch(self, mode: str, thr_count: int, stream: torch.cuda.Stream | None = None) -> None:
        g = self.g
        _lib.check(self.L.hc_solve_launch(
            ctypes.byref(self.plan), g.row_offsets.data_ptr(), _lib.ptr(g.col_indices), _lib.MODE_CODES[mode],
            int(thr_count), self.colors.data_ptr(), self.rec.data_ptr(), self.max_rec, self.info.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(stream)))

    def result(self) -> DeviceSolve:
        # the launch may have run on any stream (or as a replayed CUDA graph)
        torch.cuda.synchronize(self.g.device)
        rounds, flag, _ = (int(x) for x in self.info.cpu().tolist())
        if flag == 2:
            raise _lib.HcError(_lib.HC_ERR_STALLED, f"hc_solve_launch: no convergence after {rounds} rounds")
        if flag:
            raise _lib.HcError(_lib.HC_ERR_RECORDS, f"hc_solve_launch: {rounds} rounds exceed {self.max_rec} records")
        return DeviceSolve(self.colors[: self.g.num_nodes], self.rec[:rounds].cpu().numpy(), rounds, float("nan"))


def threshold_count(config: HybridConfig, num_nodes: int) -> int:
    """ceil(H * n) in host double arithmetic, exactly driver.py:138."""
    return math.ceil(config.threshold_fraction * num_nodes)


def _as_device(graph) -> DeviceCsr:
    if isinstance(graph, DeviceCsr):
        return graph
    if isinstance(graph, CsrGraph) or hasattr(graph, "row_offsets"):
        if not isinstance(graph, CsrGraph):  # a reference hybridcolor.CsrGraph
            graph = CsrGraph(graph.num_nodes, graph.num_edges, graph.row_offsets, graph.col_indices)
        return graph.to_device()
    raise TypeError(f"color_graph expects a CsrGraph or DeviceCsr, got {type(graph).__name__}")


def _check_kernels(kernels) -> None:
    if kernels is None:
        return
    from . import kernels as cuda_kernels

    if kernels is not cuda_kernels and getattr(kernels, "NAME", None) != cuda_kernels.NAME:
        raise ValueError(
            f"kernel backend {getattr(kernels, 'NAME', kernels)!r} not available (have: cuda)")


def color_graph(
    graph,
    config: HybridConfig | None = None,
    *,
    graph_name: str = "graph",
    kernels=None,
) -> tuple[np.ndarray, RunReport]:
    """Color the whole graph; returns (final colors int64[n], run report).

    driver.py:122-176: all nodes start uncolored with a full worklist; a round
    is topology-driven iff the worklist size strictly exceeds
    ceil(threshold_fraction * num_nodes) (hybrid), or as forced by `mode`.
    `graph` may be a host CsrGraph (uploaded, int64 -> int32 columns on the
    GPU) or a DeviceCsr.  `kernels` is accepted for signature parity and must
    be None or this package's `cuda` kernel module.
    """
    _check_kernels(kernels)
    if config is None:
        config = HybridConfig()
    dg = _as_device(graph)
    n = dg.num_nodes
    report = RunReport(graph_name, n, dg.num_undirected_edges, config)
    if n == 0:  # driver.py:145 never enters the loop
        report.valid = True
        return np.zeros(0, dtype=np.int64), report
    solver = dg.__dict__.get("_solver")
    if solver is None:  # one workspace per graph, reused by later calls (benchmarks)
        solver = dg.__dict__["_solver"] = Solver(dg)
    res = solver.run(config.mode, threshold_count(config, n))
    report.total_seconds = res.seconds
    for r in res.records:
        report.per_round.append(RoundRecord(
            round=int(r[0]), mode_used="topo" if r[1] else "data",
            worklist_size_in=int(r[2]), worklist_size_out=int(r[3]),
            conflicts=int(r[4]), wall_seconds=float(r[5]) * 1e-9))
    report.total_rounds = res.rounds
    report.colors_used = _colors_used_device(res.colors)
    report.valid = _verify_device(dg, res.colors) == 0
    # D2H into page-locked memory (straight DMA; torch caches the pinned block)
    host = torch.empty(res.colors.shape, dtype=torch.int64, pin_memory=True)
    host.copy_(res.colors, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    colors = host.numpy()
    return colors, report


def _colors_used_device(colors: torch.Tensor) -> int:
    n = int(colors.numel())
    acc = torch.zeros(2, dtype=torch.int64, device=colors.device)
    out = ctypes.c_int64(0)
    rc = _lib.load().hc_colors_used(_lib.ptr(colors), n, acc.data_ptr(), ctypes.byref(out),
                                    _lib.stream_handle())
    if rc == _lib.HC_ERR_UNCOLORED:
        raise ValueError("invalid coloring: uncolored node (color 0) present")  # driver.py:183-184
    _lib.check(rc)
    return int(out.value)


def _verify_device(dg: DeviceCsr, colors: torch.Tensor) -> int:
    acc = torch.zeros(1, dtype=torch.int64, device=colors.device)
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_verify(dg.row_offsets.data_ptr(), _lib.ptr(dg.col_indices), dg.num_nodes,
                                     _lib.ptr(colors), acc.data_ptr(), ctypes.byref(out),
                                     _lib.stream_handle()))
    return int(out.value)


def colors_used(colors) -> int:
    """Number of colors a finished run used (driver.py:179-185), on the GPU."""
    t = _to_device_i64(colors)
    if t.numel() == 0:
        return 0
    return _colors_used_device(t)


def verify_coloring(graph, colors) -> int:
    """Count invalid edges u<v with equal colors or colors[u]==0
    (driver.py:188-204), on the GPU."""
    n = graph.num_nodes
    if len(colors) != n:
        raise ValueError(f"colors array has length {len(colors)}, graph has {n} nodes")
    if graph.num_edges == 0:
        return 0
    dg = _as_device(graph)
    return _verify_device(dg, _to_device_i64(colors))


def _to_device_i64(colors) -> torch.Tensor:
    if isinstance(colors, torch.Tensor):
        t = colors
        if t.device.type != "cuda":
            t = t.to(_lib.device())
        return t.to(torch.int64).contiguous()
    arr = np.ascontiguousarray(np.asarray(colors), dtype=np.int64)
    return torch.from_numpy(arr).to(_lib.device())
