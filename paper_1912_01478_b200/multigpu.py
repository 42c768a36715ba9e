"""Device-resident multi-GPU hybrid IPGC over NVLink peer memory
(include/hcb.h hc_mg_*).

The reference has one process and one round loop (driver.py:122-176).  Here
the node range is cut into P contiguous, edge-balanced ranges; rank p owns
[lo_p, hi_p), holds only those CSR rows (a `CsrShard`: build_csr's rows
lo_p..hi_p-1 with global column ids, built on the rank's GPU by
hc_build_csr_rows) and runs ONE persistent kernel for the whole solve -- the
single-GPU solver (hcb_solve.cu) instantiated with the multi-GPU format:

  * every rank keeps a replica of the state words X[n] in its *shared region*
    (plus a mailbox); all ranks' regions are mapped into every rank
    (cudaIpc handles exchanged over torch.distributed, NVLink P2P mappings);
  * the word of an owned *boundary* node (a neighbour outside the range) is
    stored straight into every peer's replica by the thread that computes it
    -- the exchange is fused into assign / resolve, no pack / collective /
    unpack step;
  * the two grid barriers of a round are cross-GPU barriers (fence.sc.sys,
    then mailbox flags with st.release.sys / ld.acquire.sys); the end-of-round
    one also all-reduces (|W'|, conflicts), so every rank takes the identical
    hybrid decision (driver.py:147-152) and terminates in the same round.

No host round trip per round.  Round semantics read only the previous
snapshot (assign) and same-round tentatives (resolve) with id tie-breaks, so
colors, round count and every per-round record equal the single-GPU solve
(and the reference) for every partition.

`virtual_color_graph` runs P ranks in one process on one GPU (one stream and
a 1/P share of the SMs per rank, pointers instead of IPC mappings): the same
kernel, barrier and mirroring code, testable on a single B200.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .driver import HybridConfig, RoundRecord, RunReport, _colors_used_device, threshold_count
from .graph import DeviceCsr

MAX_WORLD = 8
IPC_HANDLE_BYTES = 64
HC_ERR_TIMEOUT = -8


def partition_bounds_device(row_offsets: torch.Tensor, world: int) -> list[tuple[int, int]]:
    """Edge-balanced contiguous ranges, identical to distributed.partition_bounds
    (cut p = first node whose row starts at or after m*p/P), computed on the
    device with one searchsorted."""
    n = int(row_offsets.numel()) - 1
    m = int(row_offsets[-1].item()) if n >= 0 else 0
    if m > 0 and world > 1:
        targets = torch.tensor([(m * p) // world for p in range(1, world)], dtype=torch.int64,
                               device=row_offsets.device)
        raw = torch.searchsorted(row_offsets, targets, side="left").tolist()
    else:
        raw = [(n * p) // world for p in range(1, world)]
    cuts = [0]
    for c in raw:
        cuts.append(min(max(int(c), cuts[-1]), n))
    cuts.append(n)
    return [(cuts[p], cuts[p + 1]) for p in range(world)]


@dataclass
class CsrShard:
    """Rows [lo, hi) of the graph's CSR on this rank's GPU (SURVEY.md §8(e):
    "each GPU holds its CSR rows"): row_offsets int64[hi-lo+1] (row r = node
    lo+r, starting at 0), col_indices int32 with GLOBAL node ids -- exactly
    rows lo..hi-1 of build_csr (graph.py:184-201).  num_nodes / max_degree /
    num_undirected_edges describe the whole graph (all-reduced over ranks)."""

    num_nodes: int
    lo: int
    hi: int
    row_offsets: torch.Tensor
    col_indices: torch.Tensor
    bounds: list
    max_degree: int = -1              # global (max over ranks); -1 until known
    num_undirected_edges: int = -1    # global; -1 until known

    @property
    def num_edges(self) -> int:
        """half-edges held by this shard"""
        return int(self.col_indices.numel())

    @property
    def device(self) -> torch.device:
        return self.row_offsets.device

    def local_max_degree(self) -> int:
        if self.hi == self.lo:
            return 0
        return int((self.row_offsets[1:] - self.row_offsets[:-1]).max().item())

    def nbytes(self) -> int:
        return self.row_offsets.numel() * 8 + self.col_indices.numel() * 4

    def to_host(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(row offsets, int64 column ids) in page-locked host memory -- the
        reference's CsrGraph layout of these rows (graph.py:49-67)."""
        ro = self.row_offsets.cpu().pin_memory()
        ci = self.col_indices.to(torch.int64).cpu().pin_memory()
        return ro, ci

    @classmethod
    def upload(cls, host: tuple[torch.Tensor, torch.Tensor], like: "CsrShard",
               dev: torch.device | None = None) -> "CsrShard":
        """Upload host rows (to_host) and narrow the column ids to int32 on the GPU."""
        dev = dev or like.device
        ro_h, ci_h = host
        ro = ro_h.to(dev, non_blocking=True)
        m = int(ci_h.numel())
        ci = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
        if m:
            ci64 = ci_h.to(dev, non_blocking=True)
            _lib.check(_lib.load().hc_narrow_i64_i32(ci64.data_ptr(), ci.data_ptr(), m, _lib.stream_handle()))
            del ci64
        return cls(like.num_nodes, like.lo, like.hi, ro, ci, like.bounds, like.max_degree,
                   like.num_undirected_edges)


def shard_of(graph: DeviceCsr, bounds: list[tuple[int, int]], rank: int) -> CsrShard:
    """Rank `rank`'s rows of a whole-graph DeviceCsr (virtual ranks on one GPU,
    tests): a rebased copy of the offsets and a view of the columns."""
    lo, hi = bounds[rank]
    ro = graph.row_offsets[lo : hi + 1]
    base = int(ro[0].item()) if hi >= lo else 0
    end = int(ro[-1].item())
    return CsrShard(graph.num_nodes, lo, hi, (ro - base).contiguous(), graph.col_indices[base:end], bounds,
                    max_degree=graph.max_degree, num_undirected_edges=graph.num_undirected_edges)


def edge_partition_bounds(d_edges: torch.Tensor, num_nodes: int, world: int) -> list[tuple[int, int]]:
    """Edge-balanced contiguous ranges cut on the pair list's half-edge
    counts (loops dropped, duplicates kept: hc_edge_degrees) -- every rank
    computes the same bounds from the same generated pairs before any shard
    exists (partition_bounds_device's rule on that prefix)."""
    L = _lib.load()
    n = int(num_nodes)
    m = int(d_edges.shape[0]) if d_edges.numel() else 0
    deg = torch.empty(max(n, 1), dtype=torch.int64, device=d_edges.device)
    _lib.check(L.hc_edge_degrees(_lib.ptr(d_edges), m, n, deg.data_ptr(), _lib.stream_handle()))
    ro = torch.zeros(n + 1, dtype=torch.int64, device=d_edges.device)
    if n:
        torch.cumsum(deg[:n], 0, out=ro[1:])
    return partition_bounds_device(ro, world), ro


def build_shard(d_edges: torch.Tensor, num_nodes: int, bounds: list[tuple[int, int]], rank: int,
                raw_offsets: torch.Tensor | None = None) -> CsrShard:
    """build_csr's rows [lo, hi) of the pair list `d_edges` (int64[m, 2] on this
    rank's GPU), global column ids, without building any other row
    (hc_build_csr_rows)."""
    L = _lib.load()
    dev = d_edges.device
    n = int(num_nodes)
    m = int(d_edges.shape[0]) if d_edges.numel() else 0
    lo, hi = bounds[rank]
    if raw_offsets is None:
        _, raw_offsets = edge_partition_bounds(d_edges, n, len(bounds))
    cap = int(raw_offsets[hi].item() - raw_offsets[lo].item())  # directed entries before dedupe
    ro = torch.zeros(hi - lo + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    ws = _lib.workspace(L.hc_build_csr_rows_workspace_bytes(n, lo, hi, cap), dev)
    md = ctypes.c_int64(0)
    _lib.check(L.hc_build_csr_rows(_lib.ptr(d_edges), m, n, lo, hi, cap, ro.data_ptr(), ci.data_ptr(),
                                   ctypes.byref(md), ws.data_ptr(), ws.numel(), _lib.stream_handle()))
    del ws
    k = int(md.value)
    return CsrShard(n, lo, hi, ro, ci[:k].clone() if k else ci[:0], bounds)


class RankSolver:
    """One rank's reusable solve state for the owned range [lo, hi):
    workspace, owned colors and the (global) per-round records."""

    def __init__(self, shard: CsrShard, rank: int, world: int,
                 shared_ptrs: list[int], *, max_rec: int | None = None, ctas: int = 0,
                 timeout_ms: int = 60000):
        if not 1 <= world <= MAX_WORLD:
            raise ValueError(f"world size {world} not in [1, {MAX_WORLD}]")
        if shard.max_degree < 0:
            raise ValueError("shard.max_degree (the global max over ranks) must be set")
        self.L = _lib.load()
        self.g = shard
        bounds = shard.bounds
        self.lo, self.hi, self.rank, self.world = int(shard.lo), int(shard.hi), int(rank), int(world)
        assert (self.lo, self.hi) == tuple(bounds[rank])
        self.cuts = (ctypes.c_int64 * (world + 1))(*([b[0] for b in bounds] + [bounds[-1][1]]))
        dev = shard.device
        n = shard.num_nodes
        self.ws = _lib.workspace(self.L.hc_mg_workspace_bytes(n, shard.num_edges, self.lo, self.hi), dev)
        self.colors = torch.empty(max(self.hi - self.lo, 1), dtype=torch.int64, device=dev)
        self.max_rec = int(max_rec if max_rec is not None else max(1, min(n, 1 << 20)))
        self.rec = torch.empty((self.max_rec, _lib.REC_FIELDS), dtype=torch.int64, device=dev)
        self.shared = (ctypes.c_void_p * world)(*[ctypes.c_void_p(p) for p in shared_ptrs])
        self.ctas = int(ctas)
        self.timeout_ms = int(timeout_ms)

    def launch(self, mode: str, thr_count: int, stream: torch.cuda.Stream | None = None) -> None:
        self.prepare(mode, thr_count, stream)
        _lib.check(self.L.hc_mg_launch(self.ws.data_ptr(), _lib.stream_handle(stream)))

    def prepare(self, mode: str, thr_count: int, stream: torch.cuda.Stream | None = None) -> None:
        """Preprocessing of the owned range (synchronous); hc_mg_launch starts the solve."""
        g = self.g
        _lib.check(self.L.hc_mg_prepare(
            g.row_offsets.data_ptr(), _lib.ptr(g.col_indices), g.num_nodes, g.num_edges,
            ctypes.cast(self.cuts, ctypes.c_void_p), self.rank, self.world, ctypes.cast(self.shared, ctypes.c_void_p),
            _lib.MODE_CODES[mode], int(thr_count),
            self.colors.data_ptr(), self.rec.data_ptr(), self.max_rec, self.ctas, self.timeout_ms,
            int(g.max_degree), self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(stream)))

    def wait(self, stream: torch.cuda.Stream | None = None) -> int:
        rounds = ctypes.c_int64(0)
        _lib.check(self.L.hc_mg_wait(self.ws.data_ptr(), ctypes.byref(rounds), _lib.stream_handle(stream)))
        return int(rounds.value)

    def records(self, rounds: int) -> np.ndarray:
        return self.rec[:rounds].cpu().numpy()


def _report(graph_name, num_nodes, num_undirected_edges, config, recs, rounds, seconds) -> RunReport:
    report = RunReport(graph_name, num_nodes, num_undirected_edges, config)
    for r in recs:
        report.per_round.append(RoundRecord(
            round=int(r[0]), mode_used="topo" if r[1] else "data", worklist_size_in=int(r[2]),
            worklist_size_out=int(r[3]), conflicts=int(r[4]), wall_seconds=float(r[5]) * 1e-9))
    report.total_rounds = rounds
    report.total_seconds = seconds
    return report


@dataclass
class MgResult:
    colors: np.ndarray          # int64[n], the whole coloring
    report: RunReport           # global per-round records (rank 0's copy)
    bounds: list                # owned ranges
    rank_records: list          # per-rank record arrays (all equal)
    seconds: float


# --------------------------------------------------------------------------
# P ranks in one process on one GPU (tests)
# --------------------------------------------------------------------------
class VirtualMesh:
    """`world` ranks sharing the current GPU: one shared region, stream and
    1/world of the resident CTAs per rank."""

    def __init__(self, graph: DeviceCsr, world: int, *, timeout_ms: int = 20000,
                 ctas_per_rank: int | None = None):
        L = _lib.load()
        dev = graph.device
        n = graph.num_nodes
        self.world = world
        self.bounds = partition_bounds_device(graph.row_offsets, world)
        sms, per_sm = ctypes.c_int(0), ctypes.c_int(0)
        _lib.check(L.hc_device_info(ctypes.byref(sms), ctypes.byref(per_sm)))
        cap = sms.value * per_sm.value
        ctas = ctas_per_rank if ctas_per_rank is not None else max(1, cap // world)
        if ctas * world > cap:
            raise ValueError(f"{world} ranks x {ctas} CTAs exceed the {cap} resident CTAs")
        self.regions = [torch.zeros(L.hc_mg_shared_bytes(n), dtype=torch.uint8, device=dev)
                        for _ in range(world)]
        ptrs = [r.data_ptr() for r in self.regions]
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
        graph = graph.ensure_lower_first()
        self.shards = [shard_of(graph, self.bounds, p) for p in range(world)]
        self.ranks = [RankSolver(self.shards[p], p, world, ptrs, ctas=ctas, timeout_ms=timeout_ms)
                      for p in range(world)]
        torch.cuda.synchronize()

    def solve(self, mode: str, thr_count: int):
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        start = torch.cuda.Event(enable_timing=True)
        start.record(cur)
        for s in self.streams:
            s.wait_event(start)
        # preprocessing of every rank first: no rank's preprocessing kernels
        # may queue behind another rank's persistent kernel on the shared GPU
        for rk, s in zip(self.ranks, self.streams):
            rk.prepare(mode, thr_count, s)
        for rk, s in zip(self.ranks, self.streams):
            _lib.check(rk.L.hc_mg_launch(rk.ws.data_ptr(), _lib.stream_handle(s)))
        rounds = [rk.wait(s) for rk, s in zip(self.ranks, self.streams)]
        stop = torch.cuda.Event(enable_timing=True)
        for s in self.streams:
            cur.wait_stream(s)
        stop.record(cur)
        stop.synchronize()
        return rounds, start.elapsed_time(stop) / 1e3


def virtual_color_graph(graph: DeviceCsr, config: HybridConfig | None = None, world: int = 2, *,
                        graph_name: str = "graph", timeout_ms: int = 20000,
                        mesh: VirtualMesh | None = None) -> MgResult:
    """The multi-GPU solve with `world` ranks sharing the current GPU."""
    config = config or HybridConfig()
    mesh = mesh or VirtualMesh(graph, world, timeout_ms=timeout_ms)
    thr = threshold_count(config, graph.num_nodes)
    rounds, secs = mesh.solve(config.mode, thr)
    if len(set(rounds)) != 1:
        raise RuntimeError(f"ranks disagree on the round count: {rounds}")
    recs = [rk.records(rounds[0]) for rk in mesh.ranks]
    dcolors = torch.cat([rk.colors[: rk.hi - rk.lo] for rk in mesh.ranks])
    rep = _report(graph_name, graph.num_nodes, graph.num_undirected_edges, config, recs[0], rounds[0], secs)
    rep.valid = sum(_verify_shard(sh, dcolors) for sh in mesh.shards) == 0
    rep.colors_used = _colors_used_device(dcolors) if rep.valid else int(dcolors.max().item())
    return MgResult(dcolors.cpu().numpy(), rep, mesh.bounds, recs, secs)


def _verify_shard(shard: CsrShard, colors: torch.Tensor) -> int:
    """verify_coloring (driver.py:188-204) over the shard's rows, colors global."""
    acc = torch.zeros(1, dtype=torch.int64, device=colors.device)
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_verify_rows(shard.row_offsets.data_ptr(), _lib.ptr(shard.col_indices), shard.lo,
                                          shard.hi, _lib.ptr(colors), acc.data_ptr(), ctypes.byref(out),
                                          _lib.stream_handle()))
    return int(out.value)


# --------------------------------------------------------------------------
# one process per GPU (torch.distributed group; NVLink peer mappings)
# --------------------------------------------------------------------------
class PeerGroup:
    """This rank's shared region plus every peer's, mapped into this process
    through cudaIpc handles exchanged over the torch.distributed group."""

    def __init__(self, num_nodes: int, group=None):
        import torch.distributed as dist

        self.L = L = _lib.load()
        dev = _lib.device()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > MAX_WORLD:
            raise ValueError(f"world size {self.world} > {MAX_WORLD}")
        # own cudaMalloc allocation: exportable whatever torch's allocator does
        reg = ctypes.c_void_p(0)
        _lib.check(L.hc_mg_alloc_shared(L.hc_mg_shared_bytes(num_nodes), ctypes.byref(reg)))
        self.region_ptr = int(reg.value)
        handle = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        off = ctypes.c_int64(0)
        _lib.check(L.hc_mg_ipc_export(self.region_ptr, handle, ctypes.byref(off)))
        mine = (bytes(handle.raw), int(off.value))
        allinfo = [None] * self.world
        dist.all_gather_object(allinfo, mine, group=group)
        self.ptrs, self._opened = [], []
        err = None
        try:
            for q, (h, o) in enumerate(allinfo):
                if q == self.rank:
                    self.ptrs.append(self.region_ptr)
                    continue
                p = ctypes.c_void_p(0)
                _lib.check(L.hc_mg_ipc_import(ctypes.create_string_buffer(h, IPC_HANDLE_BYTES), o,
                                              ctypes.byref(p)))
                self.ptrs.append(int(p.value))
                self._opened.append((int(p.value), o))
        except Exception as exc:  # every rank must learn that the mapping failed somewhere
            err = exc
        flags = [None] * self.world
        dist.all_gather_object(flags, err is None, group=group)
        if not all(flags):
            for p, o in self._opened:
                L.hc_mg_ipc_close(ctypes.c_void_p(p), o)
            self._opened = []
            dist.barrier(group=group)
            L.hc_mg_free_shared(ctypes.c_void_p(self.region_ptr))
            self.region_ptr = 0
            raise RuntimeError(f"peer mapping failed on ranks {[q for q, f in enumerate(flags) if not f]}: "
                               f"{err!r}")

    def close(self):
        import torch.distributed as dist

        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # no peer still writes into a mapping
        for p, o in self._opened:
            _lib.check(self.L.hc_mg_ipc_close(ctypes.c_void_p(p), o))
        self._opened = []
        dist.barrier(group=self.group)  # every peer unmapped this rank's region
        if self.region_ptr:
            _lib.check(self.L.hc_mg_free_shared(ctypes.c_void_p(self.region_ptr)))
            self.region_ptr = 0


class MgSolver:
    """Reusable per-rank multi-GPU solve of one graph.  Every rank holds only
    its shard (CsrShard); a whole DeviceCsr is accepted too (each rank then
    keeps only a view of its own rows: tests, single-box runs)."""

    def __init__(self, graph: CsrShard | DeviceCsr, group=None, *, timeout_ms: int = 60000):
        import torch.distributed as dist

        self.group = group
        if isinstance(graph, DeviceCsr):
            world = dist.get_world_size(group)
            graph = graph.ensure_lower_first()
            graph = shard_of(graph, partition_bounds_device(graph.row_offsets, world), dist.get_rank(group))
        shard = graph
        # whole-graph facts every rank must agree on (state-word width, report)
        if shard.max_degree < 0 or shard.num_undirected_edges < 0:
            cdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else shard.device
            t = torch.tensor([shard.local_max_degree()], dtype=torch.int64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            e = torch.tensor([shard.num_edges], dtype=torch.int64, device=cdev)
            dist.all_reduce(e, op=dist.ReduceOp.SUM, group=group)
            shard.max_degree, shard.num_undirected_edges = int(t.item()), int(e.item()) // 2
        self.shard = shard
        self.peers = PeerGroup(shard.num_nodes, group)
        self.world, self.rank = self.peers.world, self.peers.rank
        if len(shard.bounds) != self.world:
            raise ValueError(f"shard cut for {len(shard.bounds)} ranks, group has {self.world}")
        self.bounds = shard.bounds
        self.rs = RankSolver(shard, self.rank, self.world, self.peers.ptrs, timeout_ms=timeout_ms)
        self.mx = max(h - l for l, h in self.bounds)
        self.start = torch.cuda.Event(enable_timing=True)
        self.stop = torch.cuda.Event(enable_timing=True)

    @property
    def num_nodes(self) -> int:
        return self.shard.num_nodes

    def replace_shard(self, shard: CsrShard) -> None:
        """Solve a freshly uploaded copy of the same rows next time (e2e bench)."""
        shard.max_degree, shard.num_undirected_edges = self.shard.max_degree, self.shard.num_undirected_edges
        self.shard = self.rs.g = shard

    def run(self, mode: str, thr_count: int) -> tuple[int, float]:
        st = torch.cuda.current_stream()
        self.start.record(st)
        self.rs.launch(mode, thr_count, st)
        self.stop.record(st)
        rounds = self.rs.wait(st)
        return rounds, self.start.elapsed_time(self.stop) / 1e3

    def gather_colors(self) -> torch.Tensor:
        import torch.distributed as dist

        rs = self.rs
        # gloo (tests: several processes on one GPU) gathers host tensors
        dev = torch.device("cpu") if dist.get_backend(self.group) == "gloo" else rs.colors.device
        buf = torch.zeros(max(self.mx, 1), dtype=torch.int64, device=dev)
        buf[: rs.hi - rs.lo] = rs.colors[: rs.hi - rs.lo].to(dev)
        out = torch.empty(self.world * buf.numel(), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        out = out.view(self.world, -1)
        return torch.cat([out[p, : hi - lo] for p, (lo, hi) in enumerate(self.bounds)])

    def verify(self, colors: torch.Tensor) -> int:
        """Invalid edges of the whole coloring (driver.py:188-204): each rank
        checks its rows, summed over the group."""
        import torch.distributed as dist

        bad = _verify_shard(self.shard, colors.to(self.shard.device))
        cdev = torch.device("cpu") if dist.get_backend(self.group) == "gloo" else self.shard.device
        t = torch.tensor([bad], dtype=torch.int64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def close(self):
        self.peers.close()


def mg_color_graph(graph: CsrShard | DeviceCsr, config: HybridConfig | None = None, *, group=None,
                   graph_name: str = "graph", solver: MgSolver | None = None) -> MgResult:
    """Partitioned solve of the whole graph, one process per GPU.  Returns the
    whole coloring and the global RunReport (valid / colors_used included,
    driver.py:170-176) on every rank."""
    config = config or HybridConfig()
    own = solver is None
    solver = solver or MgSolver(graph, group)
    try:
        n = solver.num_nodes
        rounds, secs = solver.run(config.mode, threshold_count(config, n))
        recs = solver.rs.records(rounds)
        dcolors = solver.gather_colors()
        bad = solver.verify(dcolors)
    finally:
        if own:
            solver.close()
    rep = _report(graph_name, n, solver.shard.num_undirected_edges, config, recs, rounds, secs)
    rep.valid = bad == 0
    colors = dcolors.cpu().numpy()
    if colors.size and colors.min() < 1:
        raise ValueError("invalid coloring: uncolored node (color 0) present")  # driver.py:183-184
    rep.colors_used = int(colors.max()) if colors.size else 0
    return MgResult(colors, rep, solver.bounds, [recs], secs)
