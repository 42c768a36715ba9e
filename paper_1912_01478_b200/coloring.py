"""Per-round IPGC operations on device state (pkg/src/hybridcolor/coloring.py).

`ColorState` (coloring.py:37-52) keeps the reference's double-buffered int64
colors plus stamps, as CUDA tensors.  `data_driven_iteration` (113-142) and
`topology_driven_iteration` (145-176) run one round through the `cuda`
kernel module with the reference's commits (105-110) and worklist swap.
This is the per-round path (golden round traces, plugin parity); the solve
itself (`color_graph`) fuses all rounds into one device-resident kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import torch

from . import _lib
from . import kernels as cuda_kernels
from .graph import CsrGraph, DeviceCsr
from .worklist import Worklist


@dataclass
class ColorState:
    colors_read: torch.Tensor
    colors_write: torch.Tensor
    active_stamp: torch.Tensor

    @classmethod
    def fresh(cls, num_nodes: int) -> "ColorState":
        dev = _lib.device()
        z = lambda: torch.zeros(num_nodes, dtype=torch.int64, device=dev)  # noqa: E731
        return cls(colors_read=z(), colors_write=z(), active_stamp=z())


@dataclass
class RoundOutcome:
    colored_permanently: int
    pushed_back: int
    conflicts_detected: int


def _device_graph(graph) -> DeviceCsr:
    if isinstance(graph, CsrGraph):
        # a host CsrGraph is frozen (graph.py:60-63): upload it once and keep
        # the device copy with it, so per-round calls do no H2D traffic
        dg = graph.__dict__.get("_device_csr")
        if dg is None:
            dg = graph.to_device()
            dg.host = None  # no host <-> device cycle: the copy goes with the host graph
            graph.__dict__["_device_csr"] = dg
        graph = dg
    if not isinstance(graph, DeviceCsr):
        raise TypeError("expected CsrGraph or DeviceCsr")
    return graph


def _graph_arrays(graph):
    graph = _device_graph(graph)
    return graph.row_offsets, graph.col_indices_i64, graph.max_degree


def mex_positive(forbidden: Iterable[int]) -> int:
    """Smallest integer c >= 1 not in `forbidden` (coloring.py:64-70).

    The reference's scalar helper for a host-side set (its kernels, and the
    device assign here, compute the same mex over a node's committed
    neighbour colors)."""
    taken = set(forbidden)
    c = 1
    while c in taken:
        c += 1
    return c


def _node_tensor(node: int) -> torch.Tensor:
    return torch.tensor([int(node)], dtype=torch.int64, device=_lib.device())


def assign_color(graph, state: ColorState, node: int, round_no: int) -> int:
    """Speculative single-node assignment against the read snapshot
    (coloring.py:73-85): the device assign kernel over a one-node list."""
    assert int(state.colors_read[node]) == 0, f"assign_color on inactive node {node}"
    ro, ci, maxdeg = _graph_arrays(graph)
    cuda_kernels.assign_from_list(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                                  _node_tensor(node), round_no, maxdeg, 1, 1)
    return int(state.colors_write[node])


def resolve_conflicts(graph, state: ColorState, node: int, round_no: int, wl: Worklist) -> bool:
    """Uncolor `node` if a lower-id neighbour took the same color this round
    (coloring.py:88-102); a loser gets colors_write = 0 and is pushed onto
    `wl`.  Returns True iff the node lost."""
    ro, ci, _ = _graph_arrays(graph)
    lost = cuda_kernels.resolve_from_list(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                                          _node_tensor(node), round_no, wl.next_storage, wl.cursor, 1, 1) > 0
    if lost and wl.next_count > wl.capacity:  # the kernel dropped the push (pos >= cap, _kernels.pyx:117)
        wl.cursor.fill_(wl.capacity)          # worklist.push raises with the cursor unchanged
        raise RuntimeError("worklist overflow: more pushes than capacity "
                           "(at-most-once-per-iteration contract broken)")
    return lost


def _kmod(kernels):
    if kernels is not None and kernels is not cuda_kernels:
        raise ValueError("only the cuda kernel module is available")
    return cuda_kernels


def data_driven_iteration(graph, state: ColorState, wl: Worklist, round_no: int, *,
                          workers: int = 1, chunk_size: int = 1024, kernels=None) -> RoundOutcome:
    """coloring.py:113-142"""
    k = _kmod(kernels)
    ro, ci, maxdeg = _graph_arrays(graph)
    nodes = wl.current
    k.assign_from_list(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                       nodes, round_no, maxdeg, workers, chunk_size)
    k.commit_list(state.colors_read, state.colors_write, nodes)
    conflicts = k.resolve_from_list(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                                    nodes, round_no, wl.next_storage, wl.cursor, workers, chunk_size)
    k.commit_list(state.colors_read, state.colors_write, nodes)
    n_in = int(nodes.numel())
    pushed = wl.swap_and_sort()
    return RoundOutcome(n_in - pushed, pushed, int(conflicts))


def topology_driven_iteration(graph, state: ColorState, wl: Worklist, round_no: int, *,
                              workers: int = 1, chunk_size: int = 1024, kernels=None) -> RoundOutcome:
    """coloring.py:145-176"""
    k = _kmod(kernels)
    ro, ci, maxdeg = _graph_arrays(graph)
    processed = k.assign_sweep(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                               round_no, maxdeg, workers, chunk_size)
    k.commit_stamped(state.colors_read, state.colors_write, state.active_stamp, round_no)
    conflicts = k.resolve_sweep(ro, ci, state.colors_read, state.colors_write, state.active_stamp,
                                round_no, wl.next_storage, wl.cursor, workers, chunk_size)
    k.commit_stamped(state.colors_read, state.colors_write, state.active_stamp, round_no)
    pushed = wl.swap_and_sort()
    return RoundOutcome(int(processed) - pushed, pushed, int(conflicts))
