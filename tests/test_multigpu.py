"""Multi-process tests of the 1D-partitioned solve.

CPU (gloo, world_size 2 and 3): the distributed driver with the CPU stand-in
ops must reproduce the reference's colors and per-round records exactly.
GPU (gloo, 2 ranks sharing cuda:0): the same with the device kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import MODES
from oracle import oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graphs():
    rng = np.random.default_rng(7)
    out = []
    for n, m in ((40, 90), (120, 600), (300, 900)):
        ro, ci = O.build_csr(n, rng.integers(0, n, (m, 2)))
        out.append((ro, ci))
    ro, ci = O.build_csr(1 << 10, O.gen_rmat(10, 16, 3))
    out.append((ro, ci))
    ro, ci = O.build_csr(30 * 20, O.gen_grid(30, 20))
    out.append((ro, ci))
    return out


def _worker(rank, world, port, use_gpu, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1912_01478_b200 as hc
        from paper_1912_01478_b200.distributed import dist_color_graph
        from dist_cpu_ops import CpuOps

        results = []
        for ro, ci in _graphs():
            n = len(ro) - 1
            for mode in MODES:
                cfg = hc.HybridConfig(mode=mode)
                if use_gpu:
                    dev = torch.device("cuda", 0)
                    rot = torch.from_numpy(ro).to(dev)
                    cit = torch.from_numpy(ci.astype(np.int32)).to(dev)
                    res = dist_color_graph(rot, cit, n, cfg, host_row_offsets=ro)
                else:
                    res = dist_color_graph(torch.from_numpy(ro), torch.from_numpy(ci.astype(np.int32)), n, cfg,
                                           ops=CpuOps(ro, ci, n), host_row_offsets=ro)
                rec = np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out,
                                 r.conflicts] for r in res.report.per_round], dtype=np.int64).reshape(-1, 4)
                results.append((res.colors, rec))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def _run(world, use_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, use_gpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for ro, ci in _graphs():
        for mode in MODES:
            want.append(O.color(ro, ci, mode))
    for rank in range(world):
        assert len(out[rank]) == len(want)
        for (colors, rec), (wc, wr) in zip(out[rank], want):
            assert np.array_equal(colors, wc)
            assert np.array_equal(rec, wr)


def test_partition_bounds_edge_balanced():
    from paper_1912_01478_b200.distributed import partition_bounds

    ro, _ = O.build_csr(1 << 10, O.gen_rmat(10, 16, 3))
    for world in (1, 2, 3, 8):
        b = partition_bounds(ro, world)
        assert b[0][0] == 0 and b[-1][1] == len(ro) - 1
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        edges = [ro[hi] - ro[lo] for lo, hi in b]
        assert max(edges) - min(edges) <= max(np.diff(ro)) + ro[-1] // world // 10 + 1
    assert partition_bounds(np.zeros(5, np.int64), 2) == [(0, 2), (2, 4)]


def test_partition_bounds_device_form_matches_host():
    """multigpu.partition_bounds_device (searchsorted on the row-offset tensor,
    used by the peer-memory solve) == distributed.partition_bounds, on CPU
    tensors here."""
    from paper_1912_01478_b200.distributed import partition_bounds
    from paper_1912_01478_b200.multigpu import partition_bounds_device

    rng = np.random.default_rng(4)
    graphs = [O.build_csr(1 << 10, O.gen_rmat(10, 16, 3))[0], O.build_csr(500, rng.integers(0, 500, (3000, 2)))[0],
              np.zeros(8, np.int64), O.build_csr(30 * 20, O.gen_grid(30, 20))[0]]
    for ro in graphs:
        for world in (1, 2, 3, 5, 8):
            assert partition_bounds_device(torch.from_numpy(ro), world) == partition_bounds(ro, world)


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_solve_gloo_cpu(world):
    _run(world, use_gpu=False)


@pytest.mark.gpu
def test_partitioned_solve_device_kernels_two_ranks():
    _run(2, use_gpu=True)
