"""Device-resident multi-GPU solve over peer memory (hc_mg_*).

One B200 is available per test box, so the P ranks share it:
  * virtual ranks -- one process, P streams, P persistent kernels each on a
    1/P share of the SMs, the shared regions as plain device pointers.  Same
    kernel, mirrored stores, cross-GPU barrier + mailbox all-reduce as on P
    GPUs;
  * two processes on cuda:0 -- the cudaIpc export / import path that
    one-process-per-GPU uses (kernels time-slice between the contexts).
Everything must equal the single-GPU solve and the reference goldens
bit-for-bit: colors, round count and every per-round (mode, wl_in, wl_out,
conflicts).
"""

import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import MODES, THRESHOLDS
from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_1912_01478_b200 as hc  # noqa: E402
from paper_1912_01478_b200 import _lib  # noqa: E402
from paper_1912_01478_b200 import graph as G  # noqa: E402
from paper_1912_01478_b200.distributed import partition_bounds  # noqa: E402
from paper_1912_01478_b200.multigpu import (VirtualMesh, partition_bounds_device,  # noqa: E402
                                            virtual_color_graph)


def _recs4(report):
    return np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                     for r in report.per_round], dtype=np.int64).reshape(-1, 4)


def _dev(ro, ci):
    return hc.CsrGraph(len(ro) - 1, len(ci), ro, ci).to_device()


def _check(dg, world, mode, thr, want_colors=None, want_recs=None):
    cfg = hc.HybridConfig(mode=mode, threshold_fraction=thr)
    if want_colors is None:
        want_colors, rep1 = hc.color_graph(dg, cfg)
        want_recs = _recs4(rep1)
    res = virtual_color_graph(dg, cfg, world)
    assert np.array_equal(res.colors, want_colors), (world, mode, thr)
    assert np.array_equal(_recs4(res.report), want_recs), (world, mode, thr)
    for r in res.rank_records[1:]:  # every rank holds the same global records
        assert np.array_equal(r[:, :5], res.rank_records[0][:, :5])
    return res


def test_partition_bounds_device_matches_host():
    for n, m in ((50, 300), (1000, 9000), (7, 0)):
        ro, _ = O.build_csr(n, np.random.default_rng(n).integers(0, n, (m, 2))) if m else \
            (np.zeros(n + 1, np.int64), None)
        for w in (1, 2, 3, 4, 8):
            assert partition_bounds_device(torch.from_numpy(ro).cuda(), w) == partition_bounds(ro, w)


def test_virtual_ranks_match_reference_corpus(corpus):
    """A slice of the reference's seeded corpora, P = 2 and 3 ranks, every
    mode, two thresholds: colors + records equal the reference goldens."""
    for i, g in enumerate(corpus[::7]):
        if g.n < 2:
            continue
        dg = _dev(g.ro, g.ci)
        world = 2 + (i % 2)
        for mode in MODES:
            for thr in (THRESHOLDS[0], THRESHOLDS[2]):
                _check(dg, world, mode, thr, g.colors, g.records[(mode, thr)])


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_virtual_ranks_synthetic(world):
    graphs = [
        G.build_csr_device(G.gen_rmat_edges(12, 16, 1), 1 << 12),      # hubs, skew
        G.build_csr_device(G.gen_er_edges(5000, 5000 * 16, 3), 5000),   # uniform
        G.grid_graph(64, 48),                                            # delta columns
    ]
    for dg in graphs:
        for mode in MODES:
            _check(dg, world, mode, 0.6)


def test_virtual_ranks_hub_graph_and_formats():
    """32-bit state words (max degree > 16384), int64 offsets, and the
    absolute-column format, each forced, on a graph with a split-hub regime."""
    rng = np.random.default_rng(5)
    n = 40000
    hub = np.column_stack([np.zeros(20000, np.int64), rng.integers(1, n, 20000)])
    rest = rng.integers(0, n, (60000, 2))
    ro, ci = O.build_csr(n, np.vstack([hub, rest]))
    dg = _dev(ro, ci)
    want, rep = hc.color_graph(dg)
    try:
        for fmt in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)):
            _lib.load().hc_solve_set_formats(*fmt)
            res = virtual_color_graph(dg, hc.HybridConfig(), 3)
            assert np.array_equal(res.colors, want), fmt
            assert np.array_equal(_recs4(res.report), _recs4(rep)), fmt
    finally:
        _lib.load().hc_solve_set_formats(0, 0, 0)


@pytest.mark.parametrize("exchange", [1, 2])
def test_virtual_ranks_forced_exchange_modes(exchange):
    """Mirrored stores only (1) and zone copies only (2), each alone, must
    reproduce the single-GPU solve (auto mode mixes them per round)."""
    L = _lib.load()
    L.hc_mg_set_exchange(exchange)
    try:
        graphs = [G.build_csr_device(G.gen_rmat_edges(11, 16, 5), 1 << 11), G.grid_graph(70, 50),
                  G.build_csr_device(G.gen_er_edges(3000, 3000 * 12, 8), 3000)]
        for dg in graphs:
            for world in (2, 3, 5):
                for mode in MODES:
                    _check(dg, world, mode, 0.6)
    finally:
        L.hc_mg_set_exchange(0)


def test_virtual_ranks_repeated_solves_and_empty_ranges():
    # barrier epochs continue across solves on the same mesh
    dg = G.build_csr_device(G.gen_rmat_edges(10, 16, 4), 1 << 10)
    want, rep = hc.color_graph(dg)
    mesh = VirtualMesh(dg, 3)
    for mode in ("hybrid", "data", "topo", "hybrid"):
        res = virtual_color_graph(dg, hc.HybridConfig(mode=mode), 3, mesh=mesh)
        w, r = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert np.array_equal(res.colors, w) and np.array_equal(_recs4(res.report), _recs4(r))
    # more ranks than nodes with edges: some ranks own nothing
    k3 = _dev(np.array([0, 2, 4, 6]), np.array([1, 2, 0, 2, 0, 1]))
    res = virtual_color_graph(k3, hc.HybridConfig(), 4)
    assert res.colors.tolist() == [1, 2, 3] and res.report.total_rounds == 3


def test_virtual_ranks_grid_closed_form():
    r, c = 256, 200
    res = virtual_color_graph(G.grid_graph(r, c), hc.HybridConfig(), 4)
    i, j = np.divmod(np.arange(r * c), c)
    assert np.array_equal(res.colors, 1 + (i + j) % 2)
    assert res.report.total_rounds == (r + c + 1) // 2


# ---------------------------------------------------------------- two processes
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1912_01478_b200.multigpu import MgSolver, mg_color_graph

        dg = G.build_csr_device(G.gen_rmat_edges(8, 8, 2), 1 << 8)
        solver = MgSolver(dg, timeout_ms=60000)
        out = []
        for mode in ("hybrid", "data"):
            res = mg_color_graph(dg, hc.HybridConfig(mode=mode), solver=solver)
            out.append((mode, res.colors, _recs4(res.report)))
        solver.close()
        q.put((rank, out, None))
    except Exception as exc:  # reported to the parent
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_share_one_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, out, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        got[rank] = out
    for p in procs:
        p.join(timeout=60)
    dg = G.build_csr_device(G.gen_rmat_edges(8, 8, 2), 1 << 8)
    for mode, colors, recs in got[0]:
        want, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert np.array_equal(colors, want) and np.array_equal(recs, _recs4(rep)), mode
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


# ---------------------------------------------------------------- per-rank shards
def test_shard_build_equals_build_csr_rows():
    """hc_build_csr_rows: rank p's shard == rows [lo_p, hi_p) of build_csr
    (graph.py:184-201), global column ids; the shards partition the half-edges
    (per-rank CSR bytes ~ m_dir / P on an edge-balanced cut)."""
    from paper_1912_01478_b200.multigpu import build_shard, edge_partition_bounds

    for edges, n in ((G.gen_rmat_edges(14, 16, 3), 1 << 14), (G.gen_er_edges(5000, 40000, 9), 5000),
                     (G.gen_grid_edges(60, 70), 4200)):
        full = G.build_csr_device(edges, n)
        ro, ci = full.row_offsets.cpu().numpy(), full.col_indices.cpu().numpy()
        for world in (1, 2, 3, 8):
            bounds, raw = edge_partition_bounds(edges, n, world)
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
            total = 0
            for p in range(world):
                sh = build_shard(edges, n, bounds, p, raw)
                lo, hi = bounds[p]
                want_ro = ro[lo:hi + 1] - ro[lo]
                assert np.array_equal(sh.row_offsets.cpu().numpy(), want_ro), (n, world, p)
                assert np.array_equal(sh.col_indices.cpu().numpy(), ci[ro[lo]:ro[hi]]), (n, world, p)
                total += sh.num_edges
                if world > 1 and n > 4000:  # edge-balanced: no rank holds much more than its share
                    assert sh.num_edges <= 1.25 * full.num_edges / world + 64, (n, world, p, sh.num_edges)
            assert total == full.num_edges


def _ipc_shard_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1912_01478_b200.multigpu import MgSolver, build_shard, edge_partition_bounds, mg_color_graph

        n = 1 << 10
        edges = G.gen_rmat_edges(10, 8, 5)
        bounds, raw = edge_partition_bounds(edges, n, world)
        shard = build_shard(edges, n, bounds, rank, raw)
        del edges, raw
        solver = MgSolver(shard, timeout_ms=60000)
        out = []
        for mode in ("hybrid", "topo"):
            res = mg_color_graph(shard, hc.HybridConfig(mode=mode), solver=solver)
            out.append((mode, res.colors, _recs4(res.report), res.report.valid, res.report.colors_used,
                        res.report.num_undirected_edges, shard.num_edges))
        solver.close()
        q.put((rank, out, None))
    except Exception as exc:  # reported to the parent
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_processes_sharded_csr():
    """One process per rank, each generating the pairs, cutting the same
    edge-balanced bounds and building ONLY its own rows; the solve, the
    records, valid and colors_used equal the single-GPU solve of the whole graph."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, out, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        got[rank] = out
    for p in procs:
        p.join(timeout=60)
    dg = G.build_csr_device(G.gen_rmat_edges(10, 8, 5), 1 << 10)
    for mode, colors, recs, valid, used, und, _ in got[0]:
        want, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert np.array_equal(colors, want) and np.array_equal(recs, _recs4(rep)), mode
        assert valid and used == rep.colors_used and und == dg.num_undirected_edges
    assert got[0][0][6] + got[1][0][6] == dg.num_edges  # the shards partition the half-edges


def test_virtual_report_valid_and_colors_used():
    dg = G.rmat_graph(11, 16, 4)
    res = virtual_color_graph(dg, hc.HybridConfig(), 3)
    want, rep = hc.color_graph(dg)
    assert res.report.valid and res.report.colors_used == rep.colors_used


def test_bench_two_ranks_share_gpu_line():
    """bench.py's N>1 path end to end (torchrun, 2 ranks, per-rank CSR shards,
    the peer-memory solve) with both ranks on cuda:0 (--share-gpu: gloo, the
    persistent kernels time-slice): one JSON line from rank 0, a valid
    coloring with RMAT-16's round count, half the CSR per rank."""
    import json
    import os
    import subprocess
    import sys

    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
           "--share-gpu", "--config", "rmat16", "--steps", "1", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=str(Path(__file__).resolve().parents[1]), env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["valid"] is True
    assert line["config"]["rounds"] == 96
    assert line["config"]["csr_shard_bytes_max"] < 0.7 * line["config"]["csr_bytes_total"]
