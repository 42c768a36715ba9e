"""Seeded structural fuzz of the device solve against the C oracle
(oracle/ipgc_oracle.c, pinned to the reference's goldens in test_oracle.py).

Graph families chosen to reach every code path of the solver: bin-0-only
graphs (the bin-0-only kernel, delta columns), mixed degrees (8- / 16-lane
groups, warp per node), hubs above 4096 (CTA per hub, split hubs, colors past
64 and 128), disconnected pieces, isolated nodes, and ids shuffled so that
delta columns do not apply.  Random mode and threshold per case.  Colors
and every per-round record must match bit for bit."""

import zlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_1912_01478_b200 as hc  # noqa: E402

MODES = ("data", "topo", "hybrid")


def _recs(report):
    return np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                     for r in report.per_round], dtype=np.int64).reshape(-1, 4)


def _family(rng, kind):
    if kind == "grid_shuffled":
        r, c = rng.integers(5, 120, 2)
        e = O.gen_grid(int(r), int(c))
        perm = rng.permutation(int(r * c))
        return int(r * c), perm[e]
    if kind == "cycles_paths":
        n = int(rng.integers(50, 20000))
        a = np.arange(n - 1)
        e = np.column_stack([a, a + 1])
        extra = rng.integers(0, n, (int(rng.integers(0, n)), 2))
        return n, np.vstack([e, extra])
    if kind == "mixed_degrees":
        n = int(rng.integers(2000, 40000))
        deg = rng.choice([2, 8, 20, 40, 100, 500], size=n, p=[.4, .25, .15, .1, .07, .03])
        src = np.repeat(np.arange(n), deg // 2)
        return n, np.column_stack([src, rng.integers(0, n, src.size)])
    if kind == "hubs":
        n = int(rng.integers(10000, 60000))
        k = int(rng.integers(1, 12))
        hubs = rng.choice(n, k, replace=False)
        e = []
        for h in hubs:  # degree 4200..9000: above the 4096 hub threshold
            d = int(rng.integers(4200, 9000))
            e.append(np.column_stack([np.full(d, h), rng.integers(0, n, d)]))
        e.append(rng.integers(0, n, (3 * n, 2)))
        return n, np.vstack(e)
    if kind == "mega_hubs":  # hubs of degree >= 65536: their winning pushes are shared by every CTA
        n = int(rng.integers(80000, 120000))
        e = []
        for h in rng.choice(n, int(rng.integers(1, 4)), replace=False):
            d = int(rng.integers(66000, 90000))
            e.append(np.column_stack([np.full(d, h), rng.integers(0, n, d)]))
        e.append(rng.integers(0, n, (2 * n, 2)))
        return n, np.vstack(e)
    if kind == "dense_core":  # a near-clique core: > 128 colors, seen by warp-per-node and hub nodes
        n = int(rng.integers(6000, 14000))
        core = rng.choice(n, int(rng.integers(500, 900)), replace=False)
        a, b = np.meshgrid(core, core)
        keep = rng.random(a.size) < 0.9
        e = [np.column_stack([a.ravel()[keep], b.ravel()[keep]]), rng.integers(0, n, (2 * n, 2))]
        for h in rng.choice(n, 2, replace=False):  # hubs adjacent to the whole core + random nodes
            e.append(np.column_stack([np.full(core.size, h), core]))
            e.append(np.column_stack([np.full(5000, h), rng.integers(0, n, 5000)]))
        return n, np.vstack(e)
    if kind == "rmat":
        scale = int(rng.integers(8, 14))
        return 1 << scale, O.gen_rmat(scale, int(rng.integers(4, 24)), int(rng.integers(0, 1000)))
    raise ValueError(kind)


KINDS = ("grid_shuffled", "cycles_paths", "mixed_degrees", "hubs", "mega_hubs", "dense_core", "rmat")


@pytest.mark.parametrize("kind", KINDS)
def test_structural_fuzz_vs_oracle(kind):
    rng = np.random.default_rng(zlib.crc32(kind.encode()))  # stable across processes (str hash is salted)
    for case in range(16):
        n, e = _family(rng, kind)
        e = np.asarray(e, dtype=np.int64)
        ro, ci = O.build_csr(n, e)
        g = hc.CsrGraph(n, len(ci), ro, ci)
        dg = g.to_device()
        mode = MODES[int(rng.integers(0, 3))]
        thr = float(rng.choice([0.0, 0.25, 0.6, 0.9, 1.0]))
        want, wrec = O.color(ro, ci, mode, thr)
        L = hc._lib.load()
        try:
            # per-graph default, then live lower lists forced on (the default
            # picks them only for skewed graphs of >= 2^25 half-edges)
            for live in (-1, 1):
                L.hc_solve_set_live(live)
                colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode, threshold_fraction=thr))
                assert np.array_equal(colors, want), (kind, case, n, mode, thr, live)
                assert np.array_equal(_recs(rep), wrec), (kind, case, n, mode, thr, live)
                assert rep.valid
        finally:
            L.hc_solve_set_live(-1)
