"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck)."""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1912_01478_b200 as hc
from oracle import oracle as O
from paper_1912_01478_b200.pushbench import BenchConfig, run_push_bench

from paper_1912_01478_b200 import _lib as _L0

for scale in (8, 10):
    dg = hc.rmat_graph(scale, 16, 1)
    ro, ci = O.build_csr(1 << scale, O.gen_rmat(scale, 16, 1))
    for live in (-1, 1):  # per-graph default, then the live-lower-list instantiation forced
        _L0.load().hc_solve_set_live(live)
        for mode in ("data", "topo", "hybrid"):
            c, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
            want, _ = O.color(ro, ci, mode)
            assert np.array_equal(c, want)
    _L0.load().hc_solve_set_live(-1)
dg = hc.grid_graph(40, 30)
c, rep = hc.color_graph(dg)
# 8-bit state words (every degree <= 128), and their overflow rerun (K_128)
ro, ci = O.build_csr(2000, O.gen_er(2000, 2000 * 30, 3))
c, rep = hc.color_graph(hc.CsrGraph(2000, len(ci), ro, ci).to_device())
assert np.array_equal(c, O.color(ro, ci, "hybrid")[0])
iu, ju = np.triu_indices(128, 1)
ro, ci = O.build_csr(128, np.stack([iu, ju], 1).astype(np.int64))
c, rep = hc.color_graph(hc.CsrGraph(128, len(ci), ro, ci).to_device())
assert np.array_equal(c, O.color(ro, ci, "hybrid")[0])
# star hub (bin 4, split slices) + per-round plugin API + worklist sort
n = 6000
e = np.concatenate([np.column_stack([np.zeros(n - 1, np.int64), np.arange(1, n)]),
                    np.random.default_rng(1).integers(0, n, (3000, 2))])
g = hc.build_csr(hc.EdgeList(n, e))
c, rep = hc.color_graph(g)
state, wl = hc.ColorState.fresh(n), hc.Worklist.init_full(n)
hc.data_driven_iteration(g, state, wl, 1)
hc.topology_driven_iteration(g, state, wl, 2)
run_push_bench(5000, BenchConfig(batch_size=300, repetitions=1))
print("sanitize workload ok")

# bin-0-only kernel on a delta-column grid, multi-GPU virtual ranks (both
# exchange modes), device MatrixMarket parse and degree statistics
from paper_1912_01478_b200 import _lib
from paper_1912_01478_b200.multigpu import virtual_color_graph

import os

dg = hc.grid_graph(50, 37)
want, _ = hc.color_graph(dg)
# virtual ranks need their persistent kernels to run concurrently, which the
# sanitizers serialize: only world = 1 there unless SANITIZE_MG=1
worlds = (2, 3) if os.environ.get("SANITIZE_MG") == "1" else (1,)
for ex in (0, 1, 2):
    _lib.load().hc_mg_set_exchange(ex)
    for world in worlds:
        r = virtual_color_graph(dg, hc.HybridConfig(), world, timeout_ms=120000)
        assert np.array_equal(r.colors, want)
    r = virtual_color_graph(hc.rmat_graph(9, 16, 2), hc.HybridConfig(), worlds[-1], timeout_ms=120000)
_lib.load().hc_mg_set_exchange(0)
el = hc.parse_matrix_market("%%MatrixMarket matrix coordinate pattern general\n4 4 3\n1 2\n% c\n3 4 7\n\n2 3\n")
assert el.edges.tolist() == [[0, 1], [2, 3], [1, 2]]
s = hc.degree_stats(hc.rmat_graph(10, 16, 3))
print("sanitize workload ok (incl. multi-GPU + ingestion)")
