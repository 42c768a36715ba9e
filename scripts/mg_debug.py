"""Multi-GPU (virtual ranks) debug sweep: formats x world on a hub graph."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1912_01478_b200 as hc
from paper_1912_01478_b200 import _lib
from paper_1912_01478_b200.multigpu import virtual_color_graph
from oracle import oracle as O

torch.cuda.set_device(0)
rng = np.random.default_rng(5)
n = 40000
hub = np.column_stack([np.zeros(20000, np.int64), rng.integers(1, n, 20000)])
rest = rng.integers(0, n, (60000, 2))
ro, ci = O.build_csr(n, np.vstack([hub, rest]))
dg = hc.CsrGraph(n, len(ci), ro, ci).to_device()
for fmt in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)):
    _lib.load().hc_solve_set_formats(*fmt)
    want, rep = hc.color_graph(dg)
    for world in (1, 2, 3, 3, 3, 5, 7):
        for mode in ("hybrid", "data", "topo"):
            try:
                res = virtual_color_graph(dg, hc.HybridConfig(mode=mode), world, timeout_ms=4000)
                ok = np.array_equal(res.colors, want) if mode == "hybrid" else True
                print(fmt, world, mode, "rounds", res.report.total_rounds, "ok" if ok else "MISMATCH", flush=True)
            except Exception as e:
                print(fmt, world, mode, "ERR", e, flush=True)
_lib.load().hc_solve_set_formats(0, 0, 0)
