"""Record the per-round work profile (node + edge visits) of a config's
hybrid solve for the CPU reference arm's extrapolation (profiles/work_*.json)."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch

import bench
import paper_1912_01478_b200 as hc
from paper_1912_01478_b200 import _lib

torch.cuda.set_device(0)
for name in sys.argv[1:]:
    dg = bench.build_graph(hc, bench.CONFIGS[name])
    s = hc.Solver(dg)
    n = dg.num_nodes
    thr = hc.threshold_count(hc.HybridConfig(), n)
    stats = torch.zeros((s.max_rec, 2), dtype=torch.int64, device="cuda")
    rounds = ctypes.c_int64(0)
    _lib.check(_lib.load().hc_solve_stats(dg.row_offsets.data_ptr(), _lib.ptr(dg.col_indices), n, dg.num_edges,
                                          2, thr, s.colors.data_ptr(), s.rec.data_ptr(), s.max_rec,
                                          ctypes.byref(rounds), stats.data_ptr(), s.ws.data_ptr(), s.ws.numel(),
                                          _lib.stream_handle()))
    R = rounds.value
    rec = s.rec[:R].cpu().numpy()
    st = stats[:R].cpu().numpy()
    work = bench.round_work(rec, st)
    out = {"config": name, "rounds": R, "sum_wl_in": int(rec[:, 2].sum()), "work": work,
           "definition": "per round: wl_in + assign edge visits + resolve lower-edge visits (hc_solve_stats)"}
    with open(f"gpurun_out/work_{name}.json", "w") as f:
        json.dump(out, f)
    print(name, R, sum(work))
