"""Full-size parity against the REFERENCE itself on the BASELINE configs.

For each config: generate + build the CSR on the GPU, solve on the GPU in
every mode asked for, copy the CSR to the host (bit-identical to the
reference's build_csr -- checked at smaller scales by tests/test_gpu_parity.py)
and run the reference's own `hybridcolor.color_graph` (oracle/_ref, its
compiled Cython/OpenMP backend, all host cores) on it.  Colors, round count,
colors_used and every per-round (mode, wl_in, wl_out, conflicts) must match.
The grid is checked against its closed form instead (the reference needs
~35 min of CPU for 4096^2): colors 1+((i+j) mod 2), rounds ceil((r+c)/2),
round-1 conflicts = #undirected edges.

    python scripts/full_parity.py rmat16 rmat22 er25 rmat26 grid4096 > out.json
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1912_01478_b200 as hc  # noqa: E402
from oracle import oracle as O  # noqa: E402

CONFIGS = {
    "rmat16": lambda: hc.rmat_graph(16, 16, 0),
    "rmat22": lambda: hc.rmat_graph(22, 16, 0),
    "er25": lambda: hc.er_graph(1 << 25, 32, 0),
    "rmat26": lambda: hc.rmat_graph(26, 16, 0),
    "grid4096": lambda: hc.grid_graph(4096, 4096),
}


def recs(report):
    return [[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
            for r in report.per_round]


def main():
    torch.cuda.set_device(0)
    ref = O.reference_module()
    modes = os.environ.get("MODES", "hybrid").split(",")
    workers = os.cpu_count() or 1
    out = []
    for name in sys.argv[1:]:
        dg = CONFIGS[name]()
        row = {"config": name, "num_nodes": dg.num_nodes, "num_undirected_edges": dg.num_undirected_edges}
        for mode in modes:
            cfg = hc.HybridConfig(mode=mode)
            colors, rep = hc.color_graph(dg, cfg)
            r = {"rounds": rep.total_rounds, "colors_used": rep.colors_used, "valid": rep.valid}
            if name.startswith("grid"):
                k = int(name[4:])
                i, j = np.divmod(np.arange(k * k), k)
                r["closed_form_colors"] = bool(np.array_equal(colors, 1 + (i + j) % 2))
                r["closed_form_rounds"] = rep.total_rounds == (k + k + 1) // 2
                r["round1_conflicts"] = rep.per_round[0].conflicts == dg.num_undirected_edges
                r["match"] = r["closed_form_colors"] and r["closed_form_rounds"] and r["round1_conflicts"]
            else:
                host = dg.to_host()
                g = ref.CsrGraph(host.num_nodes, host.num_edges, host.row_offsets, host.col_indices)
                t0 = time.perf_counter()
                rc, rrep = ref.color_graph(g, ref.HybridConfig(mode=mode, workers=workers))
                r["reference_seconds"] = time.perf_counter() - t0
                r["reference_workers"] = workers
                r["colors_equal"] = bool(np.array_equal(colors, rc))
                r["records_equal"] = recs(rep) == [[int(x.mode_used == "topo"), x.worklist_size_in,
                                                    x.worklist_size_out, x.conflicts] for x in rrep.per_round]
                r["rounds_equal"] = rep.total_rounds == rrep.total_rounds
                r["colors_used_equal"] = rep.colors_used == rrep.colors_used
                r["match"] = all(r[k] for k in ("colors_equal", "records_equal", "rounds_equal", "colors_used_equal"))
                del host, g, rc, rrep
            row[mode] = r
            print(json.dumps({name: {mode: r}}), file=sys.stderr, flush=True)
        out.append(row)
        del dg
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
