"""Reference-generated full-size digests for the BASELINE configs C1/C3/C4/C5.

Run on the GPU box host (the reference is CPU code; the graph is generated and
CSR-built on the GPU, copied to the host as int64 -- bit-identical to the
reference's build_csr, tests/test_gpu_parity.py -- and handed to the reference's
own `hybridcolor.color_graph` from oracle/_ref, Cython/OpenMP backend, all host
cores).  For every (config, mode) it records

  * sha256 of the reference's int64 colors,
  * sha256 of the int64 (rounds x 4) array (topo?, wl_in, wl_out, conflicts)
    of the reference's per-round records (driver.py:159-168),
  * rounds, colors_used, reference seconds,
  * sha256 of the CSR it colored (pins the generator + build),

and the GPU's own solve of the same graph next to it.  The output is committed as
tests/golden/full_digests.json; tests/test_full_parity.py (-m gpu) recomputes
the GPU digests and compares them with the REFERENCE's.  Results are appended to
gpurun_out/ref_digests.jsonl as they finish so a cut-off run keeps its rows.

    python scripts/ref_digests.py rmat16 rmat22 er25 rmat26   # MODES=hybrid,data,topo
"""

import hashlib
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
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rec_array(per_round) -> np.ndarray:
    return np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                     for r in per_round], dtype=np.int64).reshape(-1, 4)


def main():
    torch.cuda.set_device(0)
    ref = O.reference_module()
    modes = os.environ.get("MODES", "hybrid,data,topo").split(",")
    workers = os.cpu_count() or 1
    os.makedirs("gpurun_out", exist_ok=True)
    log = open("gpurun_out/ref_digests.jsonl", "a")
    for name in sys.argv[1:]:
        dg = CONFIGS[name]()
        host = dg.to_host()
        csr = {"ro": sha(host.row_offsets.astype("<i8")), "ci": sha(host.col_indices.astype("<i8"))}
        g = ref.CsrGraph(host.num_nodes, host.num_edges, host.row_offsets, host.col_indices)
        ref.color_graph(ref.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1])))  # warm start
        for mode in modes:
            colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
            t0 = time.perf_counter()
            rc, rrep = ref.color_graph(g, ref.HybridConfig(mode=mode, workers=workers))
            secs = time.perf_counter() - t0
            row = {
                "config": name, "mode": mode, "num_nodes": host.num_nodes, "num_edges": host.num_edges,
                "csr_sha256": csr,
                "reference": {"colors_sha256": sha(np.asarray(rc, dtype="<i8")),
                              "records_sha256": sha(rec_array(rrep.per_round)),
                              "rounds": rrep.total_rounds, "colors_used": rrep.colors_used,
                              "valid": rrep.valid, "seconds": secs, "workers": workers,
                              "round1": rec_array(rrep.per_round)[0].tolist()},
                "gpu": {"colors_sha256": sha(colors.astype("<i8")), "records_sha256": sha(rec_array(rep.per_round)),
                        "rounds": rep.total_rounds, "colors_used": rep.colors_used, "valid": rep.valid},
            }
            row["match"] = all(row["gpu"][k] == row["reference"][k]
                               for k in ("colors_sha256", "records_sha256", "rounds", "colors_used"))
            print(json.dumps(row), file=log, flush=True)
            print(json.dumps({name: {mode: row["match"], "ref_s": round(secs, 2)}}), flush=True)
            del rc, rrep, colors
        del host, g, dg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
