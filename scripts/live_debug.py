"""Small-graph check of the solve against the oracle (dev aid for kernel changes)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1912_01478_b200 as hc
from oracle import oracle as O

torch.cuda.set_device(0)
cases = [("rmat", 10, 1), ("rmat", 12, 2), ("er", 1 << 12, 3), ("rmat", 14, 0), ("er", 1 << 15, 5), ("rmat", 16, 0)]
for kind, a, seed in cases:
    if kind == "rmat":
        n = 1 << a; e = O.gen_rmat(a, 16, seed)
    else:
        n = a; e = O.gen_er(n, n * 16, seed)
    ro, ci = O.build_csr(n, e)
    g = hc.CsrGraph(n, len(ci), ro, ci)
    for mode in ("data", "topo", "hybrid"):
        want, rec = O.color(ro, ci, mode)
        try:
            colors, rep = hc.color_graph(g, hc.HybridConfig(mode=mode))
        except Exception as exc:
            print(kind, a, mode, "ERROR", exc, flush=True)
            continue
        got = np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                        for r in rep.per_round], dtype=np.int64).reshape(-1, 4)
        ok = np.array_equal(colors, want) and np.array_equal(got, rec)
        print(kind, a, mode, "ok" if ok else "MISMATCH", rep.total_rounds, len(rec), flush=True)
        if not ok:
            for i in range(min(len(got), len(rec))):
                if not np.array_equal(got[i], rec[i]):
                    print("   first diff round", i + 1, got[i], rec[i]); break
