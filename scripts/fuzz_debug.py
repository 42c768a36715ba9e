"""Seeded fuzz of one graph family against the oracle, printing failing seeds
(dev aid): python scripts/fuzz_debug.py KIND N_SEEDS"""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import torch
import paper_1912_01478_b200 as hc
from oracle import oracle as O
from test_gpu_fuzz import _family, _recs

torch.cuda.set_device(0)
kind, nseeds = sys.argv[1], int(sys.argv[2])
bad = 0
for seed in range(nseeds):
    rng = np.random.default_rng(seed)
    n, e = _family(rng, kind)
    ro, ci = O.build_csr(n, np.asarray(e, dtype=np.int64))
    g = hc.CsrGraph(n, len(ci), ro, ci)
    for mode in ("data", "topo", "hybrid"):
        for thr in (0.0, 0.6):
            want, wrec = O.color(ro, ci, mode, thr)
            colors, rep = hc.color_graph(g, hc.HybridConfig(mode=mode, threshold_fraction=thr))
            got = _recs(rep)
            if not (np.array_equal(colors, want) and np.array_equal(got, wrec)):
                bad += 1
                i = next((i for i in range(min(len(got), len(wrec))) if not np.array_equal(got[i], wrec[i])), None)
                print(f"seed {seed} n={n} mode={mode} thr={thr}: colors_eq={np.array_equal(colors, want)} "
                      f"rounds {len(got)}/{len(wrec)} first diff round {None if i is None else i + 1}: "
                      f"{None if i is None else (got[i].tolist(), wrec[i].tolist())}", flush=True)
print(kind, "bad", bad, flush=True)
