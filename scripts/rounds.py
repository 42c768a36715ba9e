"""Per-round timing profile of one solve (development aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1912_01478_b200 as hc

def graph(w):
    if w.startswith("rmat"):
        return hc.rmat_graph(int(w[4:]))
    if w.startswith("grid"):
        k = int(w[4:]); return hc.grid_graph(k, k)
    return hc.er_graph(1 << int(w[2:]), 32)

torch.cuda.set_device(0)
for w in sys.argv[1:]:
    dg = graph(w)
    h = dg.to_host() if dg.num_nodes <= (1 << 22) else None
    if h is not None:
        deg = np.diff(h.row_offsets)
        print(w, "bins: small", int((deg <= 16).sum()), "mid", int(((deg > 16) & (deg <= 2046)).sum()),
              "hub", int((deg > 2046).sum()), "maxdeg", int(deg.max()))
    s = hc.Solver(dg)
    thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
    s.run("hybrid", thr)
    r = s.run("hybrid", thr)
    rec = r.records
    ns = rec[:, 5] / 1e3
    print(f"{w}: total {r.seconds*1e3:.2f} ms, rounds {r.rounds}, sum(round us) {ns.sum()/1e3:.2f} ms")
    idx = list(range(min(8, len(rec)))) + list(range(8, len(rec), max(1, len(rec) // 24)))
    for i in idx:
        print(f"  r{rec[i,0]:5d} {'topo' if rec[i,1] else 'data'} wl_in={rec[i,2]:9d} conf={rec[i,4]:9d} {ns[i]:9.1f} us")
    print("  us/round quantiles 10/50/90/max:", np.percentile(ns, [10, 50, 90, 100]).round(1))
