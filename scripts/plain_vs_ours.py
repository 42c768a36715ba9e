"""Per-round times of the production solve vs the Plain variant (dev aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1912_01478_b200 as hc

torch.cuda.set_device(0)
w = sys.argv[1]
dg = hc.rmat_graph(int(w[4:])) if w.startswith("rmat") else hc.er_graph(1 << int(w[2:]), 32)
s = hc.Solver(dg)
thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
res = {}
for plain in (False, True):
    for _ in range(3):
        r = s.run("hybrid", thr, plain=plain)
    res[plain] = (r.seconds, r.records[:, 5] / 1e3)
print(f"{w}: ours {res[False][0]*1e3:.3f} ms (rounds {res[False][1].sum()/1e3:.3f}), plain {res[True][0]*1e3:.3f} ms (rounds {res[True][1].sum()/1e3:.3f})")
a, b = res[False][1], res[True][1]
for i in list(range(0, 10)) + list(range(10, len(a), max(1, len(a) // 15))):
    print(f"  r{i+1:4d} ours {a[i]:8.1f} us  plain {b[i]:8.1f} us")
