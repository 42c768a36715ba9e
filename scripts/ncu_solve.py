"""Run a few solves of one config (for ncu capture; development aid)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1912_01478_b200 as hc
torch.cuda.set_device(0)
w = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if w.startswith("rmat"):
    dg = hc.rmat_graph(int(w[4:]))
elif w.startswith("grid"):
    k = int(w[4:]); dg = hc.grid_graph(k, k)
else:
    dg = hc.er_graph(1 << int(w[2:]), 32)
s = hc.Solver(dg)
thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
for _ in range(reps):
    r = s.run(mode, thr, fetch_records=False)
    print(w, mode, f"{r.seconds*1e3:.2f} ms", r.rounds)
