"""Where the time of one small solve goes outside the solve kernel (dev aid):
CUDA-event time of hc_solve vs the kernel-only time from the per-round records."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1912_01478_b200 as hc

torch.cuda.set_device(0)
w = sys.argv[1] if len(sys.argv) > 1 else "rmat16"
dg = hc.rmat_graph(int(w[4:])) if w.startswith("rmat") else hc.grid_graph(int(w[4:]), int(w[4:]))
s = hc.Solver(dg)
thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
for _ in range(3):
    s.run("hybrid", thr)
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = s.run("hybrid", thr)
    t1 = time.perf_counter()
    print(f"{w}: event {r.seconds*1e3:.3f} ms  host wall {1e3*(t1-t0):.3f} ms  rounds-sum {r.records[:,5].sum()/1e6:.3f} ms")
