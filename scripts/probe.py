"""Quick timing probe (development aid): solve times per mode on named graphs."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1912_01478_b200 as hc

def run(name, dg, reps=3):
    for mode in ("hybrid", "data", "topo"):
        s = hc.Solver(dg)
        thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
        s.run(mode, thr)  # warm
        ts = [s.run(mode, thr, fetch_records=False).seconds for _ in range(reps)]
        r = s.run(mode, thr)
        print(f"{name:10s} {mode:6s} n={dg.num_nodes} m={dg.num_edges} rounds={r.rounds} "
              f"best={min(ts)*1e3:.2f}ms med={sorted(ts)[len(ts)//2]*1e3:.2f}ms "
              f"und_edges/s={dg.num_edges/2/min(ts)/1e9:.3f}G", flush=True)

torch.cuda.set_device(0)
which = sys.argv[1:] or ["rmat16", "grid1024", "rmat22", "grid4096", "er25"]
for w in which:
    t = time.time()
    if w.startswith("rmat"):
        dg = hc.rmat_graph(int(w[4:]))
    elif w.startswith("grid"):
        k = int(w[4:]); dg = hc.grid_graph(k, k)
    elif w.startswith("er"):
        dg = hc.er_graph(1 << int(w[2:]), 32)
    torch.cuda.synchronize()
    print(f"{w}: build {time.time()-t:.2f}s", flush=True)
    run(w, dg)
    del dg
    torch.cuda.empty_cache()
