"""Time solves under alternative in-tree builds (HCB_LIB=...; tuning aid).
usage: python scripts/variant_timing.py LIB[,LIB...] CONFIG[,CONFIG...]"""
import os, subprocess, sys
libs, cfgs = sys.argv[1].split(","), sys.argv[2].split(",")
code = r'''
import sys, torch; sys.path.insert(0, ".")
import paper_1912_01478_b200 as hc
torch.cuda.set_device(0)
for w in sys.argv[1].split(","):
    dg = hc.grid_graph(int(w[4:]), int(w[4:])) if w.startswith("grid") else (hc.rmat_graph(int(w[4:])) if w.startswith("rmat") else hc.er_graph(1 << int(w[2:]), 32))
    s = hc.Solver(dg); thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for mode in ("hybrid", "topo", "data"):
        s.run(mode, thr, fetch_records=False); ts = []
        for _ in range(3):
            flush.zero_(); ts.append(s.run(mode, thr, fetch_records=False).seconds * 1e3)
        print(f"{w:9s} {mode:6s} {min(ts):9.2f} ms", flush=True)
'''
for lib in libs:
    env = dict(os.environ, HCB_LIB=lib)
    print("==", lib, flush=True)
    subprocess.run([sys.executable, "-c", code, ",".join(cfgs)], env=env)
