"""Time solves under alternative in-tree builds (HCB_LIB=...; tuning aid).
usage: python scripts/variant_timing.py LIB[,LIB...] CONFIG[,CONFIG...]
A LIB may carry runtime knobs: libhcb.so:ell=0:small=0:l2=0"""
import os, subprocess, sys
libs, cfgs = sys.argv[1].split(","), sys.argv[2].split(",")
code = r'''
import sys, torch; sys.path.insert(0, ".")
import paper_1912_01478_b200 as hc
torch.cuda.set_device(0)
L = hc._lib.load()
for kv in sys.argv[2].split(":") if len(sys.argv) > 2 and sys.argv[2] else []:
    k, v = kv.split("=")
    {"ell": L.hc_solve_set_ell, "small": L.hc_solve_set_small, "l2": L.hc_solve_set_l2_window, "live": L.hc_solve_set_live, "x8": L.hc_solve_set_x8}[k](int(v))
for w in sys.argv[1].split(","):
    dg = hc.grid_graph(int(w[4:]), int(w[4:])) if w.startswith("grid") else (hc.rmat_graph(int(w[4:])) if w.startswith("rmat") else hc.er_graph(1 << int(w[2:]), 32))
    s = hc.Solver(dg); thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for mode in ("hybrid", "topo", "data"):
        s.run(mode, thr, fetch_records=False); ts = []
        for _ in range(3):
            flush.zero_(); ts.append(s.run(mode, thr, fetch_records=False).seconds * 1e3)
        print(f"{w:9s} {mode:6s} {min(ts):9.2f} ms", flush=True)
    col, rep = hc.color_graph(dg, hc.HybridConfig())
    print(f"{w:9s} valid={rep.valid} colors={rep.colors_used} rounds={rep.total_rounds}", flush=True)
    del s, dg, flush; torch.cuda.empty_cache()
'''
for spec in libs:
    lib, *knobs = spec.split(":")
    env = dict(os.environ, HCB_LIB=lib)
    print("==", spec, flush=True)
    subprocess.run([sys.executable, "-c", code, ",".join(cfgs), ":".join(knobs)], env=env)
