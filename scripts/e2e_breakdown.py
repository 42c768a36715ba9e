"""Where the end-to-end color_graph time goes (grid4096 default; dev aid)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1912_01478_b200 as hc

torch.cuda.set_device(0)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dg = hc.grid_graph(k, k)
host = hc.CsrGraph.pinned(dg.to_host())
cfg = hc.HybridConfig()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d2 = host.to_device(); torch.cuda.synchronize(); t1 = time.perf_counter()
    s = hc.Solver(d2); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = s.run("hybrid", hc.threshold_count(cfg, d2.num_nodes)); t3 = time.perf_counter()
    used = hc.driver._colors_used_device(r.colors); bad = hc.driver._verify_device(d2, r.colors); t4 = time.perf_counter()
    h = torch.empty(r.colors.shape, dtype=torch.int64, pin_memory=True); h.copy_(r.colors, non_blocking=True)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    torch.cuda.synchronize(); t6 = time.perf_counter()
    c, rep = hc.color_graph(host, cfg); torch.cuda.synchronize(); t7 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.1f}  solver {1e3*(t2-t1):.1f}  solve {1e3*(t3-t2):.1f} (dev {1e3*r.seconds:.1f})  "
          f"used+verify {1e3*(t4-t3):.1f}  d2h {1e3*(t5-t4):.1f}  | color_graph total {1e3*(t7-t6):.1f} ms", flush=True)
