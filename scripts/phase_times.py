"""Per-round assign / resolve phase times of one solve (development aid;
needs a build with -DHC_PHASE_TIMES=1, e.g. HCB_LIB=libhcb_pt.so).
usage: python scripts/phase_times.py CONFIG [MODE]"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1912_01478_b200 as hc
from paper_1912_01478_b200 import _lib

torch.cuda.set_device(0)
w = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
dg = hc.grid_graph(int(w[4:]), int(w[4:])) if w.startswith("grid") else (
    hc.rmat_graph(int(w[4:])) if w.startswith("rmat") else hc.er_graph(1 << int(w[2:]), 32))
s = hc.Solver(dg)
L = _lib.load()
thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
M = s.max_rec
stats = torch.zeros(13 * M, dtype=torch.int64, device="cuda")
rounds = ctypes.c_int64(0)
for _ in range(2):
    stats.zero_()
    _lib.check(L.hc_solve_stats(dg.row_offsets.data_ptr(), _lib.ptr(dg.col_indices), dg.num_nodes, dg.num_edges,
                                _lib.MODE_CODES[mode], thr, s.colors.data_ptr(), s.rec.data_ptr(), M,
                                ctypes.byref(rounds), stats.data_ptr(), s.ws.data_ptr(), s.ws.numel(),
                                _lib.stream_handle()))
torch.cuda.synchronize()
R = int(rounds.value)
rec = s.rec[:R].cpu().numpy()
st = stats.cpu().numpy()
ed = st[: 2 * M].reshape(M, 2)[:R]
tm = st[2 * M: 2 * M + 3 * R].reshape(R, 3)
uk = st[5 * M: 5 * M + 8 * R].reshape(R, 8) / 1e3  # longest unit per kind (hub, bin3..bin0), busiest CTA
a_us = (tm[:, 1] - tm[:, 0]) / 1e3
r_us = (tm[:, 2] - tm[:, 1]) / 1e3
print(f"{w} {mode}: rounds {R}, assign {a_us.sum()/1e3:.2f} ms, resolve {r_us.sum()/1e3:.2f} ms")
idx = list(range(min(6, R))) + list(range(6, R, max(1, R // 30)))
for i in idx:
    print(f"  r{rec[i,0]:5d} {'topo' if rec[i,1] else 'data'} wl={rec[i,2]:9d} conf={rec[i,4]:10d} "
          f"Ea={ed[i,0]:11d} El={ed[i,1]:11d}  assign {a_us[i]:8.1f} us  resolve {r_us[i]:8.1f} us"
          f"  | max unit hub {uk[i,0]:6.1f} b3 {uk[i,1]:6.1f} b2 {uk[i,2]:6.1f} b1 {uk[i,3]:6.1f} b0 {uk[i,4]:6.1f} busy {uk[i,5]:6.1f} push {uk[i,6]:6.1f}")
