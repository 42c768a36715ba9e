"""Multi-GPU path overhead on ONE GPU: hc_solve vs the peer-memory solve with
P virtual ranks sharing the GPU (same total CTAs).  Not a scaling number --
the ranks share one GPU's SMs and HBM -- but it prices the cross-GPU barrier
protocol (fence.sys + mailbox all-reduce) and the mirrored stores."""
import sys
sys.path.insert(0, ".")
import json
import torch
import paper_1912_01478_b200 as hc
from paper_1912_01478_b200.multigpu import VirtualMesh, virtual_color_graph

torch.cuda.set_device(0)
out = {}
for name in sys.argv[1:] or ["grid4096", "rmat22"]:
    if name.startswith("grid"):
        k = int(name[4:]); dg = hc.grid_graph(k, k)
    elif name.startswith("rmat"):
        dg = hc.rmat_graph(int(name[4:]))
    else:
        dg = hc.er_graph(1 << int(name[2:]), 32)
    cfg = hc.HybridConfig()
    s = hc.Solver(dg)
    thr = hc.threshold_count(cfg, dg.num_nodes)
    s.run("hybrid", thr, fetch_records=False)
    single = min(s.run("hybrid", thr, fetch_records=False).seconds for _ in range(3))
    want = s.run("hybrid", thr).colors.cpu().numpy()
    row = {"single_ms": single * 1e3}
    for world in [int(w) for w in __import__("os").environ.get("WORLDS", "1,2,4,8").split(",")]:
        mesh = VirtualMesh(dg, world, timeout_ms=60000)
        virtual_color_graph(dg, cfg, world, mesh=mesh)
        ts = []
        for _ in range(3):
            r = virtual_color_graph(dg, cfg, world, mesh=mesh)
            ts.append(r.seconds)
        assert (r.colors == want).all()
        row[f"virtual{world}_ms"] = min(ts) * 1e3
        row["rounds"] = r.report.total_rounds
        del mesh
    out[name] = row
    print(name, json.dumps(row), flush=True)
