"""Benchmark: edges/sec per IPGC solve (BASELINE.json metric), hybrid vs
data-driven vs topology-driven, on the BASELINE configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config grid4096]
                    [--impl ours|reference]

A step = one complete hybrid IPGC solve (hc_solve: bin preprocessing + the
device-resident round loop) of the config's graph, inputs resident in HBM.
L2 is flushed between timed steps (a 512 MiB write, outside the events).
value = num_undirected_edges * steps / (sum of per-step CUDA-event times),
max over ranks.  e2e = the same metric through the public drop-in API
`color_graph(CsrGraph on pinned host memory)`: H2D of the CSR, solve, D2H of
the colors, device verification.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref: hybridcolor with its compiled Cython/OpenMP
backend) on the same graph -- see cpu_sample() for the bounded-sample rule.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

CONFIGS = {
    # BASELINE.json configs[0..4]
    "rmat16": dict(kind="rmat", scale=16, edgefactor=16, seed=0),
    "grid4096": dict(kind="grid", rows=4096, cols=4096),
    "rmat22": dict(kind="rmat", scale=22, edgefactor=16, seed=0),
    "er25": dict(kind="er", n=1 << 25, avg_degree=32, seed=0),
    "rmat26": dict(kind="rmat", scale=26, edgefactor=16, seed=0),
}
DESCRIPTIONS = {
    "rmat16": "RMAT scale-16 edgefactor-16 undirected, seed 0 (configs[0])",
    "grid4096": "2D grid 4096x4096 4-neighbor (configs[1])",
    "rmat22": "RMAT scale-22 edgefactor-16, seed 0 (configs[2])",
    "er25": "Erdos-Renyi 2^25 nodes avg degree 32, seed 0 (configs[3])",
    "rmat26": "RMAT scale-26 edgefactor-16, seed 0 (configs[4])",
}
METRIC = "edges/sec per IPGC solve (hybrid)"
UNIT = "undirected_edges/s"


def peaks():
    try:
        return json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
# algorithmic byte models.  Per round t: W = processed nodes (wl_in), E = sum
# of their degrees, El = their lower-id neighbours (hc_solve_stats), W' =
# wl_out; n nodes, m directed half-edges.
#
# SURVEY.md §8(d) (the roofline.achieved numerator; scan-based assign, int32
# ids/colors, int64 offsets, int64 packed (t,T)):
#   assign : data 20|W| + 8E         topo 4n + 16|W| + 8E
#   resolve: data 24|W| + 12El + 4|W'|   topo 4n + 20|W| + 12El + 4|W'|
#
# the implemented algorithm (bitmap assign, one 4 B state word,
# 4 B ids): assign reads the list entry and the node's forbidden-color word and
# writes the tentative word; resolve reads list, offsets, own word and per lower
# neighbour (column + word), writes the word or the push; every winner adds
# its color to each neighbour's bitmap once per solve (column + RED word):
#   assign : data 12|W|              topo 4n + 8|W|
#   resolve: data 20|W| + 8El        topo 4n + 16|W| + 8El
#   + 8m per solve
# --------------------------------------------------------------------------
def survey_bytes(records: np.ndarray, stats: np.ndarray, n: int) -> int:
    total = 0
    for r, (ea, er) in zip(records, stats):
        topo, w, w2 = int(r[1]), int(r[2]), int(r[3])
        if topo:
            total += 4 * n + 16 * w + 8 * int(ea) + 4 * n + 20 * w + 12 * int(er) + 4 * w2
        else:
            total += 20 * w + 8 * int(ea) + 24 * w + 12 * int(er) + 4 * w2
    return total


def own_bytes(records: np.ndarray, stats: np.ndarray, n: int, m: int) -> int:
    total = 8 * m
    for r, (_, er) in zip(records, stats):
        topo, w = int(r[1]), int(r[2])
        if topo:
            total += 4 * n + 8 * w + 4 * n + 16 * w + 8 * int(er)
        else:
            total += 12 * w + 20 * w + 8 * int(er)
    return total


def measured_traffic(config):
    """DRAM bytes (read + write), duration and L2 hit rate of one solve_kernel
    launch of this config from the committed ncu capture of the current code
    (profiles/r02_<config>_traffic.csv, scripts/profile_configs.sh:
    dram__bytes_read.sum + dram__bytes_write.sum, gpu__time_duration.sum,
    --clock-control none), or None when there is no capture."""
    import csv

    p = REPO / "profiles" / f"r02_{config}_traffic.csv"
    if not p.exists():
        return None
    per = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "ms": 1e6,
             "s": 1e9, "%": 1}
    with p.open() as f:
        for row in csv.DictReader(ln for ln in f if ln.startswith('"')):
            if "solve_kernel" not in row.get("Kernel Name", ""):
                continue
            d = per.setdefault(row["ID"], {})
            v = float(row["Metric Value"].replace(",", "")) * scale.get(row.get("Metric Unit", ""), 1)
            d[row["Metric Name"]] = v
    rows = [d for d in per.values() if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d]
    if not rows:
        return None
    k = len(rows)
    out = {"bytes": int(sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in rows) / k),
           "ns": int(sum(d.get("gpu__time_duration.sum", 0) for d in rows) / k)}
    if all("lts__t_sector_hit_rate.pct" in d for d in rows):
        out["l2_hit_pct"] = sum(d["lts__t_sector_hit_rate.pct"] for d in rows) / k
    return out


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# CPU side: the reference's own implementation on the host cores
# --------------------------------------------------------------------------
def host_csr(cfg):
    """The config's graph built on the CPU by the oracle (test infrastructure;
    bit-identical to the device build and to the reference build_csr, see
    tests/test_oracle.py + tests/test_gpu_parity.py)."""
    from oracle import oracle as O

    if cfg["kind"] == "grid":
        n = cfg["rows"] * cfg["cols"]
        e = O.gen_grid(cfg["rows"], cfg["cols"])
    elif cfg["kind"] == "er":
        n = cfg["n"]
        e = O.gen_er(n, n * cfg["avg_degree"] // 2, cfg["seed"])
    else:
        n = 1 << cfg["scale"]
        e = O.gen_rmat(cfg["scale"], cfg["edgefactor"], cfg["seed"])
    ro, ci = O.build_csr(n, e)
    return n, ro, ci


def cpu_sample(ref, g, budget_s: float, work: list | None):
    """Run the reference's hybrid loop (driver.py:143-169, through its public
    data_driven_iteration / topology_driven_iteration) on the host for at most
    `budget_s` seconds.  If the solve finishes, the rate is exact; otherwise the
    full-solve time is extrapolated from the sampled rounds by per-round work
    (node visits + edge visits of round t, known exactly from the
    bit-identical GPU trajectory, hc_solve_stats):
        T_full = T_sample * sum_t work_t / sum_{t<=R} work_t."""
    workers = os.cpu_count() or 1
    cfgr = ref.HybridConfig(mode="hybrid", workers=workers)
    n = g.num_nodes
    thr = math.ceil(cfgr.threshold_fraction * n)
    state = ref.ColorState.fresh(n)
    wl = ref.Worklist.init_full(n)
    round_no, t_loop = 1, 0.0
    t0 = time.perf_counter()
    while len(wl.current) > 0:
        size_in = len(wl.current)
        it = ref.topology_driven_iteration if size_in > thr else ref.data_driven_iteration
        ts = time.perf_counter()
        it(g, state, wl, round_no, workers=workers, chunk_size=cfgr.chunk_size)
        t_loop += time.perf_counter() - ts
        round_no += 1
        if time.perf_counter() - t0 > budget_s:
            break
    rounds = round_no - 1
    finished = len(wl.current) == 0
    if finished:
        secs = t_loop
        sample = f"full hybrid solve ({rounds} rounds)"
    else:
        if not work:
            return None
        done = float(sum(work[:rounds]))
        total = float(sum(work))
        secs = t_loop * total / done
        sample = (f"first {rounds} of {len(work)} rounds of the hybrid solve ({100 * done / total:.2f}% of the "
                  f"node+edge visits), extrapolated by per-round work")
    return {"value": (g.num_edges // 2) / secs, "unit": UNIT, "cores": workers, "kind": "reference",
            "sample": sample, "solve_seconds": secs, "finished": finished, "sample_seconds": t_loop,
            "rounds_run": rounds, "extrapolated": not finished}


def reference_module():
    from oracle import oracle as O

    ref = O.reference_module()
    if ref is None:
        raise RuntimeError("oracle/_ref missing: run oracle/build_ref.sh in the build container")
    assert "cython" in ref.available_backends()
    return ref


def warm_reference(ref):
    g = ref.build_csr(ref.EdgeList(64, np.column_stack([np.arange(63), np.arange(1, 64)])))
    ref.color_graph(g, ref.HybridConfig(workers=os.cpu_count() or 1))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = reference_module()
    warm_reference(ref)
    n, ro, ci = host_csr(cfg)
    g = ref.CsrGraph(n, len(ci), ro, ci)
    work = known_work(args.config)
    steps = max(1, args.steps)
    per_step = min(30.0, max(5.0, 150.0 / (steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(ref, g, per_step / 3, work)
    vals, sample_s = [], []
    last = None
    for _ in range(steps):
        last = cpu_sample(ref, g, per_step, work)
        vals.append(last["value"])
        sample_s.append(last["sample_seconds"])
    value = float(statistics.mean(vals))
    # ms_per_step is the wall time of one timed step (the bounded sample the
    # host actually ran); the full-solve time it stands for is reported beside it
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(statistics.mean(sample_s)),
        "ms_per_full_solve": (g.num_edges // 2) / value * 1e3, "extrapolated": bool(last["extrapolated"]),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (BASELINE generator spec, SURVEY.md Appendix C)",
        "config": {"workload": DESCRIPTIONS[args.config], "name": args.config, "mode": "hybrid",
                   "num_nodes": n, "num_undirected_edges": len(ci) // 2},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "reference",
                         "sample": last["sample"], "extrapolated": bool(last["extrapolated"])},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def known_work(config):
    """Per-round work (node + edge visits) of the full hybrid solve, recorded
    from the bit-identical GPU trajectory (profiles/work_<config>.json, written
    by scripts/work_profile.py) -- the reference arm runs without a GPU."""
    p = REPO / "profiles" / f"work_{config}.json"
    if p.exists():
        return json.loads(p.read_text())["work"]
    return None


def round_work(records, stats):
    """node visits + edge visits per round (assign edges + resolve lower edges)."""
    return [int(r[2]) + int(a) + int(b) for r, (a, b) in zip(records, stats)]


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def build_graph(hc, cfg):
    if cfg["kind"] == "grid":
        return hc.grid_graph(cfg["rows"], cfg["cols"])
    if cfg["kind"] == "er":
        return hc.er_graph(cfg["n"], cfg["avg_degree"], cfg["seed"])
    return hc.rmat_graph(cfg["scale"], cfg["edgefactor"], cfg["seed"])


def gen_edges(hc, cfg):
    """The config's pair list generated on the current GPU."""
    from paper_1912_01478_b200 import graph as G

    if cfg["kind"] == "grid":
        return G.gen_grid_edges(cfg["rows"], cfg["cols"]), cfg["rows"] * cfg["cols"]
    if cfg["kind"] == "er":
        return G.gen_er_edges(cfg["n"], cfg["n"] * cfg["avg_degree"] // 2, cfg["seed"]), cfg["n"]
    return G.gen_rmat_edges(cfg["scale"], cfg["edgefactor"], cfg["seed"]), 1 << cfg["scale"]


def run_distributed(args, cfg):
    """N > 1: one rank per GPU, 1D edge-balanced vertex partition of the same
    graph (strong scaling).  Every rank generates the pair list, cuts the same
    bounds and builds ONLY its own CSR rows (multigpu.build_shard); the solve
    is the device-resident peer-memory solve (multigpu.MgSolver: one
    persistent kernel per GPU, boundary words stored into the peers' replicas
    over NVLink, cross-GPU mailbox barriers).  No fallback: a refused peer
    mapping is an error."""
    import torch
    import torch.distributed as dist

    import paper_1912_01478_b200 as hc
    from paper_1912_01478_b200.multigpu import CsrShard, MgSolver, build_shard, edge_partition_bounds

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:  # test knob: every rank on cuda:0 (gloo; kernels time-slice)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.share_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    edges, n = gen_edges(hc, cfg)
    bounds, raw = edge_partition_bounds(edges, n, world)
    shard = build_shard(edges, n, bounds, rank, raw)
    del edges, raw
    torch.cuda.empty_cache()
    solver = MgSolver(shard)
    und = shard.num_undirected_edges
    hcfg = hc.HybridConfig(mode=args.mode)
    thr = hc.threshold_count(hcfg, n)
    exchange = ("peer memory: one persistent kernel per GPU; boundary state words reach the ranks that read "
                "them by NVLink stores (mirrored at write time, or boundary-zone copies per phase, chosen per "
                "round); cross-GPU mailbox barriers carry the (|W|, conflicts) all-reduce")

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        solver.run(args.mode, thr)
    stream = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    rounds = 0
    torch.cuda.synchronize()
    dist.barrier()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            starts[i].record(stream)
            rounds, _ = solver.run(args.mode, thr)
            stops[i].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    cdev = torch.device("cpu") if args.share_gpu else dev
    t = torch.tensor([float(sum(step_ms))], device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = und * args.steps / (total_ms / 1e3)

    # correctness of the timed path: the global coloring is valid
    colors = solver.gather_colors()
    valid = solver.verify(colors) == 0

    # e2e: every rank uploads ITS rows from pinned host memory (one CSR in
    # total), solves, gathers the colors and copies them back
    host = shard.to_host()
    shard_bytes = 8 * host[0].numel() + 8 * host[1].numel()
    e2e_total = 0.0
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        solver.replace_shard(CsrShard.upload(host, shard, dev))  # the peer mapping is made once
        solver.run(args.mode, thr)
        solver.gather_colors().cpu()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_total += (time.perf_counter() - t0) * 1e3
    t = torch.tensor([e2e_total, float(shard_bytes), float(shard.nbytes())], device=cdev)
    tm = t.clone()
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    e2e_total = float(tm[0].item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (BASELINE generator spec, SURVEY.md Appendix C), built on the GPUs (per-rank shards)",
            "config": {"workload": DESCRIPTIONS[args.config], "name": args.config, "mode": args.mode,
                       "num_nodes": n, "num_undirected_edges": und, "rounds": rounds,
                       "parallelism": f"1d-partition x{world} (edge-balanced, per-rank CSR shards)",
                       "exchange": exchange, "valid": valid, "bounds": bounds,
                       "csr_shard_bytes_max": int(tm[2].item()), "csr_bytes_total": int(t[2].item()),
                       "l2": "flushed between timed steps (512 MiB write)"},
            "clocks": clk.summary(),
            # bucket sort (3) + copy_totals + fill_od + narrow + delta + boundary flags + the solve kernel
            "gpu_launches": 9 * args.steps,
            "e2e": {"value": und * args.steps / (e2e_total / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(t[1].item()), "d2h_bytes_per_step": 8 * n},
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    dist.destroy_process_group()
    return 0


def measure(args, name: str, steps: int, warmup: int, *, e2e_steps: int, mode_reps: int,
            cpu_budget: float) -> dict:
    """One config on this GPU: the timed hybrid steps, the GPU's own data /
    topology modes, e2e through color_graph on pinned host buffers, the
    roofline of the solve under both byte models, and the reference's CPU
    solve on the host cores (a full solve when it fits cpu_budget)."""
    import ctypes

    import torch

    import paper_1912_01478_b200 as hc
    from paper_1912_01478_b200 import _lib

    cfg = CONFIGS[name]
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = build_graph(hc, cfg)
    torch.cuda.synchronize()
    n, und, m = dg.num_nodes, dg.num_undirected_edges, dg.num_edges
    hcfg = hc.HybridConfig(mode=args.mode)
    thr = hc.threshold_count(hcfg, n)
    solver = hc.Solver(dg)
    L = _lib.load()

    # one instrumented solve (outside the timed region) for the byte models
    stats = torch.zeros((solver.max_rec, 2), dtype=torch.int64, device=dev)
    rounds = ctypes.c_int64(0)
    _lib.check(L.hc_solve_stats(dg.row_offsets.data_ptr(), _lib.ptr(dg.col_indices), n, m,
                                _lib.MODE_CODES[args.mode], thr, solver.colors.data_ptr(),
                                solver.rec.data_ptr(), solver.max_rec, ctypes.byref(rounds),
                                stats.data_ptr(), solver.ws.data_ptr(), solver.ws.numel(),
                                _lib.stream_handle()))
    R = int(rounds.value)
    recs = solver.rec[:R].cpu().numpy()
    st = stats[:R].cpu().numpy()
    b_survey = survey_bytes(recs, st, n)
    b_own = own_bytes(recs, st, n, m)

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(warmup):
        solver.run(args.mode, thr, fetch_records=False)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    stream = torch.cuda.current_stream()
    # bucket count/scan/scatter + copy_totals + fill_od + narrow_offsets and
    # delta_columns (int32-offset graphs) + fbx memset + solve_kernel (see the ncu launch list)
    narrow = m < (1 << 31) - 1
    launches_per_step = 3 + 1 + 1 + (1 if narrow else 0) + (1 if narrow and m else 0) + 1
    torch.cuda.synchronize()
    with Clocks(dev.index) as clk:
        for i in range(steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            starts[i].record(stream)
            rc = L.hc_solve(dg.row_offsets.data_ptr(), _lib.ptr(dg.col_indices), n, m,
                            _lib.MODE_CODES[args.mode], thr, solver.colors.data_ptr(),
                            solver.rec.data_ptr(), solver.max_rec, ctypes.byref(rounds),
                            solver.ws.data_ptr(), solver.ws.numel(), _lib.stream_handle(stream))
            stops[i].record(stream)
            _lib.check(rc)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    total_ms = float(sum(step_ms))
    ms_per_step = total_ms / steps
    value = und * steps / (total_ms / 1e3)

    # hybrid vs the GPU's own pure data / topology modes
    modes = {}
    if not args.skip_modes:
        for mode in ("hybrid", "data", "topo"):
            ts = []
            for _ in range(mode_reps):
                flush.zero_()
                ts.append(solver.run(mode, thr, fetch_records=False).seconds)
            modes[mode] = {"ms": min(ts) * 1e3, "und_edges_per_s": und / min(ts)}
        # the paper's Plain data-driven baseline (IrGL worklist,
        # atomic pushes, no ordering): hc_solve_plain, data mode
        ts = []
        for _ in range(mode_reps):
            flush.zero_()
            ts.append(solver.run("data", thr, fetch_records=False, plain=True).seconds)
        modes["plain_data"] = {"ms": min(ts) * 1e3, "und_edges_per_s": und / min(ts),
                               "what": "data-driven, warp-aggregated atomic pushes into unordered lists "
                                       "(paper's IrGL Plain; bench-only)"}
        modes["hybrid_speedup_vs_data"] = modes["data"]["ms"] / modes["hybrid"]["ms"]
        modes["hybrid_speedup_vs_topo"] = modes["topo"]["ms"] / modes["hybrid"]["ms"]
        modes["hybrid_speedup_vs_plain_data"] = modes["plain_data"]["ms"] / modes["hybrid"]["ms"]
    del solver

    # e2e through the public API on pinned host buffers
    host = dg.to_host()
    pinned = hc.CsrGraph.pinned(host)
    e2e_ms = []
    for i in range(1 + e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        colors, rep = hc.color_graph(pinned, hcfg)
        torch.cuda.synchronize()
        if i >= 1:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert rep.valid
        del colors, rep
    del pinned
    e2e_total = float(sum(e2e_ms))

    hbm, peak_kind = peaks()
    achieved = b_survey / (ms_per_step / 1e3) / 1e9
    own = b_own / (ms_per_step / 1e3) / 1e9
    traffic = measured_traffic(name)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic["bytes"] if traffic else None, "peak_kind": peak_kind,
            "kernel": "solve_kernel (+ bin preprocessing, whole hc_solve step)",
            "model": "SURVEY.md §8(d) per-round bytes (scan-based assign, 8 B packed (t,T))",
            "algorithmic_bytes_per_launch": b_survey,
            "own_model": {"bytes_per_launch": b_own, "achieved": own, "frac": own / hbm,
                          "model": "bitmap assign + lower-neighbour resolve + per-solve winner pushes "
                                   "(bench.py own_bytes)"}}
    if traffic:
        roof["dram"] = {"bytes_per_launch": traffic["bytes"], "ncu_ms": traffic["ns"] / 1e6,
                        "achieved": traffic["bytes"] / (traffic["ns"] / 1e9) / 1e9 if traffic["ns"] else None,
                        "frac": traffic["bytes"] / (traffic["ns"] / 1e9) / 1e9 / hbm if traffic["ns"] else None,
                        "l2_hit_pct": traffic.get("l2_hit_pct"),
                        "source": f"profiles/r02_{name}_traffic.csv (ncu, cold L2, serialised)"}
    out = {
        "workload": DESCRIPTIONS[name], "value": value, "unit": UNIT, "ms_per_step": ms_per_step,
        "steps": steps, "warmup": warmup, "num_nodes": n, "num_undirected_edges": und, "rounds": R,
        "sum_wl_in": int(recs[:, 2].sum()), "roofline": roof, "clocks": clk.summary(),
        "gpu_launches": launches_per_step * steps, "modes": modes,
        "e2e": {"value": und * e2e_steps / (e2e_total / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": 8 * (n + 1) + 8 * m, "d2h_bytes_per_step": 8 * n + 48 * R,
                "ms_per_step": e2e_total / e2e_steps},
        "step_ms": step_ms,
    }
    if not args.skip_cpu:
        try:
            ref = reference_module()
            warm_reference(ref)
            g = ref.CsrGraph(host.num_nodes, host.num_edges, host.row_offsets, host.col_indices)
            out["cpu_baseline"] = cpu_sample(ref, g, cpu_budget, round_work(recs, st))
            del g
        except Exception as exc:  # reported, not fatal
            out["cpu_baseline"] = {"value": None, "unavailable": repr(exc)}
    del host, dg, flush
    torch.cuda.empty_cache()
    return out


def run_ours(args, cfg):
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))  # N > 1: run_distributed
    torch.cuda.set_device(local)
    head = measure(args, args.config, args.steps, args.warmup, e2e_steps=args.steps, mode_reps=3,
                   cpu_budget=args.cpu_budget)
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (BASELINE generator spec, SURVEY.md Appendix C), built on the GPU",
        "config": {"workload": head["workload"], "name": args.config, "mode": args.mode,
                   "num_nodes": head["num_nodes"], "num_undirected_edges": head["num_undirected_edges"],
                   "rounds": head["rounds"], "sum_wl_in": head["sum_wl_in"],
                   "l2": "flushed between timed steps (512 MiB write)", "parallelism": "single-gpu"},
        "roofline": head["roofline"], "clocks": head["clocks"], "gpu_launches": head["gpu_launches"],
        "modes": head["modes"], "e2e": head["e2e"], "step_ms": head["step_ms"],
    }
    if "cpu_baseline" in head:
        line["cpu_baseline"] = head["cpu_baseline"]
    if args.all_configs:
        # the other BASELINE configs (parity cases of the headline, reported
        # like compare_backends.py:53-67: every mode, e2e, roofline, CPU solve)
        line["configs"] = {}
        for name in CONFIGS:
            if name == args.config:
                continue
            line["configs"][name] = measure(args, name, min(args.steps, 5), 3, e2e_steps=3,
                                            mode_reps=2 if name == "rmat26" else 3,
                                            cpu_budget=args.cpu_budget_configs)
            line["gpu_launches"] += line["configs"][name]["gpu_launches"]
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="grid4096")
    ap.add_argument("--mode", choices=("hybrid", "data", "topo"), default="hybrid")
    ap.add_argument("--skip-modes", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of reference CPU solve for the headline config (grid: extrapolated)")
    ap.add_argument("--cpu-budget-configs", type=float, default=60.0,
                    help="the same for the other configs (full reference solves of C1/C3/C4 fit)")
    ap.add_argument("--all-configs", dest="all_configs", action="store_true", default=True,
                    help="also measure the other BASELINE configs under the line's 'configs' key (default)")
    ap.add_argument("--headline-only", dest="all_configs", action="store_false")
    ap.add_argument("--share-gpu", action="store_true",
                    help="N>1 test knob: all ranks on cuda:0 over gloo (correctness only, not a bench)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_distributed(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
