"""`python -m paper_1912_01478_b200` -- the reference's command-line front end
(pkg/src/hybridcolor/cli.py) over the GPU path.

Subcommands, options, stdout layouts, report files and exit codes follow the
reference: 0 success, 1 invalid coloring / unequal benchmark work, 2 usage or
input error, 3 I/O error on an output path (cli.py:1-22, 157-164).  A graph
argument (.mtx or .npz cache) is loaded straight into HBM
(ingest.load_graph_device: device MatrixMarket parse + device CSR build), so
`stats` and `color` never walk the edges on the host.
"""

from __future__ import annotations

import argparse
import io
import json
import sys
from pathlib import Path

from . import __version__
from ._backend import backend_name
from .driver import MODES, HybridConfig, color_graph
from .ingest import MatrixMarketError, degree_stats, load_graph_device
from .pushbench import BenchConfig, collect_deactivations, detect_crossovers, run_push_bench, write_tti_csv

EXIT_OK, EXIT_INVALID_COLORING, EXIT_USAGE, EXIT_IO = 0, 1, 2, 3
GRAPH_HELP = "path to .mtx file or .npz CSR cache"


class OutputError(Exception):
    """An output path could not be written (exit code 3)."""


def _write_text(path: str, text: str) -> None:
    try:
        Path(path).write_text(text, encoding="utf-8")
    except OSError as exc:
        raise OutputError(f"cannot write {path}: {exc}") from exc


def _stats(args) -> int:
    s = degree_stats(load_graph_device(args.graph))
    if args.format == "json":
        print(json.dumps(s.__dict__, indent=2, sort_keys=True))
    else:
        print(f"{s.num_nodes} nodes, {s.num_undirected_edges} edges, "
              f"δ {s.min_degree}/{s.median_degree}/{s.max_degree}")
    return EXIT_OK


def _color(args) -> int:
    cfg = HybridConfig(threshold_fraction=args.threshold, mode=args.mode, workers=args.workers)
    _, report = color_graph(load_graph_device(args.graph), cfg, graph_name=Path(args.graph).stem)
    if args.format == "json":
        print(report.to_json())
    elif args.format == "csv":
        report.write_round_csv(sys.stdout)
    else:
        summary = [
            f"graph: {report.graph_name} ({report.num_nodes} nodes, {report.num_undirected_edges} undirected edges)",
            f"mode: {cfg.mode}  threshold: {cfg.threshold_fraction}  workers: {cfg.workers}  "
            f"backend: {backend_name()}",
            f"colors_used: {report.colors_used}",
            f"total_rounds: {report.total_rounds}",
            f"valid: {str(report.valid).lower()}",
            f"total_micros: {report.total_seconds * 1e6:.1f}",
            report.rows_table(),
        ]
        print("\n".join(summary))
    if args.out:
        _write_text(args.out, report.to_json() + "\n")
    return EXIT_OK if report.valid else EXIT_INVALID_COLORING


def _bench(args) -> int:
    graph = load_graph_device(args.graph)
    series = [run_push_bench(graph, BenchConfig(batch_size=args.batch, variant=v, repetitions=args.reps),
                             workers=args.workers) for v in ("push_wl", "push_nowl")]
    wl, nowl = (collect_deactivations(graph, BenchConfig(batch_size=args.batch, variant=v, repetitions=1),
                                      workers=args.workers) for v in ("push_wl", "push_nowl"))
    same = len(wl) == len(nowl) and all((a == b).all() for a, b in zip(wl, nowl))
    buf = io.StringIO()
    write_tti_csv(buf, series)
    _write_text(args.out, buf.getvalue())
    print(f"wrote {args.out} ({len(series)} variants x {len(series[0].per_iteration)} iterations)")
    print(f"deactivation sets identical across variants: {'yes' if same else 'NO'}")
    cross = detect_crossovers(series[0], series[1])
    print("crossovers: " + (" ".join(str(c) for c in cross) if cross else "none"))
    return EXIT_OK if same else EXIT_INVALID_COLORING


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="hybridcolor",
                                description="Worklist-persistent parallel graph coloring and kernel "
                                            "micro-benchmarks (B200 / CUDA)")
    p.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = p.add_subparsers(dest="subcommand", required=True)

    s = sub.add_parser("stats", help="node/edge counts and degree statistics")
    s.add_argument("graph", help=GRAPH_HELP)
    s.add_argument("--format", choices=["table", "json"], default="table")
    s.set_defaults(handler=_stats)

    c = sub.add_parser("color", help="color the graph and report the result")
    c.add_argument("graph", help=GRAPH_HELP)
    c.add_argument("--mode", choices=list(MODES), default="hybrid")
    c.add_argument("--threshold", type=float, default=0.6,
                   help="worklist-size fraction above which hybrid goes topology-driven")
    c.add_argument("--workers", type=int, default=1)
    c.add_argument("--format", choices=["table", "json", "csv"], default="table")
    c.add_argument("--out", metavar="PATH", help="write the JSON run report here")
    c.set_defaults(handler=_color)

    b = sub.add_parser("bench", help="run the push_wl / push_nowl micro-benchmark pair")
    b.add_argument("graph", help=GRAPH_HELP)
    b.add_argument("--batch", type=int, default=1000, help="active nodes deactivated per iteration")
    b.add_argument("--reps", type=int, default=10, help="runs to average TTI over")
    b.add_argument("--workers", type=int, default=1)
    b.add_argument("--out", metavar="PATH", required=True, help="TTI CSV output path")
    b.set_defaults(handler=_bench)
    return p


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    checks = (("threshold", lambda v: 0.0 <= v <= 1.0, "--threshold must be in [0, 1], got {}"),
              ("workers", lambda v: v >= 1, "--workers must be >= 1"),
              ("batch", lambda v: v >= 1, "--batch must be >= 1"),
              ("reps", lambda v: v >= 1, "--reps must be >= 1"))
    for name, ok, msg in checks:
        v = getattr(args, name, None)
        if v is not None and not ok(v):
            parser.error(msg.format(v))
    try:
        return args.handler(args)
    except OutputError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (FileNotFoundError, MatrixMarketError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE


def entrypoint() -> None:
    sys.exit(main())
