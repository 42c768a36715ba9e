"""B200-native hybrid IPGC (arXiv 1912.01478) -- drop-in for `hybridcolor`'s
coloring path.

The public names mirror the reference package's solve path
(pkg/src/hybridcolor/__init__.py:11-69): `color_graph`, `HybridConfig`,
`RunReport`, `RoundRecord`, `colors_used`, `verify_coloring`, `CsrGraph`,
`EdgeList`, `build_csr`, the per-round `ColorState` / `Worklist` /
`data_driven_iteration` / `topology_driven_iteration` / `assign_color` /
`resolve_conflicts` / `mex_positive`, and the kernel-module
registry (`get_kernels`, `available_backends`, `backend_name`).  Everything
computes on the GPU through libhcb.so (include/hcb.h); there is no CPU path.
"""

from ._backend import available_backends, backend_name, get_kernels
from .coloring import (
    ColorState,
    RoundOutcome,
    assign_color,
    data_driven_iteration,
    mex_positive,
    resolve_conflicts,
    topology_driven_iteration,
)
from .driver import (
    MODES,
    HybridConfig,
    RoundRecord,
    RunReport,
    PlannedSolver,
    Solver,
    color_graph,
    colors_used,
    threshold_count,
    verify_coloring,
)
from .graph import (
    CsrGraph,
    DeviceCsr,
    EdgeList,
    build_csr,
    build_csr_device,
    er_graph,
    gen_er_edges,
    gen_grid_edges,
    gen_rmat_edges,
    grid_graph,
    rmat_graph,
    synthetic,
)
from .ingest import (
    DegreeStats,
    MatrixMarketError,
    degree_stats,
    load_csr_cache,
    load_graph,
    load_graph_device,
    parse_matrix_market,
    save_csr_cache,
)
from .pushbench import (
    BenchConfig,
    TtiRecord,
    TtiSeries,
    collect_deactivations,
    detect_crossovers,
    expected_iterations,
    run_push_bench,
    write_tti_csv,
)
from .worklist import Worklist, init_full

__version__ = "0.1.0"

__all__ = [
    "available_backends", "backend_name", "get_kernels",
    "ColorState", "RoundOutcome", "assign_color", "data_driven_iteration", "mex_positive",
    "resolve_conflicts", "topology_driven_iteration",
    "MODES", "HybridConfig", "RoundRecord", "RunReport", "Solver", "PlannedSolver",
    "color_graph", "colors_used", "threshold_count", "verify_coloring",
    "CsrGraph", "DeviceCsr", "EdgeList", "build_csr", "build_csr_device",
    "er_graph", "gen_er_edges", "gen_grid_edges", "gen_rmat_edges", "grid_graph",
    "rmat_graph", "synthetic",
    "DegreeStats", "MatrixMarketError", "degree_stats", "load_csr_cache", "load_graph",
    "load_graph_device", "parse_matrix_market", "save_csr_cache",
    "BenchConfig", "TtiRecord", "TtiSeries", "collect_deactivations", "detect_crossovers",
    "expected_iterations", "run_push_bench", "write_tti_csv",
    "Worklist", "init_full",
    "__version__",
]
