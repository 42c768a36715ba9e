"""Shared fixtures: golden corpora produced by the REFERENCE
(tests/golden/make_golden.py) and graph helpers.

Markers: `gpu` -- needs a CUDA device (run on the B200 via gpurun);
everything else runs on CPU in the build container.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

MODES = ("data", "topo", "hybrid")
THRESHOLDS = (0.0, 0.3, 0.6, 1.0)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running full-size parity checks")


@dataclass
class GoldenGraph:
    name: str
    n: int
    ro: np.ndarray
    ci: np.ndarray
    colors: np.ndarray
    colors_used: int
    records: dict  # (mode, thr) -> int64[rounds, 4] (topo, wl_in, wl_out, conflicts)


def load_corpus() -> list[GoldenGraph]:
    z = np.load(GOLDEN / "corpus.npz")
    out = []
    ro_off, ci_off, col_off, rec_off = z["ro_off"], z["ci_off"], z["colors_off"], z["rec_off"]
    r = 0
    for i, name in enumerate(z["names"].tolist()):
        recs = {}
        for mode in MODES:
            for thr in THRESHOLDS:
                recs[(mode, thr)] = z["rec"][rec_off[r]:rec_off[r + 1]]
                r += 1
        out.append(GoldenGraph(
            name=name, n=int(z["n"][i]),
            ro=z["ro"][ro_off[i]:ro_off[i + 1]].astype(np.int64),
            ci=z["ci"][ci_off[i]:ci_off[i + 1]].astype(np.int64),
            colors=z["colors"][col_off[i]:col_off[i + 1]].astype(np.int64),
            colors_used=int(z["colors_used"][i]), records=recs))
    return out


def load_configs() -> dict:
    z = np.load(GOLDEN / "configs.npz")
    cases = {}
    for key in z["cases"].tolist():
        cases[key] = {
            "n": int(z[f"{key}__n"]), "m": int(z[f"{key}__m"]), "sha": str(z[f"{key}__sha"]),
            "maxdeg": int(z[f"{key}__maxdeg"]), "colors": z[f"{key}__colors"].astype(np.int64),
            "colors_used": int(z[f"{key}__colors_used"]), "rounds": int(z[f"{key}__rounds"]),
            "rec": {m: z[f"{key}__{m}__rec"] for m in MODES},
        }
    return cases


CONFIG_SPECS = {
    "rmat16": ("rmat", dict(scale=16, edgefactor=16, seed=0)),
    "rmat14s7": ("rmat", dict(scale=14, edgefactor=16, seed=7)),
    "grid256": ("grid", dict(rows=256, cols=256)),
    "grid64x96": ("grid", dict(rows=64, cols=96)),
    "er16": ("er", dict(n=1 << 16, m=(1 << 16) * 16, seed=0)),
}


@pytest.fixture(scope="session")
def corpus():
    return load_corpus()


@pytest.fixture(scope="session")
def configs():
    return load_configs()


def csr_sha(ro, ci) -> str:
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ro, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int64).tobytes())
    return h.hexdigest()


def grid_closed_form(rows: int, cols: int):
    """Checkerboard colors 1+((i+j) mod 2), rounds ceil((r+c)/2)."""
    i, j = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    return (1 + ((i + j) % 2)).ravel().astype(np.int64), -(-(rows + cols) // 2)


def grid_records(rows: int, cols: int, mode: str = "hybrid", threshold_fraction: float = 0.6) -> np.ndarray:
    """Closed form of every per-round record (topo?, wl_in, wl_out, conflicts)
    of color_graph on the rows x cols 4-neighbour grid (ids i*cols+j).

    Lower-id neighbours of (i,j) are (i-1,j) and (i,j-1), both on antidiagonal
    d-1 (d = i+j).  Round 1 everyone takes color 1 and only node 0 wins.  In
    round t >= 2 antidiagonal 2t-3 (its lower neighbours committed with color 1)
    takes 2 and wins, antidiagonal 2t-2 takes 1 and wins (its lower neighbours
    hold 2), every later antidiagonal takes 1 and loses to its lower
    neighbours.  So after round t antidiagonals 0..2t-2 are final:
      wl_out(t) = n - F(2t-2),  wl_in(t) = wl_out(t-1) (wl_in(1) = n),
      conflicts(t) = m_und - S(2t-2),
    F(k) / S(k) = nodes / lower-neighbour edges on antidiagonals <= k.  The mode
    is driver.py:147-152 with thr = ceil(H*n) (driver.py:138).  Pinned against
    the reference's own records (tests/golden/grids.npz, make_grid_golden.py)."""
    import math

    n = rows * cols
    if n == 0:
        return np.zeros((0, 4), np.int64)
    d = np.arange(rows + cols - 1, dtype=np.int64)
    cnt = np.minimum(d, rows - 1) - np.maximum(0, d - cols + 1) + 1
    low = 2 * cnt - (d <= cols - 1) - (d <= rows - 1)  # i>0 nodes + j>0 nodes
    F = np.concatenate(([0], np.cumsum(cnt)))            # F[k+1] = nodes on diagonals <= k
    S = np.concatenate(([0], np.cumsum(low)))
    m_und = int(S[-1])
    R = -(-(rows + cols) // 2)
    thr = math.ceil(threshold_fraction * n)
    out = np.zeros((R, 4), np.int64)
    for t in range(1, R + 1):
        k_out = min(2 * t - 2, rows + cols - 2)
        wl_in = n if t == 1 else n - int(F[min(2 * t - 4, rows + cols - 2) + 1])
        topo = mode == "topo" or (mode == "hybrid" and wl_in > thr)
        out[t - 1] = (int(topo), wl_in, n - int(F[k_out + 1]), m_und - int(S[k_out + 1]))
    return out
