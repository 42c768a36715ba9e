"""Reference records for grids, pinning the per-round closed form
(tests/conftest.py:grid_records) that the -m gpu suite applies to the full
4096^2 headline grid (configs[1]) in every mode.

Run in the build container (needs oracle/_ref, the reference package built by
oracle/build_ref.sh, and /root/reference/pkg/tests/conftest.py's grid builder):

    python tests/golden/make_grid_golden.py

For every shape it builds the grid with the reference's own test builder
(conftest.py:30-41 -> build_csr) and records the reference's color_graph
(driver.py:122-176, Cython/OpenMP backend) per mode x threshold: the int64
(topo?, wl_in, wl_out, conflicts) records and the colors' sha256.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import load_reference  # noqa: E402

SHAPES = [(1, 1), (1, 2), (2, 1), (1, 9), (9, 1), (2, 2), (3, 3), (5, 7), (7, 5), (33, 17), (17, 33),
          (300, 41), (41, 300), (2, 1000), (64, 64), (128, 128), (128, 64), (64, 128), (256, 256),
          (512, 512)]
SETTINGS = [("data", 0.6), ("topo", 0.6), ("hybrid", 0.6), ("hybrid", 0.3), ("hybrid", 0.0), ("hybrid", 1.0)]


def main():
    ref, conf = load_reference()
    workers = os.cpu_count() or 1
    out = {"shapes": np.array(SHAPES, np.int64),
           "settings": np.array([f"{m}:{t}" for m, t in SETTINGS])}
    for r, c in SHAPES:
        g = conf.grid_graph(r, c)
        for mode, thr in SETTINGS:
            colors, rep = ref.color_graph(g, ref.HybridConfig(mode=mode, threshold_fraction=thr,
                                                              workers=workers))
            rec = np.array([[int(x.mode_used == "topo"), x.worklist_size_in, x.worklist_size_out, x.conflicts]
                            for x in rep.per_round], np.int64).reshape(-1, 4)
            key = f"{r}x{c}__{mode}__{thr}"
            out[key + "__rec"] = rec
            out[key + "__colors_sha"] = np.array(hashlib.sha256(np.asarray(colors, "<i8").tobytes()).hexdigest())
        print(f"{r}x{c}: {len(rec)} rounds", flush=True)
    np.savez_compressed(HERE / "grids.npz", **out)


if __name__ == "__main__":
    main()
