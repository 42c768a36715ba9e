"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `hybridcolor` (oracle/_ref when built by
oracle/build_ref.sh -- the reference's own Cython backend -- else the source
tree /root/reference/pkg/src with its numpy backend; both are bitwise equal per
pkg/tests/test_backends.py:36-69) and the reference's own test graph builders
(pkg/tests/conftest.py:18-59), runs `color_graph` (driver.py:122-176) and
records what the reference produced.  Nothing at test time reads
/root/reference: the tests only read the .npz files written here.

Fixtures:
  corpus.npz   every graph of the reference's seeded test corpora
               (test_acceptance.py:58-91 seed 20260810; test_coloring.py:195-209
               seed 23; test_driver.py:51-73 seeds 17, 29; test_backends.py:36-69
               seeds 101-105; test_acceptance.py:187-203 seed 55; the small
               named graphs) with CSR, final colors and per-round records for
               every mode x threshold the reference tests sweep.
  configs.npz  BASELINE config C1 (RMAT-16 ef16 seed 0) plus small shapes of the
               other configs (grid 256x256 and 64x96, ER 2^16 d32 seed 0,
               RMAT-14 seed 7): CSR sha256, colors, records per mode.
"""

from __future__ import annotations

import hashlib
import importlib.util
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_PKG = Path("/root/reference/pkg")

sys.path.insert(0, str(REPO))
from oracle import oracle as O  # noqa: E402  (generators only; pinned separately)


def load_reference():
    ref = O.reference_module()
    if ref is None:
        sys.path.insert(0, str(REF_PKG / "src"))
        import hybridcolor as ref  # type: ignore
    spec = importlib.util.spec_from_file_location("ref_conftest", REF_PKG / "tests" / "conftest.py")
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    return ref, conf


MODES = ("data", "topo", "hybrid")
THRESHOLDS = (0.0, 0.3, 0.6, 1.0)


def corpus(ref, conf):
    """The reference's seeded corpora, rebuilt with its own builders."""
    graphs = []
    # acceptance corpus, test_acceptance.py:58-91
    rng = np.random.default_rng(20260810)
    er_plan = [
        (10, (0.05, 0.15, 0.3, 0.6)), (20, (0.05, 0.15, 0.3, 0.6)), (50, (0.05, 0.15, 0.3, 0.6)),
        (100, (0.01, 0.05, 0.1)), (200, (0.01, 0.05, 0.1)), (500, (0.002, 0.01, 0.02)),
        (1000, (0.002, 0.01, 0.02)), (2000, (0.001, 0.005)),
    ]
    for n, ps in er_plan:
        for p in ps:
            for _ in range(6):
                graphs.append((f"acc_er{n}_p{p}", conf.er_graph(rng, n, p)))
    for r in range(2, 7):
        for c in range(2, 8):
            graphs.append((f"acc_grid{r}x{c}", conf.grid_graph(r, c)))
    for k in (1, 2, 3, 5, 10, 50, 100, 500):
        graphs.append((f"acc_star{k}", conf.star_graph(k)))
    for k in range(1, 9):
        graphs.append((f"acc_k{k}", conf.clique_graph(k)))
    for n in (1, 5, 17):
        graphs.append((f"acc_isolated{n}", conf.csr_from_edges(n, [])))
    for _ in range(5):
        n = int(rng.integers(20, 60))
        m = int(rng.integers(5, 40))
        edges = np.column_stack([rng.integers(0, n // 2, m), rng.integers(0, n // 2, m)])
        graphs.append((f"acc_mixed{n}", ref.build_csr(ref.EdgeList(n, edges))))
    # test_coloring.py:195-209 (seed 23)
    rng = np.random.default_rng(23)
    for i in range(25):
        graphs.append((f"col23_{i}", conf.er_graph(rng, int(rng.integers(1, 60)), float(rng.choice([0.05, 0.15, 0.4])))))
    # test_driver.py:51-64 (seed 17) and 66-73 (seed 29)
    rng = np.random.default_rng(17)
    for i in range(10):
        graphs.append((f"drv17_{i}", conf.er_graph(rng, int(rng.integers(2, 120)), 0.08)))
    rng = np.random.default_rng(29)
    for i in range(15):
        graphs.append((f"drv29_{i}", conf.er_graph(rng, int(rng.integers(1, 80)), 0.1)))
    # test_backends.py:36-57 (seed 101), 58-66 (102), 72-91 (104, 105)
    rng = np.random.default_rng(101)
    for i in range(20):
        graphs.append((f"bk101_{i}", conf.er_graph(rng, int(rng.integers(2, 300)), float(rng.choice([0.01, 0.05, 0.2])))))
    rng = np.random.default_rng(102)
    graphs.append(("bk102", conf.er_graph(rng, 400, 0.02)))
    rng = np.random.default_rng(104)
    for i in range(8):
        graphs.append((f"bk104_{i}", conf.er_graph(rng, 500, 0.02)))
    rng = np.random.default_rng(105)
    graphs.append(("bk105", conf.er_graph(rng, 300, 0.05)))
    # test_acceptance.py:187-203 (seed 55)
    rng = np.random.default_rng(55)
    for i in range(30):
        graphs.append((f"acc55_{i}", conf.er_graph(rng, int(rng.integers(1, 400)), 0.03)))
    # named shapes used across the reference tests
    for k in range(1, 9):
        graphs.append((f"path{k}", conf.path_graph(k)))
    for k in range(3, 21):
        graphs.append((f"cycle{k}", conf.cycle_graph(k)))
    graphs.append(("empty0", conf.csr_from_edges(0, [])))
    return graphs


def run_all(ref, g):
    """color_graph under every mode x threshold; returns colors + stacked records."""
    out = {}
    base = None
    for mode in MODES:
        for thr in THRESHOLDS:
            colors, rep = ref.color_graph(g, ref.HybridConfig(mode=mode, threshold_fraction=thr))
            recs = np.array(
                [[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                 for r in rep.per_round], dtype=np.int64).reshape(-1, 4)
            if base is None:
                base = colors
            assert np.array_equal(base, colors)  # the reference's own mode-equivalence
            out[(mode, thr)] = (colors, recs, rep.colors_used, rep.valid)
    return out


def make_corpus(ref, conf):
    graphs = corpus(ref, conf)
    names, ns, ro_all, ci_all, col_all, rec_all = [], [], [], [], [], []
    ro_off, ci_off, col_off, rec_off = [0], [0], [0], [0]
    colors_used = []
    for name, g in graphs:
        res = run_all(ref, g)
        names.append(name)
        ns.append(g.num_nodes)
        ro_all.append(g.row_offsets); ro_off.append(ro_off[-1] + len(g.row_offsets))
        ci_all.append(g.col_indices); ci_off.append(ci_off[-1] + len(g.col_indices))
        colors = res[("hybrid", 0.6)][0]
        col_all.append(colors); col_off.append(col_off[-1] + len(colors))
        colors_used.append(res[("hybrid", 0.6)][2])
        # records per (mode, thr) in MODES x THRESHOLDS order
        for mode in MODES:
            for thr in THRESHOLDS:
                recs = res[(mode, thr)][1]
                rec_all.append(recs); rec_off.append(rec_off[-1] + len(recs))
    np.savez_compressed(
        HERE / "corpus.npz",
        names=np.array(names), n=np.array(ns, dtype=np.int64),
        ro=np.concatenate(ro_all), ro_off=np.array(ro_off, dtype=np.int64),
        ci=np.concatenate(ci_all).astype(np.int32), ci_off=np.array(ci_off, dtype=np.int64),
        colors=np.concatenate(col_all).astype(np.int32), colors_off=np.array(col_off, dtype=np.int64),
        rec=np.concatenate(rec_all).astype(np.int64), rec_off=np.array(rec_off, dtype=np.int64),
        colors_used=np.array(colors_used, dtype=np.int64),
        modes=np.array(MODES), thresholds=np.array(THRESHOLDS),
    )
    print(f"corpus.npz: {len(graphs)} graphs")


def csr_sha(ro, ci) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ro, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int64).tobytes())
    return h.hexdigest()


def make_configs(ref):
    cases = {
        # BASELINE.json configs[0]: RMAT scale-16 edgefactor-16, seed 0 (full size)
        "rmat16": ("rmat", dict(scale=16, edgefactor=16, seed=0)),
        "rmat14s7": ("rmat", dict(scale=14, edgefactor=16, seed=7)),
        # configs[1] shape at reduced size (full 4096^2 is pinned by closed form)
        "grid256": ("grid", dict(rows=256, cols=256)),
        "grid64x96": ("grid", dict(rows=64, cols=96)),
        # configs[3] shape at reduced size: n=2^16, avg degree 32
        "er16": ("er", dict(n=1 << 16, m=(1 << 16) * 16, seed=0)),
    }
    payload = {}
    for key, (kind, kw) in cases.items():
        if kind == "rmat":
            n = 1 << kw["scale"]
            e = O.np_gen_rmat(kw["scale"], kw["edgefactor"], kw["seed"])
        elif kind == "grid":
            n = kw["rows"] * kw["cols"]
            e = O.np_gen_grid(kw["rows"], kw["cols"])
        else:
            n = kw["n"]
            e = O.np_gen_er(kw["n"], kw["m"], kw["seed"])
        g = ref.build_csr(ref.EdgeList(n, e))  # graph.py:184-201
        payload[f"{key}__n"] = np.int64(n)
        payload[f"{key}__m"] = np.int64(g.num_edges)
        payload[f"{key}__sha"] = np.array(csr_sha(g.row_offsets, g.col_indices))
        payload[f"{key}__maxdeg"] = np.int64(g.max_degree)
        for mode in MODES:
            colors, rep = ref.color_graph(g, ref.HybridConfig(mode=mode, workers=8))
            recs = np.array(
                [[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                 for r in rep.per_round], dtype=np.int64).reshape(-1, 4)
            payload[f"{key}__{mode}__rec"] = recs
            if mode == "hybrid":
                payload[f"{key}__colors"] = colors.astype(np.int32)
                payload[f"{key}__colors_used"] = np.int64(rep.colors_used)
                payload[f"{key}__rounds"] = np.int64(rep.total_rounds)
            assert rep.valid
        print(f"configs.npz: {key} n={n} m_dir={g.num_edges} rounds={payload[f'{key}__rounds']} "
              f"colors={payload[f'{key}__colors_used']}")
    payload["cases"] = np.array(list(cases))
    np.savez_compressed(HERE / "configs.npz", **payload)


def main():
    ref, conf = load_reference()
    print("reference:", ref.__file__, "backends:", ref.available_backends())
    make_corpus(ref, conf)
    make_configs(ref)


if __name__ == "__main__":
    main()
