"""CPU: pin the oracle (oracle/ipgc_oracle.c) against the reference's own
outputs recorded in tests/golden (and the reference's known answers)."""

import numpy as np
import pytest

from conftest import CONFIG_SPECS, GOLDEN, MODES, THRESHOLDS, csr_sha, grid_closed_form, grid_records
from oracle import oracle as O


def _rec_cols(rec):
    return rec[:, 1:5] if rec.shape[1] == 6 else rec


def test_generators_c_equal_numpy_twin():
    assert np.array_equal(O.gen_grid(7, 5), O.np_gen_grid(7, 5))
    assert np.array_equal(O.gen_er(1000, 20000, 3), O.np_gen_er(1000, 20000, 3))
    assert np.array_equal(O.gen_rmat(11, 16, 5), O.np_gen_rmat(11, 16, 5))


def test_known_answers_p3_k3():
    # test_coloring.py:169-193, test_driver.py:30-36
    ro, ci = O.build_csr(3, np.array([[0, 1], [1, 2]]))
    colors, rec = O.color(ro, ci, "data")
    assert colors.tolist() == [1, 2, 1] and rec[:, 1].tolist() == [3, 2]
    assert rec[0, 3] == 2  # P3 round 1 conflicts (test_coloring.py:112)
    ro, ci = O.build_csr(3, np.array([[0, 1], [0, 2], [1, 2]]))
    colors, rec = O.color(ro, ci, "hybrid", 0.6)
    assert colors.tolist() == [1, 2, 3]
    assert rec[:, 0].tolist() == [1, 0, 0] and rec[:, 1].tolist() == [3, 2, 1]


def test_empty_and_isolated():
    ro, ci = O.build_csr(0, np.zeros((0, 2), np.int64))
    colors, rec = O.color(ro, ci)
    assert colors.size == 0 and rec.shape[0] == 0
    ro, ci = O.build_csr(5, np.zeros((0, 2), np.int64))
    colors, rec = O.color(ro, ci)
    assert colors.tolist() == [1] * 5 and rec.shape[0] == 1


def test_oracle_matches_reference_corpus(corpus):
    """Every graph of the reference's seeded corpora x every mode x threshold."""
    assert len(corpus) >= 300
    for g in corpus:
        for mode in MODES:
            for thr in THRESHOLDS:
                colors, rec = O.color(g.ro, g.ci, mode, thr)
                assert np.array_equal(colors, g.colors), (g.name, mode, thr)
                assert np.array_equal(rec, g.records[(mode, thr)]), (g.name, mode, thr)


def test_oracle_csr_and_solve_match_reference_configs(configs):
    for key, (kind, kw) in CONFIG_SPECS.items():
        want = configs[key]
        if kind == "rmat":
            e = O.gen_rmat(kw["scale"], kw["edgefactor"], kw["seed"])
        elif kind == "grid":
            e = O.gen_grid(kw["rows"], kw["cols"])
        else:
            e = O.gen_er(kw["n"], kw["m"], kw["seed"])
        ro, ci = O.build_csr(want["n"], e)
        assert csr_sha(ro, ci) == want["sha"], key
        for mode in MODES:
            colors, rec = O.color(ro, ci, mode)
            assert np.array_equal(rec, want["rec"][mode]), (key, mode)
            if mode == "hybrid":
                assert np.array_equal(colors, want["colors"]), key
        assert O.verify(ro, ci, colors) == 0


@pytest.mark.parametrize("rows,cols", [(3, 3), (5, 7), (33, 17), (128, 64)])
def test_grid_closed_form(rows, cols):
    ro, ci = O.build_csr(rows * cols, O.gen_grid(rows, cols))
    colors, rec = O.color(ro, ci)
    want, rounds = grid_closed_form(rows, cols)
    assert np.array_equal(colors, want) and rec.shape[0] == rounds
    assert rec[0, 3] == O.grid_num_edges(rows, cols)  # round-1 conflicts = #undirected edges


def test_grid_record_closed_form_vs_reference():
    """The per-round closed form (conftest.grid_records) equals the REFERENCE's
    records (tests/golden/grids.npz, make_grid_golden.py: the reference's
    color_graph on its own grid builder) on every shape up to 512^2 and on
    rectangles, in every mode and threshold recorded; the colors are the
    checkerboard."""
    import hashlib

    z = np.load(GOLDEN / "grids.npz")
    checked = 0
    for r, c in z["shapes"].tolist():
        want_colors, rounds = grid_closed_form(r, c)
        sha = hashlib.sha256(want_colors.astype("<i8").tobytes()).hexdigest()
        for setting in z["settings"].tolist():
            mode, thr = setting.split(":")
            key = f"{r}x{c}__{mode}__{thr}"
            ref = z[key + "__rec"]
            assert np.array_equal(grid_records(r, c, mode, float(thr)), ref), key
            assert ref.shape[0] == rounds and str(z[key + "__colors_sha"]) == sha, key
            checked += 1
    assert checked == 20 * 6


@pytest.mark.parametrize("seed", [0, 1])
def test_grid_record_closed_form_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(12):
        r, c = (int(x) for x in rng.integers(1, 90, 2))
        ro, ci = O.build_csr(r * c, O.gen_grid(r, c))
        for mode in MODES:
            thr = float(rng.choice(THRESHOLDS))
            _, rec = O.color(ro, ci, mode, thr)
            assert np.array_equal(rec, grid_records(r, c, mode, thr)), (r, c, mode, thr)
