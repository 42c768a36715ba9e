"""GPU parity: the CUDA path (through libhcb's C-ABI) against the reference's
recorded outputs (tests/golden) and the oracle, bit-exact."""

import numpy as np
import pytest
import torch

from conftest import CONFIG_SPECS, MODES, THRESHOLDS, csr_sha, grid_closed_form, grid_records
from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_1912_01478_b200 as hc  # noqa: E402
from paper_1912_01478_b200 import graph as G  # noqa: E402


def _recs(report):
    return np.array([[int(r.mode_used == "topo"), r.worklist_size_in, r.worklist_size_out, r.conflicts]
                     for r in report.per_round], dtype=np.int64).reshape(-1, 4)


def _csr(g):
    return hc.CsrGraph(g.n, len(g.ci), g.ro, g.ci)


# ---------------------------------------------------------------- solve
def test_solve_matches_reference_corpus(corpus):
    """347 graphs of the reference's seeded corpora x 3 modes x 4 thresholds."""
    for g in corpus:
        dg = _csr(g).to_device() if g.n else _csr(g)
        for mode in MODES:
            for thr in THRESHOLDS:
                colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode, threshold_fraction=thr))
                assert colors.dtype == np.int64  # test_acceptance.py:162
                assert np.array_equal(colors, g.colors), (g.name, mode, thr)
                assert np.array_equal(_recs(rep), g.records[(mode, thr)]), (g.name, mode, thr)
                assert rep.valid and rep.total_rounds == len(g.records[(mode, thr)])
                assert rep.colors_used == g.colors_used


def test_golden_traces():
    # P3 / K3 (test_coloring.py:169-193), K3 hybrid schedule (test_driver.py:30-36)
    p3 = hc.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    c, rep = hc.color_graph(p3)
    assert c.tolist() == [1, 2, 1] and [r.worklist_size_in for r in rep.per_round] == [3, 2]
    k3 = hc.CsrGraph(3, 6, np.array([0, 2, 4, 6]), np.array([1, 2, 0, 2, 0, 1]))
    c, rep = hc.color_graph(k3, hc.HybridConfig(threshold_fraction=0.6))
    assert [r.mode_used for r in rep.per_round] == ["topo", "data", "data"]
    assert [r.worklist_size_in for r in rep.per_round] == [3, 2, 1]
    assert c.tolist() == [1, 2, 3] and rep.colors_used == 3 and rep.valid
    # empty graph and isolated nodes (test_driver.py:88-98)
    c, rep = hc.color_graph(hc.CsrGraph(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64)))
    assert c.size == 0 and rep.total_rounds == 0 and rep.colors_used == 0 and rep.valid
    c, rep = hc.color_graph(hc.CsrGraph(5, 0, np.zeros(6, np.int64), np.zeros(0, np.int64)))
    assert c.tolist() == [1] * 5 and rep.total_rounds == 1


def test_report_invariants_and_timing():
    e = O.gen_er(3000, 40000, 11)
    ro, ci = O.build_csr(3000, e)
    colors, rep = hc.color_graph(hc.CsrGraph(3000, len(ci), ro, ci))
    sizes_in = [r.worklist_size_in for r in rep.per_round]
    sizes_out = [r.worklist_size_out for r in rep.per_round]
    assert sizes_out[:-1] == sizes_in[1:] and sizes_out[-1] == 0
    assert all(a > b for a, b in zip(sizes_in, sizes_out))
    assert rep.total_seconds > 0 and all(r.wall_seconds > 0 for r in rep.per_round)
    assert rep.colors_used == int(colors.max())


def test_kernels_argument_parity():
    g = hc.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    hc.color_graph(g, kernels=hc.get_kernels("cuda"))
    with pytest.raises(ValueError):
        hc.color_graph(g, kernels=object())


# ---------------------------------------------------------------- configs
def _device_graph(kind, kw):
    if kind == "rmat":
        return G.build_csr_device(G.gen_rmat_edges(kw["scale"], kw["edgefactor"], kw["seed"]), 1 << kw["scale"])
    if kind == "grid":
        return G.build_csr_device(G.gen_grid_edges(kw["rows"], kw["cols"]), kw["rows"] * kw["cols"])
    return G.build_csr_device(G.gen_er_edges(kw["n"], kw["m"], kw["seed"]), kw["n"])


@pytest.mark.parametrize("key", list(CONFIG_SPECS))
def test_device_generation_csr_and_solve_match_reference(configs, key):
    """C1 (RMAT-16 seed 0) at full size + reduced shapes of C2/C4: device
    generator + device build_csr == reference build_csr (sha256), and the
    device solve == reference color_graph in every mode."""
    kind, kw = CONFIG_SPECS[key]
    want = configs[key]
    dg = _device_graph(kind, kw)
    assert dg.num_edges == want["m"]
    host = dg.to_host()
    assert csr_sha(host.row_offsets, host.col_indices) == want["sha"]
    for mode in MODES:
        colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert np.array_equal(_recs(rep), want["rec"][mode]), (key, mode)
        assert np.array_equal(colors, want["colors"]), (key, mode)
        assert rep.valid


@pytest.mark.parametrize("rows,cols", [(1024, 1024), (1000, 37), (3, 2000)])
def test_grid_closed_form(rows, cols):
    dg = G.grid_graph(rows, cols)
    want, rounds = grid_closed_form(rows, cols)
    colors, rep = hc.color_graph(dg)
    assert np.array_equal(colors, want) and rep.total_rounds == rounds
    assert rep.per_round[0].conflicts == G.grid_num_pairs(rows, cols)


def test_headline_grid4096_every_round_every_mode():
    """configs[1] at full size: colors and all 4096 per-round records in data,
    topo and hybrid mode equal the reference-pinned closed form
    (conftest.grid_records; pinned by test_oracle.py::
    test_grid_record_closed_form_vs_reference)."""
    dg = G.grid_graph(4096, 4096)
    want, rounds = grid_closed_form(4096, 4096)
    for mode in MODES:
        colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert rep.total_rounds == rounds == 4096
        assert np.array_equal(_recs(rep), grid_records(4096, 4096, mode, 0.6)), mode
        assert np.array_equal(colors, want), mode
        assert rep.valid and rep.colors_used == 2


@pytest.mark.parametrize("rows,cols", [(1000, 37), (3, 2000), (777, 1500)])
def test_grid_records_closed_form(rows, cols):
    dg = G.grid_graph(rows, cols)
    for mode, thr in (("hybrid", 0.6), ("hybrid", 0.2), ("data", 0.6), ("topo", 0.6)):
        _, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode, threshold_fraction=thr))
        assert np.array_equal(_recs(rep), grid_records(rows, cols, mode, thr)), (mode, thr)


@pytest.mark.parametrize("scale,seed", [(12, 1), (14, 3)])
def test_rmat_vs_oracle(scale, seed):
    e = O.gen_rmat(scale, 16, seed)
    ro, ci = O.build_csr(1 << scale, e)
    dg = G.rmat_graph(scale, 16, seed)
    h = dg.to_host()
    assert np.array_equal(h.row_offsets, ro) and np.array_equal(h.col_indices, ci)
    for mode in MODES:
        oc, orec = O.color(ro, ci, mode)
        colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
        assert np.array_equal(colors, oc) and np.array_equal(_recs(rep), orec)


# ---------------------------------------------------------------- csr build
def test_build_csr_edge_cases_vs_oracle():
    rng = np.random.default_rng(7)
    cases = [
        (5, np.zeros((0, 2), np.int64)),
        (4, np.array([[0, 0], [1, 1]])),                       # loops only
        (3, np.array([[0, 1], [1, 0], [0, 1], [2, 1]])),       # dupes both directions
        (50, rng.integers(0, 50, (2000, 2))),                  # dense: rows 65..8192 path
        (30000, np.column_stack([np.zeros(50000, np.int64), rng.integers(0, 30000, 50000)])),  # hub > 8192
        (20000, rng.integers(0, 20000, (60000, 2))),
    ]
    for n, e in cases:
        ro, ci = O.build_csr(n, e)
        g = hc.build_csr(hc.EdgeList(n, e))
        assert np.array_equal(g.row_offsets, ro) and np.array_equal(g.col_indices, ci), n
        assert g.num_edges == len(ci)


def test_build_csr_rejects_out_of_range():
    with pytest.raises(ValueError):
        G.build_csr_device(torch.tensor([[0, 5]], device="cuda"), 3)


def test_generators_match_oracle():
    assert np.array_equal(G.gen_grid_edges(17, 23).cpu().numpy(), O.gen_grid(17, 23))
    assert np.array_equal(G.gen_er_edges(12345, 100000, 9).cpu().numpy(), O.gen_er(12345, 100000, 9))
    assert np.array_equal(G.gen_rmat_edges(13, 16, 4).cpu().numpy(), O.gen_rmat(13, 16, 4))


# ---------------------------------------------------------------- verify / colors_used
def test_verify_and_colors_used_semantics():
    p3 = hc.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    k3 = hc.CsrGraph(3, 6, np.array([0, 2, 4, 6]), np.array([1, 2, 0, 2, 0, 1]))
    assert hc.verify_coloring(p3, np.array([1, 2, 1])) == 0   # driver.py examples (SPEC)
    assert hc.verify_coloring(p3, np.array([1, 1, 2])) == 1
    assert hc.verify_coloring(k3, np.array([1, 1, 1])) == 3
    with pytest.raises(ValueError):
        hc.verify_coloring(p3, np.array([1, 2]))
    assert hc.colors_used(np.array([1, 2, 1])) == 2 and hc.colors_used(np.array([], np.int64)) == 0
    with pytest.raises(ValueError, match="uncolored"):
        hc.colors_used(np.array([1, 0, 2]))


# ---------------------------------------------------------------- plugin API
def test_plugin_round_functions_reference_cases():
    """test_coloring.py::TestIterations on the cuda kernel module."""
    k = hc.get_kernels("cuda")
    p3 = hc.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    state, wl = hc.ColorState.fresh(3), hc.Worklist.init_full(3)
    out = hc.data_driven_iteration(p3, state, wl, 1, kernels=k)
    assert state.colors_read.tolist() == [1, 0, 0] and wl.current.tolist() == [1, 2]
    assert (out.conflicts_detected, out.pushed_back, out.colored_permanently) == (2, 2, 1)
    k3 = hc.CsrGraph(3, 6, np.array([0, 2, 4, 6]), np.array([1, 2, 0, 2, 0, 1]))
    state, wl = hc.ColorState.fresh(3), hc.Worklist.init_full(3)
    hc.topology_driven_iteration(k3, state, wl, 1)
    assert state.colors_read.tolist() == [1, 0, 0]
    out = hc.topology_driven_iteration(k3, state, wl, 2)
    assert state.colors_read.tolist() == [1, 2, 0] and wl.current.tolist() == [2] and out.pushed_back == 1


def test_plugin_numpy_calling_convention_matches_oracle():
    """Drive the reference's round structure with numpy arrays through the
    cuda module (the _BACKENDS shim path) and compare with the oracle."""
    k = hc.get_kernels("cuda")
    rng = np.random.default_rng(23)
    for _ in range(10):
        n = int(rng.integers(2, 200))
        ro, ci = O.build_csr(n, rng.integers(0, n, (n * 3, 2)))
        want, rec = O.color(ro, ci, "data")
        cr = np.zeros(n, np.int64); cw = np.zeros(n, np.int64); st = np.zeros(n, np.int64)
        cur = np.arange(n, dtype=np.int64)
        t, sizes = 1, []
        while len(cur):
            sizes.append(len(cur))
            nxt = np.empty(n, np.int64); cursor = np.zeros(1, np.int64)
            k.assign_from_list(ro, ci, cr, cw, st, cur, t, 0, 1, 1024)
            cr[cur] = cw[cur]
            k.resolve_from_list(ro, ci, cr, cw, st, cur, t, nxt, cursor, 1, 1024)
            cr[cur] = cw[cur]
            cur = np.sort(nxt[: cursor[0]])
            t += 1
        assert np.array_equal(cr, want) and sizes == rec[:, 1].tolist()


def test_plugin_bench_kernels():
    k = hc.get_kernels("cuda")
    active = np.ones(1000, np.uint8)
    nxt, cursor = np.empty(1000, np.int64), np.zeros(1, np.int64)
    k.bench_sweep(active, 299, nxt, cursor, 1, 1024)
    assert cursor[0] == 700 and active[:300].sum() == 0 and active[300:].all()
    assert sorted(nxt[:700].tolist()) == list(range(300, 1000))
    nodes = np.arange(300, 1000, dtype=np.int64)
    nxt2, cursor2 = np.empty(1000, np.int64), np.zeros(1, np.int64)
    k.bench_from_list(nodes, active, 599, nxt2, cursor2, 1, 1024)
    assert cursor2[0] == 400 and active[300:600].sum() == 0


def test_worklist_semantics():
    wl = hc.Worklist(5)
    for u in (4, 1, 3):
        wl.push(u)
    assert wl.swap_and_sort() == 3 and wl.current.tolist() == [1, 3, 4]
    wl.push_many(np.array([2, 0]))
    assert wl.swap_and_sort() == 2 and wl.current.tolist() == [0, 2]
    wl.push(1); wl.push(1)
    with pytest.raises(AssertionError):
        wl.swap_and_sort()
    wl2 = hc.Worklist(2)
    wl2.push(0); wl2.push(1)
    with pytest.raises(RuntimeError):
        wl2.push(1)
    with pytest.raises(RuntimeError):
        wl2.push(7)


@pytest.mark.parametrize("leaves,extra", [(20000, 3000), (40000, 5000), (3000, 200000)])
def test_storage_formats_vs_oracle(leaves, extra):
    """Star hubs push the solve onto each storage format: 32-bit state words
    (a degree > 16384), int32 vs int16-delta columns (|v-u| >= 2^15 or not)."""
    rng = np.random.default_rng(leaves)
    n = leaves + 1
    e = np.concatenate([np.column_stack([np.zeros(leaves, np.int64), np.arange(1, n)]),
                        rng.integers(0, n, (extra, 2))])
    ro, ci = O.build_csr(n, e)
    g = hc.CsrGraph(n, len(ci), ro, ci)
    for mode in MODES:
        want, rec = O.color(ro, ci, mode)
        colors, rep = hc.color_graph(g, hc.HybridConfig(mode=mode))
        assert np.array_equal(colors, want) and np.array_equal(_recs(rep), rec), mode


@pytest.mark.parametrize("fmt", [(1, 1, 1), (0, 1, 1), (0, 0, 1), (0, 1, 0)])
def test_forced_storage_formats_vs_golden(configs, fmt):
    """Every (offset width, state width, column format) instantiation, with
    and without the bin-0-only kernel and its ELL4 rows, on the
    reference-recorded C1 graph (RMAT-16) and a grid (bin-0 only, degree <= 4:
    the ELL4 kernel whenever delta columns are allowed)."""
    L = hc._lib.load()
    L.hc_solve_set_formats(*fmt)
    try:
        for small, ell, live in ((1, 1, -1), (1, 0, -1), (0, 1, 0), (0, 1, 1)):
            L.hc_solve_set_small(small)
            L.hc_solve_set_ell(ell)
            L.hc_solve_set_live(live)
            for key in ("rmat16", "grid64x96"):
                kind, kw = CONFIG_SPECS[key]
                want = configs[key]
                dg = _device_graph(kind, kw)
                for mode in MODES:
                    colors, rep = hc.color_graph(dg, hc.HybridConfig(mode=mode))
                    assert np.array_equal(colors, want["colors"]), (key, mode, fmt, small, ell, live)
                    assert np.array_equal(_recs(rep), want["rec"][mode]), (key, mode, fmt, small, ell, live)
    finally:
        L.hc_solve_set_formats(0, 0, 0)
        L.hc_solve_set_small(1)
        L.hc_solve_set_ell(1)
        L.hc_solve_set_live(-1)


@pytest.mark.parametrize("x8", [1, 0])
def test_8bit_state_words_vs_oracle(x8):
    """8-bit state words (every degree <= 128) against the oracle, and with
    them forbidden: ER graphs of max degree ~60-110, a grid (bin-0-only: keeps
    16-bit words either way), and cliques K_128 / K_129 whose last tentative colors
    (128, 129) overflow 8 bits, so the solve is redone with 16-bit words."""
    L = hc._lib.load()
    L.hc_solve_set_x8(x8)
    try:
        cases = [(4000, O.gen_er(4000, 4000 * 30, 5)), (3000, O.gen_er(3000, 3000 * 40, 6)),
                 (64 * 96, O.gen_grid(64, 96))]
        for k in (128, 129):
            iu, ju = np.triu_indices(k, 1)
            cases.append((k, np.stack([iu, ju], 1).astype(np.int64)))
        for n, e in cases:
            ro, ci = O.build_csr(n, e)
            g = hc.CsrGraph(n, len(ci), ro, ci).to_device()
            for mode in MODES:
                want, rec = O.color(ro, ci, mode)
                colors, rep = hc.color_graph(g, hc.HybridConfig(mode=mode))
                assert np.array_equal(colors, want) and np.array_equal(_recs(rep), rec), (n, mode, x8)
    finally:
        L.hc_solve_set_x8(1)


# ---------------------------------------------------------------- unsorted caller CSR
def _shuffle_rows(ro, ci, rng):
    ci = ci.copy()
    for u in range(len(ro) - 1):
        rng.shuffle(ci[ro[u]:ro[u + 1]])
    return ci


def test_unsorted_rows_match_reference(corpus):
    """A caller CSR whose rows are not sorted (a user-built CsrGraph, a
    third-party .npz): the reference scans whole rows (_kernels.pyx:106-113) so
    its result does not depend on row order; the device path partitions such
    rows (lower ids first, hc_csr_partition_lower_first) and must give the
    reference's colors and records."""
    rng = np.random.default_rng(7)
    done = 0
    for g in corpus[::5]:
        if g.n == 0 or len(g.ci) == 0:
            continue
        ci = _shuffle_rows(g.ro, g.ci, rng)
        for mode in MODES:
            colors, rep = hc.color_graph(hc.CsrGraph(g.n, len(ci), g.ro, ci), hc.HybridConfig(mode=mode))
            assert np.array_equal(colors, g.colors), (g.name, mode)
            assert np.array_equal(_recs(rep), g.records[(mode, 0.6)]), (g.name, mode)
        done += 1
    assert done > 40
    # hubs and the larger bins
    e = O.gen_rmat(14, 16, 5)
    ro, ci = O.build_csr(1 << 14, e)
    want, rec = O.color(ro, ci, "hybrid")
    shuffled = _shuffle_rows(ro, ci, rng)
    dg = hc.CsrGraph(1 << 14, len(ci), ro, shuffled).to_device()
    assert dg.lower_first is None
    colors, rep = hc.color_graph(dg)
    assert np.array_equal(colors, want) and np.array_equal(_recs(rep), rec)
    part = dg.col_indices.cpu().numpy()
    for u in range(0, 1 << 14, 97):
        row = part[ro[u]:ro[u + 1]]
        low = row < u
        k = int(low.sum())
        assert low[:k].all() and not low[k:].any(), u                      # lower ids form a prefix
        assert np.array_equal(np.sort(row), ci[ro[u]:ro[u + 1]]), u          # same multiset


def test_sorted_caller_csr_is_not_copied():
    ro, ci = O.build_csr(500, O.gen_er(500, 3000, 3))
    dg = hc.CsrGraph(500, len(ci), ro, ci).to_device()
    before = dg.col_indices.data_ptr()
    dg.ensure_lower_first()
    assert dg.lower_first and dg.col_indices.data_ptr() == before


def test_plain_baseline_same_results(corpus):
    """hc_solve_plain (bench-only Plain baseline: unordered atomically pushed
    worklists) computes the same colors and records as hc_solve."""
    graphs = [G.build_csr_device(G.gen_rmat_edges(13, 16, 2), 1 << 13), G.grid_graph(200, 130),
              G.er_graph(20000, 24, 3)]
    graphs += [_csr(g).to_device() for g in corpus[::23] if g.n > 1]
    for dg in graphs:
        s = hc.Solver(dg)
        for mode in MODES:
            thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
            a = s.run(mode, thr)
            ca = a.colors.cpu().numpy().copy()
            b = s.run(mode, thr, plain=True)
            assert np.array_equal(ca, b.colors.cpu().numpy()), mode
            assert np.array_equal(a.records[:, 1:5], b.records[:, 1:5]), mode


# ---------------------------------------------------------------- CUDA-graph capture
@pytest.mark.parametrize("key", ["rmat16", "grid64x96"])
def test_planned_launch_captured_in_cuda_graph(configs, key):
    """hc_solve_plan_graph + hc_solve_launch: the launch is stream-ordered
    work only, so it is captured into a CUDA graph; two replays (and an eager
    launch) give the reference's colors and records (configs.npz goldens)."""
    import torch

    kind, kw = CONFIG_SPECS[key]
    want = configs[key]
    dg = _device_graph(kind, kw)
    thr = hc.threshold_count(hc.HybridConfig(), dg.num_nodes)
    ps = hc.PlannedSolver(dg)
    ps.launch("hybrid", thr)  # eager
    r = ps.result()
    assert np.array_equal(r.colors.cpu().numpy(), want["colors"])
    assert np.array_equal(r.records[:, 1:5], want["rec"]["hybrid"])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            ps.launch("hybrid", thr, torch.cuda.current_stream())
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        ps.colors.fill_(-1)
        graph.replay()
        r = ps.result()
        assert np.array_equal(r.colors.cpu().numpy(), want["colors"]), key
        assert np.array_equal(r.records[:, 1:5], want["rec"]["hybrid"]), key
