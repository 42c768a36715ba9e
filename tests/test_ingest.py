"""Graph ingestion (MatrixMarket on the device, .npz cache) and device
degree_stats against the reference's recorded behaviour
(tests/golden/mtx.json, written by tests/golden/make_mtx_golden.py from
hybridcolor.parse_matrix_market / load_graph / degree_stats)."""

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1912_01478_b200 as hc
from paper_1912_01478_b200 import ingest

HEADER_ERRORS = ("empty input", "malformed banner", "missing size line", "size line must",
                 "non-integer size line", "negative size entry")


@pytest.fixture(scope="module")
def golden():
    return json.loads((GOLDEN / "mtx.json").read_text())


# ---------------------------------------------------------------- CPU (host side)
def test_header_parse_matches_reference(golden):
    """Banner / size-line handling is host code: same messages as the reference."""
    for case in golden["parse"]:
        out = case["out"]
        data = case["text"].encode()
        if "error" in out and out["error"].startswith(HEADER_ERRORS):
            with pytest.raises(hc.MatrixMarketError) as ei:
                ingest._header(data, False)
            assert str(ei.value) == out["error"], case["text"]
        else:
            rows, cols, nnz, off = ingest._header(data, False)
            if "n" in out:
                assert max(rows, cols) == out["n"] and len(out["edges"]) == 2 * nnz


def test_csr_cache_roundtrip_and_version(tmp_path):
    g = hc.CsrGraph(3, 4, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]))
    p = tmp_path / "g.npz"
    hc.save_csr_cache(g, p)
    g2 = hc.load_csr_cache(p)
    assert g2.num_nodes == 3 and g2.num_edges == 4
    assert g2.row_offsets.tolist() == [0, 1, 3, 4] and g2.col_indices.tolist() == [1, 0, 2, 1]
    assert hc.load_graph(p).col_indices.tolist() == [1, 0, 2, 1]  # .npz dispatch stays on the host
    bad = tmp_path / "bad.npz"
    np.savez(bad, format_version=np.array([99]), num_nodes=np.array([1]), row_offsets=np.zeros(2),
             col_indices=np.zeros(0))
    with pytest.raises(ValueError, match="unsupported"):
        hc.load_csr_cache(bad)
    np.savez(bad, x=np.zeros(1))
    with pytest.raises(ValueError, match="missing format_version"):
        hc.load_csr_cache(bad)
    with pytest.raises(FileNotFoundError):
        hc.load_graph(tmp_path / "nope.mtx")


def test_degree_stats_empty_graph_raises():
    with pytest.raises(ValueError, match="undefined"):
        hc.degree_stats(hc.CsrGraph(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64)))


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_parse_matrix_market_matches_reference(golden):
    for case in golden["parse"]:
        out = case["out"]
        if "error" in out:
            with pytest.raises(hc.MatrixMarketError) as ei:
                hc.parse_matrix_market(case["text"])
            assert str(ei.value) == out["error"], case["text"]
        else:
            el = hc.parse_matrix_market(case["text"])
            assert el.num_nodes_declared == out["n"], case["text"]
            assert el.edges.reshape(-1).tolist() == out["edges"], case["text"]


@pytest.mark.gpu
def test_load_graph_files_match_reference(golden, tmp_path):
    """Files go through text-mode semantics (CRLF / CR line ends) and the
    device CSR build."""
    p = tmp_path / "g.mtx"
    for case in golden["files"]:
        p.write_bytes(case["raw"].encode("ascii"))
        out = case["out"]
        if "error" in out:
            with pytest.raises(hc.MatrixMarketError) as ei:
                hc.load_graph(p)
            assert str(ei.value) == out["error"], repr(case["raw"])
        else:
            g = hc.load_graph(p)
            assert g.num_nodes == out["n"], repr(case["raw"])
            assert g.row_offsets.tolist() == out["ro"] and g.col_indices.tolist() == out["ci"], repr(case["raw"])


@pytest.mark.gpu
def test_reference_test_cases():
    """pkg/tests/test_graph_core.py:21-94 and the shipped data files."""
    el = hc.parse_matrix_market("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n2 3\n")
    assert el.num_nodes_declared == 3 and el.edges.tolist() == [[0, 1], [1, 2]]
    import io

    el = hc.parse_matrix_market(io.StringIO("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n2 1\n"))
    assert el.edges.tolist() == [[1, 0]]
    el = hc.parse_matrix_market(["%%MatrixMarket matrix coordinate pattern general", "2 5 1", "1 4"])
    assert el.num_nodes_declared == 5 and el.edges.tolist() == [[0, 3]]


@pytest.mark.gpu
def test_large_file_roundtrip(tmp_path):
    """A 200k-entry file: device parse == the generating pairs; CSR == build_csr
    of them; non-ASCII bytes raise like an ascii-mode open."""
    rng = np.random.default_rng(3)
    n, m = 50000, 200000
    e = rng.integers(1, n + 1, (m, 2))
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "% generated", f"{n} {n} {m}"]
    lines += [f"{a} {b}" + (" 1.0" if i % 7 == 0 else "") for i, (a, b) in enumerate(e.tolist())]
    p = tmp_path / "big.mtx"
    p.write_text("\n".join(lines) + "\n")
    g = hc.load_graph(p)
    want = hc.build_csr(hc.EdgeList(n, e - 1))
    assert np.array_equal(g.row_offsets, want.row_offsets) and np.array_equal(g.col_indices, want.col_indices)
    el = hc.parse_matrix_market(p.read_text())
    assert np.array_equal(el.edges, e - 1)
    p.write_bytes(p.read_bytes().replace(b"% generated", b"% gen\xe9rated"))
    with pytest.raises(UnicodeDecodeError):
        hc.load_graph(p)


@pytest.mark.gpu
def test_degree_stats_matches_reference(golden):
    for case in golden["degree_stats"]:
        if case["n"] == 0:
            continue
        g = hc.CsrGraph(case["n"], len(case["ci"]), np.array(case["ro"]), np.array(case["ci"]))
        s = hc.degree_stats(g)
        assert [s.min_degree, s.median_degree, s.max_degree, s.num_nodes, s.num_undirected_edges] == case["stats"]
        s2 = hc.degree_stats(g.to_device())
        assert s2 == s


@pytest.mark.gpu
def test_degree_stats_large_vs_numpy():
    dg = hc.rmat_graph(16, 16, 0)
    deg = np.diff(dg.row_offsets.cpu().numpy())
    s = hc.degree_stats(dg)
    n = len(deg)
    assert (s.min_degree, s.median_degree, s.max_degree) == (int(deg.min()), int(np.partition(deg, n // 2)[n // 2]),
                                                             int(deg.max()))
    # wide degrees: a star with a 3M-degree hub exercises every radix digit
    n = 3_000_001
    ro = np.arange(n + 1, dtype=np.int64) + (n - 1)
    ro[0] = 0
    ro[1:] = (n - 1) + np.arange(n, dtype=np.int64)
    ci = np.concatenate([np.arange(1, n), np.zeros(n - 1, np.int64)])
    s = hc.degree_stats(hc.CsrGraph(n, len(ci), ro, ci))
    assert (s.min_degree, s.median_degree, s.max_degree) == (1, 1, n - 1)
