"""CLI parity with the reference front end (pkg/tests/test_cli.py): layouts,
report files, exit codes.  Usage / input errors are host-side and run on CPU;
everything that colors, loads or benchmarks runs on the GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
P3 = "%%MatrixMarket matrix coordinate pattern symmetric\n% path on three nodes: 1-2-3\n3 3 2\n1 2\n2 3\n"
K3 = "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 2\n1 3\n2 3\n"


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1912_01478_b200", *map(str, args)],
                          capture_output=True, text=True, cwd=REPO)


@pytest.fixture
def data(tmp_path):
    (tmp_path / "p3.mtx").write_text(P3)
    (tmp_path / "k3.mtx").write_text(K3)
    return tmp_path


def strip_timing(doc):
    if isinstance(doc, dict):
        return {k: strip_timing(v) for k, v in doc.items() if not k.endswith("micros")}
    if isinstance(doc, list):
        return [strip_timing(v) for v in doc]
    return doc


# ---------------------------------------------------------------- CPU
def test_usage_errors(data):
    assert run_cli("color", data / "k3.mtx", "--threshold", "1.5").returncode == 2
    assert run_cli("color", data / "k3.mtx", "--mode", "warp").returncode == 2
    assert run_cli("bench", data / "k3.mtx").returncode == 2  # --out required
    assert run_cli("color", data / "k3.mtx", "--workers", "0").returncode == 2


def test_missing_and_malformed_input(data):
    missing = data / "ghost.mtx"
    proc = run_cli("stats", missing)
    assert proc.returncode == 2 and str(missing) in proc.stderr
    bad = data / "bad.mtx"
    bad.write_text("not a matrix market file\n")
    proc = run_cli("stats", bad)
    assert proc.returncode == 2 and "banner" in proc.stderr


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_stats_layouts(data):
    proc = run_cli("stats", data / "p3.mtx")
    assert proc.returncode == 0 and proc.stdout.strip() == "3 nodes, 2 edges, δ 1/1/2"
    proc = run_cli("stats", data / "k3.mtx")
    assert proc.returncode == 0 and proc.stdout.strip() == "3 nodes, 3 edges, δ 2/2/2"
    doc = json.loads(run_cli("stats", data / "p3.mtx", "--format", "json").stdout)
    assert doc["median_degree"] == 1 and doc["num_undirected_edges"] == 2


@pytest.mark.gpu
def test_color_outputs(data, tmp_path):
    proc = run_cli("color", data / "k3.mtx", "--mode", "hybrid")
    assert proc.returncode == 0
    assert "colors_used: 3" in proc.stdout and "valid: true" in proc.stdout and "backend: cuda" in proc.stdout
    outs = [json.loads(run_cli("color", data / "p3.mtx", "--mode", m, "--format", "json").stdout)
            for m in ("data", "topo")]
    assert outs[0]["colors_used"] == outs[1]["colors_used"] == 2
    assert outs[0]["total_rounds"] == outs[1]["total_rounds"] == 2
    lines = run_cli("color", data / "k3.mtx", "--format", "csv").stdout.strip().splitlines()
    assert lines[0] == "round,mode,wl_in,wl_out,conflicts,micros" and len(lines) == 4
    out = tmp_path / "report.json"
    assert run_cli("color", data / "k3.mtx", "--out", out).returncode == 0
    doc = json.loads(out.read_text())
    assert doc["graph"] == "k3" and doc["valid"] is True and doc["config"]["mode"] == "hybrid"
    assert run_cli("color", data / "k3.mtx", "--out", tmp_path / "no" / "dir" / "x.json").returncode == 3
    docs = []
    for name in ("a.json", "b.json"):
        o = tmp_path / name
        assert run_cli("color", data / "k3.mtx", "--workers", "4", "--out", o).returncode == 0
        docs.append(json.dumps(strip_timing(json.loads(o.read_text())), sort_keys=True))
    assert docs[0] == docs[1]


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    graph = tmp_path / "n25.mtx"
    graph.write_text("%%MatrixMarket matrix coordinate pattern general\n25 25 0\n")
    out = tmp_path / "tti.csv"
    proc = run_cli("bench", graph, "--batch", "10", "--reps", "2", "--out", out)
    assert proc.returncode == 0, proc.stderr
    assert len(out.read_text().strip().splitlines()) == 1 + 2 * 3
    assert "deactivation sets identical across variants: yes" in proc.stdout and "crossovers:" in proc.stdout


@pytest.mark.gpu
def test_cache_accepted_as_graph_input(data, tmp_path):
    sys.path.insert(0, str(REPO))
    import paper_1912_01478_b200 as hc

    cache = tmp_path / "k3.npz"
    hc.save_csr_cache(hc.load_graph(data / "k3.mtx"), cache)
    proc = run_cli("stats", cache)
    assert proc.returncode == 0 and proc.stdout.strip() == "3 nodes, 3 edges, δ 2/2/2"
