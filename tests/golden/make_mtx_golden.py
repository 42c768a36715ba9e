"""Golden fixtures for graph ingestion, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_mtx_golden.py

For a corpus of MatrixMarket texts -- the reference's own test cases
(pkg/tests/test_graph_core.py:21-94) plus seeded fuzz: valid files with
comments, blank lines, extra value columns, every ASCII whitespace byte,
signs, leading zeros and underscores, and files broken in every way the
parser checks (too few fields, non-integers, bounds, counts, banner / size
line) -- it records what `hybridcolor.parse_matrix_market` returns (edges) or
raises (message), for str input and for a file read by `load_graph` (text
mode, universal newlines; CRLF / CR variants).  It also records
`degree_stats` on seeded graphs.  Written to tests/golden/mtx.json.
"""

from __future__ import annotations

import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import load_reference  # noqa: E402

BANNERS = ["%%MatrixMarket matrix coordinate pattern general",
           "%%MatrixMarket matrix coordinate real symmetric",
           "%%matrixmarket MATRIX Coordinate integer general"]
WS = [" ", "\t", "\x0b", "\x0c", "\x1c", "\x1f", "  ", " \t "]


def ref_cases():
    b = "%%MatrixMarket matrix coordinate pattern general\n"
    return [
        b + "3 3 2\n1 2\n2 3\n",
        "%%MatrixMarket matrix coordinate real general\n3 3 0\n",
        b + "3 3 1\n4 1\n",
        b + "3 3 1\n0 1\n",
        "%%MatrixMarket matrix array real general\n3 3 2\n",
        "% not a banner\n3 3 2\n",
        "",
        "%%MatrixMarket matrix coordinate real general\n3 3 1\n1.5 2\n",
        "%%MatrixMarket matrix coordinate real general\n3 3 1\na b\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.75\n",
        "%%MatrixMarket matrix coordinate pattern symmetric\n% comment\n\n3 3 2\n% another\n1 2\n\n2 3\n",
        "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 2\n2 3\n",
        b + "3 3 2\n1 2\n",
        b + "3 3 1\n1 2\n2 3\n",
        b + "2 2 1\n2 1\n",
        b + "2 5 1\n1 4\n",
        # header edge cases
        b, b + "% only comments\n", b + "3 3\n", b + "3 x 3\n", b + "3 -3 1\n", b + "3 3 1 1\n",
        "\n3 3 1\n1 1\n", "%%MatrixMarket matrix\n3 3 1\n",
        # entry edge cases
        b + "3 3 1\n1\n", b + "3 3 1\n+1 +2\n", b + "3 3 1\n-1 2\n", b + "3 3 1\n001 0_2\n",
        b + "3 3 1\n1_ 2\n", b + "3 3 1\n_1 2\n", b + "3 3 1\n1__2 2\n", b + "3 3 1\n1 99999999999999999999999\n",
        b + "3 3 1\n1 2e0\n", b + "3 3 1\n0x1 2\n", b + "3 3 1\n%1 2\n", b + "3 3 1\n  % c\n 1\t2  \n",
        b + "3 3 2\n1 2\n3\n3 3\n", b + "3 3 2\n1 2\n3 3\n4 4\n", b + "3 3 2\n1 2\n3 3\n1\n",
        b + "3 3 1\n1 2\n9 9\n", b + "3 3 1\n1 2 extra fields here\n", b + "1 1 1\n1 1",
        b + "3 3 0\n\n\n% x\n", b + "3 3 1\n+ 1\n", b + "3 3 1\n- 1\n", b + "3 3 1\n1 2\x0b3\n",
    ]


def fuzz_cases(rng: random.Random, count: int):
    out = []
    for _ in range(count):
        rows, cols = rng.randint(1, 60), rng.randint(1, 60)
        nnz = rng.randint(0, 40)
        lines = [rng.choice(BANNERS)]
        for _ in range(rng.randint(0, 2)):
            lines.append(rng.choice(["%c", "", "  ", "% " + "x" * rng.randint(0, 5)]))
        lines.append(f"{rows} {cols} {nnz}")
        entries = []
        for _ in range(nnz):
            r, c = rng.randint(1, rows), rng.randint(1, cols)
            fr, fc = str(r), str(c)
            if rng.random() < 0.1:
                fr = "+" + fr
            if rng.random() < 0.1:
                fc = "0" * rng.randint(1, 3) + fc
            if rng.random() < 0.05 and len(fr) > 1 and fr[-1].isdigit() and fr[-2].isdigit():
                fr = fr[:-1] + "_" + fr[-1]
            sep = rng.choice(WS)
            line = rng.choice(["", " ", "\t"]) + fr + sep + fc
            if rng.random() < 0.2:
                line += rng.choice(WS) + rng.choice(["1.5", "-3", "x", "1e9"])
            entries.append(line + rng.choice(["", " ", "\t"]))
        # interleave comments / blank lines
        body = []
        for e in entries:
            if rng.random() < 0.1:
                body.append(rng.choice(["% cm", "", "   ", "\t"]))
            body.append(e)
        # corrupt some files
        kind = rng.random()
        if body and kind < 0.4:
            i = rng.randrange(len(body))
            body[i] = rng.choice([
                "1", "x 1", "1 y", "1.0 2", f"{rows + 1} 1", f"1 {cols + 1}", "0 1", "-1 1", f"{rows} 0",
                "1__1 1", "_1 1", "1_ 1", "+ 1", "1 +", "++1 1"])
        elif kind < 0.5:
            body.append(f"{rng.randint(1, rows)} {rng.randint(1, cols)}")  # one too many
        elif kind < 0.6 and body:
            body.pop(rng.randrange(len(body)))  # one too few
        lines += body
        text = "\n".join(lines) + rng.choice(["\n", "", "\n\n"])
        out.append(text)
    return out


def run_parse(ref, text):
    try:
        el = ref.parse_matrix_market(text)
        return {"n": int(el.num_nodes_declared), "edges": el.edges.astype(int).reshape(-1).tolist()}
    except ref.MatrixMarketError as exc:
        return {"error": str(exc)}


def run_load(ref, raw: bytes):
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "g.mtx"
        p.write_bytes(raw)
        try:
            g = ref.load_graph(p)
            return {"n": int(g.num_nodes), "ro": g.row_offsets.astype(int).tolist(),
                    "ci": g.col_indices.astype(int).tolist()}
        except ref.MatrixMarketError as exc:
            return {"error": str(exc)}


def main():
    ref, conf = load_reference()
    rng = random.Random(20261017)
    texts = ref_cases() + fuzz_cases(rng, 300)
    parse = [{"text": t, "out": run_parse(ref, t)} for t in texts]
    files = []
    for t in texts[:16] + texts[60:140]:
        for nl in ("\n", "\r\n", "\r"):
            raw = t.replace("\n", nl).encode("ascii")
            files.append({"raw": raw.decode("ascii"), "out": run_load(ref, raw)})
    deg = []
    nrng = np.random.default_rng(11)
    for n, m in ((1, 0), (2, 1), (7, 12), (100, 300), (1001, 5000), (4096, 40000), (3, 0)):
        e = nrng.integers(0, n, (m, 2)) if m else np.zeros((0, 2), np.int64)
        g = ref.build_csr(ref.EdgeList(n, e))
        s = ref.degree_stats(g)
        deg.append({"n": n, "ro": g.row_offsets.astype(int).tolist(), "ci": g.col_indices.astype(int).tolist(),
                    "stats": [s.min_degree, s.median_degree, s.max_degree, s.num_nodes, s.num_undirected_edges]})
    for name, g in (("path3", conf.path_graph(3)), ("clique3", conf.clique_graph(3)), ("star3", conf.star_graph(3))):
        s = ref.degree_stats(g)
        deg.append({"n": g.num_nodes, "ro": g.row_offsets.astype(int).tolist(),
                    "ci": g.col_indices.astype(int).tolist(),
                    "stats": [s.min_degree, s.median_degree, s.max_degree, s.num_nodes, s.num_undirected_edges]})
    (HERE / "mtx.json").write_text(json.dumps({"parse": parse, "files": files, "degree_stats": deg}))
    nerr = sum("error" in c["out"] for c in parse)
    print(f"mtx.json: {len(parse)} parse cases ({nerr} errors), {len(files)} file cases, {len(deg)} degree cases")


if __name__ == "__main__":
    main()
