"""The reference's own test suite (pkg/tests, copied into oracle/_ref/tests by
oracle/build_ref.sh) run UNMODIFIED against this package's `cuda` kernel
module (the reference suite is the parity harness).

tests/refsuite_plugin.py registers the module in the reference's backend
registry; `-m gpu` because every cuda-parametrised case runs the libhcb kernels.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
SUITE = REPO / "oracle" / "_ref" / "tests"


def _run(files, default_cuda: bool):
    if not SUITE.is_dir():
        pytest.fail("oracle/_ref/tests missing: run oracle/build_ref.sh (or __graft_entry__.build())")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REPO / "tests"), str(REPO), str(REPO / "oracle" / "_ref")])
    env["HCREF_DEFAULT_CUDA"] = "1" if default_cuda else "0"
    cmd = [sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-q", "-rA", "-p", "no:cacheprovider",
           *[str(SUITE / f) for f in files]]
    out = subprocess.run(cmd, cwd=str(SUITE), env=env, capture_output=True, text=True, timeout=1800)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-6000:]
    return text


def test_reference_kernel_tests_on_cuda_backend():
    """test_coloring / test_bench / test_backends: the `kernels` fixture
    (conftest.py:110-113) includes `cuda`; the backend-agreement tests compare
    cuda's colorings, trajectories and deactivation sets with cython's and
    python's (test_backends.py:36-69)."""
    text = _run(["test_coloring.py", "test_bench.py", "test_backends.py"], default_cuda=False)
    cuda_passed = re.findall(r"^PASSED .*\[.*cuda.*\]", text, re.M)
    assert len(cuda_passed) >= 17, text[-4000:]  # 17 cuda-parametrised cases in the reference suite
    assert "FAILED" not in text and "ERROR" not in text


def test_whole_reference_suite_with_cuda_as_default_backend():
    """Every test file of the reference, with `_backend.kernels` = cuda, so
    color_graph, the iterations and the push bench all run the GPU kernels."""
    text = _run(sorted(p.name for p in SUITE.glob("test_*.py")), default_cuda=True)
    assert "default cuda" in text
    assert "FAILED" not in text and "ERROR" not in text
