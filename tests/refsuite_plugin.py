"""pytest plugin: run the REFERENCE's own test suite against the `cuda` kernel module.

Loaded with `-p refsuite_plugin` before the reference's conftest imports
`hybridcolor` (oracle/_ref, the reference package built by oracle/build_ref.sh;
its tests are copied to oracle/_ref/tests).  It registers this package's
kernel module (paper_1912_01478_b200.kernels, NAME "cuda") in the reference's
backend registry (pkg/src/hybridcolor/_backend.py:15-21), so

  * the `kernels` fixture (pkg/tests/conftest.py:110-113) parametrises every
    kernel-level test over ("cuda", "cython", "python"), and the backend
    agreement tests (test_backends.py:36-69) compare cuda with the others;
  * with HCREF_DEFAULT_CUDA=1 the reference's default module
    (`_backend.kernels`, coloring.py:125/158, bench.py:109/142) becomes cuda
    too, so every color_graph / iteration / push-bench call of the whole
    suite (driver, acceptance, CLI tests) runs on the GPU kernels.

Nothing of the reference is modified; it is the unmodified suite with one
more registered backend.  Test infrastructure only (tests/test_reference_suite.py).
"""

import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "oracle" / "_ref"
for p in (str(REF), str(REPO)):
    if p not in sys.path:
        sys.path.insert(0, p)

import hybridcolor._backend as _ref_backend  # noqa: E402

from paper_1912_01478_b200 import kernels as _cuda_kernels  # noqa: E402

_ref_backend._BACKENDS[_cuda_kernels.NAME] = _cuda_kernels
if os.environ.get("HCREF_DEFAULT_CUDA") == "1":
    _ref_backend.kernels = _cuda_kernels


def _banner():
    return (f"refsuite_plugin: reference backends {_ref_backend.available_backends()}, "
            f"default {_ref_backend.backend_name()}")


def pytest_report_header(config):
    return _banner()


def pytest_terminal_summary(terminalreporter):
    # also under -q, where the report header is not printed
    terminalreporter.write_line(_banner())
