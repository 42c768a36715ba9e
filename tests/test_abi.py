"""CPU: the C-ABI library loads and exports every entry point include/hcb.h
declares (no compute calls without a GPU)."""

import ctypes
import re

from conftest import REPO


def declared_symbols():
    text = (REPO / "include" / "hcb.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(hc_\w+)\s*\(", text, re.M)))


def test_header_declares_plugin_surface():
    names = declared_symbols()
    for fn in ("assign_from_list", "assign_sweep", "resolve_from_list", "resolve_sweep",
               "bench_from_list", "bench_sweep"):  # _kernels.pyx:29-187
        assert f"hc_k_{fn}" in names
    assert "hc_solve" in names and "hc_build_csr" in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(REPO / "paper_1912_01478_b200" / "libhcb.so"))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1912_01478_b200 import _lib

    assert set(declared_symbols()) == set(_lib.EXPORTED_SYMBOLS)
    L = _lib.load()
    assert L.hc_version() == 1
    assert L.hc_solve_workspace_bytes(1000, 5000) > 16 * 1000


def test_product_does_not_import_oracle():
    pkg = REPO / "paper_1912_01478_b200"
    for path in pkg.rglob("*.py"):
        src = path.read_text()
        assert "from oracle" not in src and "import oracle" not in src, path
