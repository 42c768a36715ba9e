"""CPU: host-side API semantics that need no device (driver.py:29-119)."""

import io
import json

import pytest

from paper_1912_01478_b200 import (
    HybridConfig,
    RoundRecord,
    RunReport,
    available_backends,
    get_kernels,
    threshold_count,
)


def test_config_defaults_and_validation():  # test_driver.py:11-27
    cfg = HybridConfig()
    assert cfg.threshold_fraction == 0.6 and cfg.mode == "hybrid"
    for bad in (-0.1, 1.5):
        with pytest.raises(ValueError):
            HybridConfig(threshold_fraction=bad)
    with pytest.raises(ValueError):
        HybridConfig(mode="gpu")
    with pytest.raises(ValueError):
        HybridConfig(workers=0)
    with pytest.raises(ValueError):
        HybridConfig(chunk_size=0)


def test_threshold_arithmetic():  # driver.py:138
    assert threshold_count(HybridConfig(threshold_fraction=0.6), 3) == 2
    assert threshold_count(HybridConfig(threshold_fraction=0.0), 10) == 0
    assert threshold_count(HybridConfig(threshold_fraction=1.0), 10) == 10
    assert threshold_count(HybridConfig(threshold_fraction=0.6), 4096 * 4096) == 10066330


def test_backend_registry_has_no_fallback():
    assert available_backends() == ("cuda",)
    assert get_kernels("auto").NAME == "cuda"
    with pytest.raises(ValueError, match="not available"):
        get_kernels("python")


def _report():
    rep = RunReport("k3", 3, 3, HybridConfig())
    rep.per_round = [RoundRecord(1, "topo", 3, 2, 3, 1e-5), RoundRecord(2, "data", 2, 1, 1, 2e-5),
                     RoundRecord(3, "data", 1, 0, 0, 3e-5)]
    rep.total_rounds, rep.colors_used, rep.valid = 3, 3, True
    return rep


def test_report_json_shape():  # test_driver.py:100-130 / driver.py:69-100
    doc = json.loads(_report().to_json())
    assert set(doc) == {"graph", "num_nodes", "num_undirected_edges", "config", "colors_used",
                        "valid", "total_rounds", "total_micros", "per_round"}
    assert set(doc["per_round"][0]) == {"round", "mode", "wl_in", "wl_out", "conflicts", "micros"}


def test_report_csv_and_table():
    buf = io.StringIO()
    _report().write_round_csv(buf)
    lines = buf.getvalue().strip().splitlines()
    assert lines[0] == "round,mode,wl_in,wl_out,conflicts,micros"
    assert lines[1].startswith("1,topo,3,2,3,")
    assert _report().rows_table().splitlines()[0].split() == ["round", "mode", "wl_in", "wl_out",
                                                             "conflicts", "micros"]
