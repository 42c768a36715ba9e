"""The §3 micro-benchmark pair (reference bench.py / test_bench.py)."""

import io
import math

import numpy as np
import pytest

from paper_1912_01478_b200.pushbench import (
    BenchConfig,
    TtiRecord,
    TtiSeries,
    collect_deactivations,
    detect_crossovers,
    expected_iterations,
    run_push_bench,
    write_tti_csv,
)


def series(variant, micros):
    return TtiSeries(variant, [TtiRecord(t, 0, m, m, 0.0) for t, m in enumerate(micros)])


# ---------------------------------------------------------------- host logic (CPU)
def test_config_defaults_and_validation():  # test_bench.py:29-40
    cfg = BenchConfig()
    assert cfg.batch_size == 1000 and cfg.repetitions == 10
    for bad in (dict(batch_size=0), dict(repetitions=0), dict(variant="push_maybe")):
        with pytest.raises(ValueError):
            BenchConfig(**bad)


def test_crossovers_and_csv():  # test_acceptance.py:220-224
    assert detect_crossovers(series("push_wl", [5, 5, 5]), series("push_nowl", [3, 3, 8])) == [2]
    assert detect_crossovers(series("push_wl", [4, 4]), series("push_nowl", [4, 4])) == []
    assert detect_crossovers(series("push_wl", [9, 9]), series("push_nowl", [1, 1])) == []
    with pytest.raises(ValueError):
        detect_crossovers(series("push_wl", [1]), series("push_nowl", [1, 2]))
    buf = io.StringIO()
    write_tti_csv(buf, [series("push_wl", [1.5])])
    assert buf.getvalue().splitlines() == ["variant,iteration,active_before,micros_mean,micros_min,micros_std",
                                           "push_wl,0,0,1.500,1.500,0.000"]
    assert expected_iterations(2500, 1000) == 3


# ---------------------------------------------------------------- device pipe
@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["push_wl", "push_nowl"])
def test_iteration_arithmetic(variant):  # test_bench.py:44-61
    s = run_push_bench(2500, BenchConfig(variant=variant, repetitions=2))
    assert [r.active_before for r in s.per_iteration] == [2500, 1500, 500]
    assert s.iterations() == [0, 1, 2]
    assert len(run_push_bench(1000, BenchConfig(repetitions=1)).per_iteration) == 1
    assert len(run_push_bench(10, BenchConfig(batch_size=1000, repetitions=1)).per_iteration) == 1
    assert all(r.micros_min > 0 and r.micros_mean >= r.micros_min for r in s.per_iteration)


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch", [(1000, 1000), (2500, 1000), (10000, 1000), (123457, 777)])
def test_equal_work(n, batch):  # test_acceptance.py:206-218
    per_variant = [collect_deactivations(n, BenchConfig(batch_size=batch, variant=v)) for v in ("push_wl", "push_nowl")]
    wl, nowl = per_variant
    assert len(wl) == len(nowl) == math.ceil(n / batch)
    assert all(np.array_equal(a, b) for a, b in zip(wl, nowl))
    assert np.array_equal(np.concatenate(wl), np.arange(n))  # every node deactivated exactly once
    assert all(len(d) == batch for d in wl[:-1])
