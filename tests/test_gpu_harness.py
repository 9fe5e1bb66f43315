"""Reference-format benchmark records on the device."""

import pytest

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import harness as H

pytestmark = pytest.mark.gpu


def test_records_and_compare():
    g = H.parse_generator_spec("u3r:n=16,seed=1")
    recs = H.run_simulate(g, 3, "fast", reps=2, with_ratio=True)
    assert len(recs) == 2 and recs[0].total_time_ns > 0
    assert set(recs[0].to_dict()) == set(H.BENCH_CSV_COLUMNS)
    assert 0 < recs[0].approx_ratio <= 1
    rows = H.run_compare([14, 16], ["exact", "fast"], lambda n: Q.random_regular_graph(n, 3, seed=0),
                         p=3, reps=2)
    assert len(rows) == 4 and all(r["max_abs_diff"] <= 1e-12 for r in rows)
    sweep = H.run_sweep_p(g, [1, 4], ["fast"], reps=2)
    assert sweep[0].normalized_time == 1.0
    csv = H.records_to_csv(recs)
    assert csv.splitlines()[0] == ",".join(H.BENCH_CSV_COLUMNS)
    assert H.parse_generator_spec("er:n=33").tot_edge == 236
    with pytest.raises(ValueError):
        H.parse_generator_spec("u3r:seed=1")


def test_compare_gate_level_baseline_vs_fused():
    """The reference's speedup table (bench.py:184-243): gate-level "baseline"
    (one device pass per gate) against the fused "bitwise" engine, behind the
    1e-10 equivalence gate; the baseline's cost and mixer times are split."""
    rows = H.run_compare([16, 18], ["baseline", "bitwise"],
                         lambda n: Q.random_regular_graph(n, 3, seed=0), p=2, reps=1)
    assert len(rows) == 4
    base = [r for r in rows if r["backend"] == "baseline"]
    fused = [r for r in rows if r["backend"] == "bitwise"]
    assert all(r["cost_time_ns"] > 0 and r["mixer_time_ns"] > 0 for r in base)
    assert all(r["max_abs_diff"] <= 1e-12 for r in fused)
    assert all(r["total_speedup"] > 1.0 for r in fused)
