"""bench.py's host-side helpers (no GPU): the config strings the JSON line
carries and the SURVEY.md 8(d) sweep-count formula."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class _Args:
    def __init__(self, n, p, graph="u3r"):
        self.n, self.p, self.graph = n, p, graph


def test_l2_note_reflects_per_gpu_state_size():
    assert bench.l2_note(16 << 30).startswith("no flush: 16 GiB")
    assert bench.l2_note(16 << 30, 8).startswith("no flush: 2 GiB")
    assert "L2-resident" in bench.l2_note(16 << 20)          # N=20: 16 MiB
    assert "partly L2-resident" in bench.l2_note(16 << 24)   # N=24: 256 MiB


def test_workload_names_tag_the_baseline_configs():
    assert "BASELINE configs[2]" in bench.workload_name(_Args(30, 10))
    assert "BASELINE configs[3]" in bench.workload_name(_Args(33, 4, "er"))
    assert "BASELINE configs[1]" in bench.workload_name(_Args(26, 4))
    odd = bench.workload_name(_Args(31, 4))
    assert "isolated node" in odd and "custom" in odd


def test_r_star_formula():
    # R*(N) = 1 + ceil(max(0, N - 13) / 10)
    r = lambda n: 1 + -(-max(0, n - 13) // 10)  # noqa: E731  (the expression bench.py uses)
    assert [r(n) for n in (12, 13, 20, 23, 24, 26, 30, 33, 34)] == [1, 1, 2, 2, 3, 3, 3, 3, 4]


def test_sweep_kinds_from_the_engine_plan():
    """The bench's roofline picks the dominant sweep kind from qaoa_plan (CPU,
    no device): N=30 p=10 is 1 launch-control + 10 low-set + 9 merged + 1 last."""
    import bench
    from paper_2312_03019_b200 import _lib

    kinds = bench.sweep_kinds(_lib.load(), 30, 10, False, 21)
    assert kinds[0].startswith("launch-control") and kinds[-1].startswith("last")
    assert kinds.count("merged level-boundary sweep") == 9
    assert kinds.count("low-set sweep S0") == 10
    assert bench.sweep_kinds(_lib.load(), 30, 10, False, 20) == ["sweep"] * 20
