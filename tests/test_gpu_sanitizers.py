"""compute-sanitizer over a small workload that launches every kernel variant
(tools/sanitize_run.py): no memory errors, no shared-memory races (the
exchanges rely on a single barrier each and on warp-synchronous transposes),
no barrier misuse.  SURVEY.md section 5 (race detection)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,summary", [("memcheck", "ERROR SUMMARY: 0 errors"),
                                          ("racecheck", "0 errors, 0 warnings"),
                                          ("synccheck", "ERROR SUMMARY: 0 errors")])
def test_sanitizer_clean(tool, summary):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    out = subprocess.run([exe, "--tool", tool, "--print-limit", "5", sys.executable,
                          os.path.join(ROOT, "tools", "sanitize_run.py")],
                         capture_output=True, text=True, timeout=900)
    text = out.stdout + out.stderr
    assert "sanitize workload done" in text, text[-2000:]
    assert summary in text, text[-2000:]
