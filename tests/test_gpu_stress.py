"""Stress: the speckled-phantom matrix of tools/stress_cases.py (3 flip
fractions x 4 seeds x both walk modes x 1 / 2 pipelines, variance tracking)
in a subprocess with a hard time limit, so a hang fails the test instead of
stalling the suite.  Every wavefront run must equal the megakernel bit for
bit (the engines share the per-history arithmetic and the integer tallies).
DESIGN.md §4.1 "Queue pushes and guards" has the history of the hang."""
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_speckled_matrix_finishes_and_engines_agree():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "stress_cases.py"), "4"], capture_output=True,
                       text=True, timeout=600, cwd=str(ROOT))
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "ALL OK" in r.stdout, r.stdout[-3000:]
    assert r.stdout.count(" ok ") == 3 * 4 * 2 * 2
