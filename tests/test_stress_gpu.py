"""Randomised parity stress (tools/stress.py): random complete/partial DFAs of 1..3000 states
and 1..256 symbols, inputs with runs / zeros / invalid bytes, chunk lengths from one byte,
every boundary and candidate rule -- match results and match positions against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_randomised_stress(cuda_device):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress.py"), "300"], capture_output=True,
                       text=True, env=dict(os.environ, STRESS_BASE="900000"), timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "mismatches: 0" in r.stdout, r.stdout[-3000:]
