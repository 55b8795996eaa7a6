"""The C ABI from plain C (examples/sweep_c.c, no Python or torch in the process): the sweep
plan over a batch of rotations with host buffers, each rotation's grid extrema checked by the
program against the exact single-configuration query at the same translations (1e-4)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_consumer_sweep():
    subprocess.check_call(["make", "-C", ROOT, "-s", "examples"])
    r = subprocess.run([os.path.join(ROOT, "examples", "sweep_c"), "8"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "OK"
    assert sum(ln.startswith("rot ") for ln in lines) == 8
