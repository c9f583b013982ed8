"""The reference's own tests, unmodified, against the drop-in.

tools/stage_reference.sh stages the reference package and its pytest files
under baseline/_ref (git-ignored; the directory travels to the GPU box with
the repo snapshot).  Each case below runs one reference test file in a fresh
interpreter with tools/zt_ref_plugin.py rebinding zeitlin's hot path (stream
solve, apply, residual gates, fixed point, midpoint step, the names the
driver and diagnostics bound at import) to paper_2206_05466_b200, and
requires every selected test to pass and the plugin to have intercepted
calls.  Selection: test_laplacian.py and test_integrator.py in full (fast and
slow cases), and test_acceptance.py criteria c2-c7 plus the N = 64 structure
and eigenvalue checks (c1 is the out-of-scope basis oracle, c8 a 37-minute
spectrum run).
"""

import os
import re
import subprocess
import sys

import pytest
from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "zeitlin_tests")

CASES = [
    ("test_laplacian.py", None),
    ("test_integrator.py", None),
    ("test_acceptance.py", "c2 or c3 or c4 or c5 or c6 or c7 or n64"),
]


@pytest.mark.skipif(not os.path.isdir(TESTS), reason="reference not staged (tools/stage_reference.sh)")
@pytest.mark.parametrize("fname,select", CASES)
def test_reference_file_passes_unmodified(fname, select, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, TESTS, os.path.join(ROOT, "tools"), ROOT])
    env.setdefault("NUMBA_CACHE_DIR", str(tmp_path / "numba"))
    cmd = [sys.executable, "-m", "pytest", "-p", "zt_ref_plugin", "-q", "-p", "no:cacheprovider",
           "--rootdir", TESTS, os.path.join(TESTS, fname)]
    if select:
        cmd += ["-k", select]
    out = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=3000)
    tail = out.stdout[-4000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    m = re.search(r"(\d+) passed", out.stdout)
    assert m and int(m.group(1)) > 0, tail
    assert "failed" not in out.stdout.splitlines()[-1], tail
    calls = re.search(r"zt_ref_plugin intercepted calls: (.*)", out.stdout)
    assert calls and "solve_stream=" in calls.group(1), tail
    print(f"{fname}: {m.group(0)}; {calls.group(1)}")
