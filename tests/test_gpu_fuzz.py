"""Short randomised parity sweeps (fixed seeds) as part of the GPU suite: random
classification shapes / launch plans vs the bit-packed kernel (and the host-fed path),
random sampling / encoding cases vs the oracle, random Stage 1 + Stage 2 runs and whole
multistate PMFs vs the oracle.  The long runs are in profiles/r2_fuzz_parity.txt."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,seed", [("fuzz_parity.py", "11"), ("fuzz_workflow.py", "12")])
def test_random_cases_match(tool, seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool), "25"], cwd=ROOT,
                       env=dict(os.environ, SEED=seed), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "equal" in r.stdout and "MISMATCH" not in r.stdout, r.stdout[-2000:]
