"""The reference package's OWN test suite (mfglobal 0.1.0, 235 tests) with
its Omega path routed to libmfg_b200 by paper_2204_14067_b200.refplug
(pair_values, the BCD half-sweep, ShiftedOperator.apply/apply_t/
project_rows). Needs the reference installed with its tests under
baseline/_ref (pip install --target baseline/_ref, tests
copied beside it); skipped when that install is absent."""

import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

REF = os.path.join(REPO, "baseline", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="reference install (baseline/_ref) not present")
def test_reference_suite_passes_on_our_kernels():
    env = dict(os.environ, PYTHONPATH=f"{REF}:{REPO}", PYTHONDONTWRITEBYTECODE="1")
    res = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-p", "no:cacheprovider",
                          "-p", "paper_2204_14067_b200.refplug_pytest"],
                         cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    tail = res.stdout[-3000:]
    print(tail)
    assert res.returncode == 0, tail
    assert "routed calls" in res.stdout and "'pair_values': 0" not in res.stdout
    assert "'half_sweep': 0" not in res.stdout and "'apply': 0" not in res.stdout
