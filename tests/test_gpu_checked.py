"""The checked build (libp3_checked.so: protocol invariants compiled in — one push per rank
and slice per iteration, pops consistent with the plan, servers reduce only what they own,
stage bounds): end-to-end runs in a subprocess must finish with the oracle's parameters and
no violated check."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
CHECKED = REPO / "paper_1905_03960_b200" / "libp3_checked.so"

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,mode,ctas", [(1, "p3", 148), (2, "p3", 4), (3, "p3", 148), (4, "baseline", 16)])
def test_checked_build_end_to_end(cuda, world, mode, ctas):
    if not CHECKED.exists():
        pytest.fail(f"{CHECKED} missing: build with paper_1905_03960_b200/csrc/build.sh")
    env = dict(os.environ, P3_LIB=str(CHECKED))
    p = subprocess.run([sys.executable, str(REPO / "tools" / "sanitize_small.py"), str(world), mode, str(ctas)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0 and "OK" in p.stdout, p.stdout[-2000:] + p.stderr[-3000:]
    assert "P3_CHECK failed" not in p.stdout + p.stderr
