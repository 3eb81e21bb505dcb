"""The reference's own unit tests, unmodified, against this package.

``import p3sync`` is redirected by a shim package (written to a temp dir) to
``paper_1905_03960_b200``'s modules, and the reference's test files under
``/root/reference/pkg/tests`` are run by pytest in a subprocess. Only present in the
development container (the reference tree does not exist on the GPU box), so these tests
are skipped elsewhere.

Deselected, with the reason:
  * GradGen tests of test_hashing.py (``gradient*``, ``gradgen*``): ``gradient_block`` runs
    the K1 device kernel, and this suite runs without a GPU. The same golden vectors
    (tests/test_hashing.py:19-34 of the reference) are asserted on the GPU in
    tests/test_gpu_kernels.py.
  * test_server.py (ShardState.aggregate_and_update runs K4 on the device; its known answers
    are GPU tests in tests/test_gpu_kernels.py), test_transport.py / test_runtime.py /
    test_cli.py (TCP sockets and process orchestration: out of scope).
Hypothesis runs with a fixed seed: ``test_sweep_monotone_without_overhead_fifo`` states a
property the reference's own simulator violates on some inputs (e.g. 4 layers, stages
(0,0,0),(0,0,0),(2,0,2),(2,4,2), aggressive-sliced: makespan 8 at slice 2, 9 at slice 1 —
identical timelines from the reference and from p3_simulate), so an unseeded run can fail on
the reference itself.
"""

import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
REPO = Path(__file__).resolve().parents[1]

SHIM = '''import importlib, sys
import paper_1905_03960_b200 as _pkg
for _n in ("plan", "hashing", "queues", "sim", "proto", "model", "metrics", "server"):
    sys.modules["p3sync." + _n] = importlib.import_module("paper_1905_03960_b200." + _n)
from paper_1905_03960_b200 import *  # noqa: F401,F403
'''

CASES = [
    ("test_plan.py", None, 26),
    ("test_proto.py", None, 15),
    ("test_sim.py", None, 23),
    ("test_queues.py", None, 10),
    ("test_metrics.py", None, 10),
    ("test_model.py", None, 20),
    ("test_hashing.py", "not gradient and not gradgen", 6),
]


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference tree not mounted (GPU box)")
@pytest.mark.parametrize("fname,select,n", CASES)
def test_reference_unit_tests_pass(tmp_path, fname, select, n):
    shim = tmp_path / "shim" / "p3sync"
    shim.mkdir(parents=True)
    (shim / "__init__.py").write_text(SHIM)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--hypothesis-seed=0",
           str(REF_TESTS / fname)]
    if select:
        cmd += ["-k", select]
    env = {"PYTHONPATH": f"{tmp_path / 'shim'}:{REPO}", "PATH": "/usr/bin:/bin", "HOME": str(tmp_path)}
    r = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert f"{n} passed" in tail, tail
