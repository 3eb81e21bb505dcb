"""World-size-2 gloo runs of the N>1 host logic (no GPU): see tests/mp/cpu_worker.py."""

import json
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def test_two_rank_host_logic(golden, tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29621", str(REPO / "tests" / "mp" / "cpu_worker.py")]
    env = dict(os.environ, P3_MP_OUT=str(tmp_path), CUDA_VISIBLE_DEVICES="")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.loads(f.read_text()) for f in sorted(tmp_path.glob("rank*.json"))]
    assert len(res) == 2
    want = {(d[0], d[1], d[2], d[4]): d[5] for d in golden["digests"]}
    for r in res:
        assert r["exchange_order"] and r["mismatch_refused"] and r["max_over_ranks"], r
        assert r["nvls_bootstrap"], r
        for name, v in r["protocol"].items():
            assert v["plan_agree"], (r["rank"], name)
            key = (name, 2, v["iters"], "distinct" if v["distinct"] else "same")
            assert v["digest"] == want[key], (r["rank"], name, v["digest"], want[key])
