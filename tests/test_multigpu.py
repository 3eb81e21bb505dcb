"""Multi-GPU P3 over NVLink (CUDA IPC peer arenas), one process per GPU under torchrun.
Skipped when fewer than two GPUs are visible."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpu() -> int:
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multiprocess_parity(world, tmp_path):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), str(REPO / "tests" / "mp" / "mp_worker.py")]
    env = dict(os.environ, P3_MP_OUT=str(tmp_path))
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    results = [json.loads(f.read_text()) for f in sorted(tmp_path.glob("rank*.json"))]
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert len(results) == world
    for r in results:
        for k, (got, want) in r["digests"].items():
            assert got == want, (r["rank"], k, got, want)
        assert r["torch_p3_exact"], r
        assert r["torch_layerwise_close"], r
        assert r["torch_p3_distinct_resnet50"], r
        assert r["torch_p3_distinct_seq2seq"], r
        assert r["torch_p3_bf16_replicas"], r
        assert r["nvls"] == "ok" or r["nvls"].startswith("unavailable"), r["nvls"]
        if r["nvls"] == "ok":  # torch-mode training with multicast broadcasts, bit-exact too
            assert r["torch_p3_distinct_resnet50_nvls"], r
        if os.environ.get("P3_EXPECT_NVLS"):  # a box known to have multicast (NVSwitch)
            assert r["nvls"] == "ok" and any(k.endswith("/nvls") for k in r["digests"]), r["nvls"]
