"""One rank of the CPU (gloo) multi-process tests, launched by tests/test_multiproc_cpu.py
under torch.distributed.run: the host side of the N>1 path — peer-handle exchange with the
plan-agreement check, the bench's cross-rank timing helpers, and the sharded protocol
(slice -> owner push, rank-ordered aggregate + SGD at the owner, broadcast) over a real
two-process transport with our C-ABI plan, checked against the reference's digests. Each
rank writes its results to $P3_MP_OUT/rank<r>.json."""
import json
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))

import numpy as np
import torch.distributed as dist

import p3_oracle as orc  # test infrastructure: the checker's math
from paper_1905_03960_b200.model import builtin_profile
from paper_1905_03960_b200.plan import PlanError, make_p3_plan, plan_to_csv
from paper_1905_03960_b200.runtime import exchange_peer_handles, plan_fingerprint


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    out = {"rank": rank, "world": world}

    # 1. handle exchange in rank order, refused when the plans differ
    fp = plan_fingerprint([10, 20], world, 50_000, "p3", 10**6, 0, True, 0.1, 0.0, "fp32")
    got = exchange_peer_handles(bytes([rank]) * 64, fp)
    out["exchange_order"] = got == [bytes([r]) * 64 for r in range(world)]
    bad = plan_fingerprint([10, 20 + rank], world, 50_000, "p3", 10**6, 0, True, 0.1, 0.0, "fp32")
    try:
        exchange_peer_handles(bytes([rank]) * 64, bad)
        out["mismatch_refused"] = False
    except PlanError:
        out["mismatch_refused"] = True

    # 2. bench timing helpers: the max over ranks
    sys.path.insert(0, str(REPO))
    import bench

    out["max_over_ranks"] = bench.max_over_ranks(float(rank + 1), world) == float(world)
    bench.barrier(world)

    # 3. the sharded protocol over gloo with the C-ABI plan
    results = {}
    for name, iters, distinct in (("resnet50-like", 4, True), ("toy3", 10, False)):
        prof = builtin_profile(name)
        counts = prof.param_counts()
        plan = make_p3_plan(prof, world)
        csvs = [None] * world
        dist.all_gather_object(csvs, plan_to_csv(plan))
        agree = len(set(csvs)) == 1
        params = [np.zeros(c, np.float32) for c in counts]
        seed = orc.rank_seed(prof.seed, rank, distinct)
        for k in range(iters):
            # push: every slice's gradient to its owner (the payload of a PUSH frame)
            mine = {}
            for i, s in enumerate(plan.slices):
                g = orc.grad_block(seed, k, s.key.layer_index, s.offset, s.length)
                mine[i] = g.tobytes()
            boxes = [None] * world
            dist.all_gather_object(boxes, {i: b for i, b in mine.items()})
            # owner: rank-ordered aggregate + SGD of its slices; then broadcast
            updated = {}
            for i, s in enumerate(plan.slices):
                if s.server != rank:
                    continue
                L = s.key.layer_index
                cur = params[L][s.offset : s.offset + s.length]
                grads = {r: np.frombuffer(boxes[r][i], np.float32) for r in range(world)}
                updated[i] = orc.shard_update(cur, grads, 0.1).tobytes()
            bc = [None] * world
            dist.all_gather_object(bc, updated)
            for part in bc:
                for i, b in part.items():
                    s = plan.slices[i]
                    params[s.key.layer_index][s.offset : s.offset + s.length] = np.frombuffer(b, np.float32)
        results[name] = {"plan_agree": agree, "digest": f"{orc.digest(params):016x}", "iters": iters,
                         "distinct": distinct}
    out["protocol"] = results

    # 4. the NVLS bootstrap (runtime.connect_nvls): arena and multicast descriptors travel over
    # Unix sockets; a stand-in context hands out descriptors of files and records what arrives
    import tempfile

    from paper_1905_03960_b200.runtime import connect_nvls

    class FdCtx:
        fingerprint = "same-plan"

        def __init__(self):
            self.dir = tempfile.mkdtemp()
            self.calls = []

        def _fd(self, name):
            return os.open(os.path.join(self.dir, name), os.O_CREAT | os.O_RDWR)

        def export_fd(self, li):
            fd = self._fd("arena")
            self.arena = os.fstat(fd).st_ino
            return fd

        def nvls_create(self):
            fd = self._fd("mc")
            self.mc = os.fstat(fd).st_ino
            return fd

        def open_peers_fd(self, fds):
            self.calls.append("open")
            self.peers = [os.fstat(f).st_ino if f >= 0 else None for f in fds]

        def nvls_attach(self, fd):
            self.calls.append("attach")
            self.mc_seen = os.fstat(fd).st_ino if fd >= 0 else getattr(self, "mc", None)

        def nvls_bind(self):
            self.calls.append("bind")

    fc = FdCtx()
    connect_nvls(fc)
    ids = [None] * world
    dist.all_gather_object(ids, (fc.arena, getattr(fc, "mc", None)))
    out["nvls_bootstrap"] = (fc.calls == ["open", "attach", "bind"]
                             and all(fc.peers[r] == (None if r == rank else ids[r][0]) for r in range(world))
                             and fc.mc_seen == ids[0][1] and ids[0][1] is not None)
    Path(os.environ["P3_MP_OUT"], f"rank{rank}.json").write_text(json.dumps(out))
    dist.destroy_process_group()


main()
