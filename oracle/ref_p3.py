"""The reference's OWN P3 sync path on host cores — BASELINE INFRASTRUCTURE ONLY.

Runs the unmodified reference package installed in ``baseline/_ref`` (``pip install
--target baseline/_ref`` of /root/reference/pkg; git-ignored, shipped to the GPU box with
the snapshot) through its own objects, one synchronous P3 iteration at a time:

  worker side  enqueue_layer -> FrameQueue(priority).put_batch in backward order, then the
               sender's poll order (worker.py:173-190); each worker materialises its push
               with GradGen.block (worker.py:166-171) — N materialisations per slice;
  server side  ShardState.on_push from every rank, then aggregate_and_update (server.py:
               36-68);
  apply side   the updated slice written into every worker's replica (worker.py:241-269).

Sockets, framing and emulated compute are left out (they are not the path being compared).
Slices run on a thread pool (numpy releases the GIL in its kernels). Used by bench.py as
``cpu_baseline`` / ``--impl reference`` with kind "reference" when baseline/_ref exists;
``cpu_p3.CpuP3`` (the numpy restatement, kind "port") otherwise. Never imported by the
product package.
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def available() -> bool:
    return (REF / "p3sync" / "__init__.py").exists()


class RefP3:
    def __init__(self, counts: list[int], world: int, seed: int = 0, lr: float = 0.1, max_slice: int = 50_000,
                 threads: int | None = None) -> None:
        if str(REF) not in sys.path:
            sys.path.insert(0, str(REF))
        from p3sync.hashing import GradGen
        from p3sync.model import LayerSpec, ModelProfile
        from p3sync.plan import make_p3_plan
        from p3sync.proto import Frame, MsgType
        from p3sync.queues import FrameQueue
        from p3sync.server import ShardState

        self._Frame, self._MsgType, self._FrameQueue = Frame, MsgType, FrameQueue
        self.counts = list(counts)
        self.world = world
        profile = ModelProfile("bench", seed, tuple(LayerSpec(i, f"t{i}", c, 0, 0) for i, c in enumerate(counts)))
        self.plan = make_p3_plan(profile, world, max_slice)
        self.rows = self.plan.slices
        self.gen = GradGen(seed)  # the reference pushes the same seed from every rank (worker.py:71)
        self.shards = {s.key: ShardState(s.key, np.zeros(s.length, dtype=np.float32), world, lr) for s in self.rows}
        self.info = {s.key: s for s in self.rows}
        self.replicas = [[np.zeros(c, dtype=np.float32) for c in counts] for _ in range(world)]  # worker.py:72
        self.threads = threads or len(os.sched_getaffinity(0))
        self.pool = ThreadPoolExecutor(self.threads)

    def _slice(self, k: int, key) -> None:
        sl = self.info[key]
        shard = self.shards[key]
        it = shard.iteration
        for r in range(self.world):  # each worker materialises and pushes its gradient
            grad = self.gen.block(k, key.layer_index, sl.offset, sl.length)
            shard.on_push(r, it, grad)
        params = shard.aggregate_and_update()
        for rep in self.replicas:  # BCAST applied by every worker
            rep[key.layer_index][sl.offset : sl.offset + sl.length] = params

    def _order(self, k: int, sample: int | None):
        q = self._FrameQueue(priority_mode=True)
        for layer in reversed(range(len(self.counts))):
            q.put_batch([self._Frame(self._MsgType.PUSH, s.priority, k, 0, s.key.layer_index, s.key.slice_index,
                                     s.offset) for s in self.plan.slices_of_layer(layer)])
        q.close()
        out = []
        while sample is None or len(out) < sample:
            f = q.poll(timeout=1.0)
            if f is None:
                break
            out.append(self.info[(self._key(f))].key)
        return out

    def _key(self, f):
        from p3sync.plan import SliceKey

        return SliceKey(f.layer_index, f.slice_index)

    def time_iteration(self, k: int, sample_slices: int | None = None) -> tuple[float, float]:
        """(seconds, fraction of the iteration's elements covered by the sample)."""
        t0 = time.perf_counter()
        keys = self._order(k, sample_slices)
        list(self.pool.map(lambda key: self._slice(k, key), keys))
        dt = time.perf_counter() - t0
        return dt, sum(self.info[key].length for key in keys) / sum(self.counts)

    def close(self) -> None:
        self.pool.shutdown()
