"""The reference P3 sync path on host cores — TEST / BASELINE INFRASTRUCTURE ONLY.

One synchronous P3 iteration exactly as the reference runtime computes it, restated with
numpy and run on a thread pool (numpy releases the GIL inside its kernels):

  worker side   (worker.py:173-190, 166-171): layers are enqueued in backward order
                (L-1 .. 0) into a priority FrameQueue; the sender pops the minimum
                (priority, layer, slice) and materialises the slice's GradGen gradient;
  server side   (server.py:55-68): per slice, the N pushes are summed in ascending rank
                order, divided by N and applied with p - lr*g (fp32);
  apply side    (worker.py:241-269): the updated slice is written into every replica.

Used by bench.py as ``cpu_baseline`` (kind "port") and as the ``--impl reference`` arm,
because the reference itself is Python that cannot travel to the GPU box. Never imported
by the product package.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from p3_oracle import HeapQueue, grad_block, p3_rows, rank_seed


class CpuP3:
    def __init__(self, counts: list[int], world: int, seed: int = 0, lr: float = 0.1, max_slice: int = 50_000,
                 threads: int | None = None) -> None:
        self.counts = list(counts)
        self.world = world
        self.seed = seed
        self.lr = np.float32(lr)
        self.rows = p3_rows(self.counts, world, max_slice)
        self.by_layer: dict[int, list] = {}
        for r in self.rows:
            self.by_layer.setdefault(r.layer, []).append(r)
        self.params = [np.zeros(c, dtype=np.float32) for c in self.counts]  # worker.py:72
        self.replicas = world
        self.threads = threads or len(os.sched_getaffinity(0))
        self.pool = ThreadPoolExecutor(self.threads)

    def _slice_job(self, k: int, row) -> None:
        acc = np.zeros(row.length, dtype=np.float32)
        for r in range(self.world):  # pushes of every rank, ascending rank order
            acc += grad_block(rank_seed(self.seed, r, False), k, row.layer, row.offset, row.length)
        g = acc / np.float32(self.world)
        p = self.params[row.layer]
        upd = p[row.offset : row.offset + row.length] - self.lr * g
        for _ in range(self.replicas):  # BCAST applied into every replica
            p[row.offset : row.offset + row.length] = upd

    def iteration(self, k: int, sample_slices: int | None = None) -> int:
        """Run one iteration (or its first ``sample_slices`` pops); returns slices done."""
        q = HeapQueue(priority_mode=True)
        for layer in reversed(range(len(self.counts))):
            q.put_layer(layer, len(self.by_layer[layer]))
        order = []
        while len(q) and (sample_slices is None or len(order) < sample_slices):
            l, s = q.poll()
            order.append(self.by_layer[l][s])
        list(self.pool.map(lambda row: self._slice_job(k, row), order))
        return len(order)

    def time_iteration(self, k: int, sample_slices: int | None = None) -> tuple[float, float]:
        """(seconds, fraction of the iteration's elements covered by the sample)."""
        t0 = time.perf_counter()
        n = self.iteration(k, sample_slices)
        dt = time.perf_counter() - t0
        q = HeapQueue(True)
        for layer in reversed(range(len(self.counts))):
            q.put_layer(layer, len(self.by_layer[layer]))
        elems = 0
        for _ in range(n):
            l, s = q.poll()
            elems += self.by_layer[l][s].length
        return dt, elems / sum(self.counts)

    def close(self) -> None:
        self.pool.shutdown()
