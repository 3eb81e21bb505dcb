"""The device slice queue (worker outbox) and the deadlock error.

``FrameQueue`` in the reference (``pkg/src/p3sync/queues.py:20-75``) is a host heap of
frames keyed by ``priority_sort_key``. Here the outbox lives in device memory and is
consumed by the persistent comm kernel: per layer an iteration tag, a publish sequence
and a claim cursor; a pop returns the lowest ready layer's next slice (priority mode) or
the earliest-published layer's next slice (FIFO mode). ``DeviceSliceQueue`` drives that
same ``warp_pop`` routine one operation at a time (scripted replay / tests).
"""

from __future__ import annotations

import ctypes
import threading

from . import _lib
from .plan import SliceKey


class DeadlockError(RuntimeError):
    """A blocking wait exceeded its deadline (queues.py:12-13)."""


class DeviceSliceQueue:
    """put_batch == put_layer (all slices of a layer, atomically); poll pops the minimum."""

    def __init__(self, slices_per_layer: list[int], priority_mode: bool = True) -> None:
        self.priority_mode = priority_mode
        self.slices_per_layer = list(slices_per_layer)
        lib = _lib.load()
        arr = (ctypes.c_uint32 * len(self.slices_per_layer))(*self.slices_per_layer)
        h = ctypes.c_void_p()
        sched = _lib.P3_SCHED_PRIORITY if priority_mode else _lib.P3_SCHED_FIFO
        _lib.check(lib.p3_queue_create(arr, len(self.slices_per_layer), sched, ctypes.byref(h)), what="p3_queue_create")
        self._h = h

    def put_layer(self, layer: int, iteration: int = 0) -> None:
        _lib.check(_lib.load().p3_queue_put_layer(self._h, layer, iteration), what="p3_queue_put_layer")

    def poll(self) -> SliceKey | None:
        l, s = ctypes.c_uint32(), ctypes.c_uint32()
        rc = _lib.load().p3_queue_poll(self._h, ctypes.byref(l), ctypes.byref(s))
        if rc == _lib.P3_ETIMEOUT:
            return None
        _lib.check(rc, what="p3_queue_poll")
        return SliceKey(int(l.value), int(s.value))

    def close(self) -> None:
        if self._h:
            _lib.load().p3_queue_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class FrameQueue:
    """FrameQueue (queues.py:20-75) with the device slice queue underneath.

    ``put_batch`` takes the frames of ONE layer — every slice of it, which is how the worker
    enqueues a layer (worker.py:173-182) and what makes the batch atomic on the device: one
    publication word; ``poll`` is the device pop (priority mode: lowest layer, ascending
    slice; FIFO mode: publish order), blocking up to ``timeout`` and raising DeadlockError
    when nothing arrives, None once closed and drained. The device keeps keys; the frames
    (descriptors, worker.py:152-164) stay on the host. A layer must be drained before it is
    queued again (the device holds one batch per layer).
    """

    def __init__(self, priority_mode: bool = True, slices_per_layer: list[int] | None = None) -> None:
        if slices_per_layer is None:
            raise ValueError("slices_per_layer (slices of each layer, from the slice plan) is required")
        self.priority_mode = priority_mode
        self._n = list(slices_per_layer)
        self._q = DeviceSliceQueue(self._n, priority_mode)
        self._frames: dict[tuple[int, int], object] = {}
        self._remaining = [0] * len(self._n)
        self._closed = False
        self._cond = threading.Condition()

    @classmethod
    def for_plan(cls, plan, priority_mode: bool = True) -> "FrameQueue":
        n = [0] * (max((s.key.layer_index for s in plan.slices), default=-1) + 1)
        for s in plan.slices:
            n[s.key.layer_index] += 1
        return cls(priority_mode, n)

    def put(self, frame) -> None:
        self.put_batch([frame])

    def put_batch(self, frames) -> None:
        frames = list(frames)
        if not frames:
            return
        layer = frames[0].layer_index
        if any(f.layer_index != layer for f in frames) or not 0 <= layer < len(self._n):
            raise ValueError("a batch holds the slices of one layer of the plan")
        if sorted(f.slice_index for f in frames) != list(range(self._n[layer])):
            raise ValueError(f"layer {layer}: a batch holds every one of its {self._n[layer]} slices")
        if self.priority_mode and any(f.priority != layer for f in frames):
            raise ValueError("priority mode orders by layer: priority must equal the layer index (plan.py:112)")
        with self._cond:
            if self._closed:
                raise RuntimeError("queue is closed")
            if self._remaining[layer]:
                raise ValueError(f"layer {layer} is still queued")
            for f in frames:
                self._frames[(layer, f.slice_index)] = f
            self._remaining[layer] = len(frames)
            self._q.put_layer(layer, 0)
            self._cond.notify_all()

    def poll(self, timeout: float | None = None):
        with self._cond:
            while True:
                if any(self._remaining):
                    key = self._q.poll()
                    if key is not None:
                        self._remaining[key.layer_index] -= 1
                        return self._frames.pop((key.layer_index, key.slice_index))
                if self._closed:
                    return None
                if not self._cond.wait(timeout):
                    raise DeadlockError(f"queue poll stalled for {timeout}s ({len(self)} queued)")

    def close(self) -> None:
        with self._cond:
            self._closed = True
            self._cond.notify_all()

    def snapshot(self) -> list:
        with self._cond:
            return list(self._frames.values())

    def __len__(self) -> int:
        return sum(self._remaining)
