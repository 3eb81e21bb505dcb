"""Slice queues: the device slice queue of the comm kernel, and FrameQueue for host frames.

``FrameQueue`` in the reference (``pkg/src/p3sync/queues.py:20-75``) is a host heap of
frames keyed by ``priority_sort_key``. On the GPU path the outbox lives in device memory
and is consumed by the comm kernel: per layer an iteration tag, a publish sequence and a
claim cursor; a pop returns the lowest ready layer's next slice (priority mode) or the
earliest-published layer's next slice (FIFO mode). ``DeviceSliceQueue`` drives that same
``warp_pop`` routine one operation at a time (scripted replay / tests).

``FrameQueue`` keeps the reference's API and semantics for frames that stay on the host
(the wire path beyond one NVSwitch domain, host tooling): blocking ``poll`` with deadlock
timeout, atomic ``put_batch``, close-then-drain, ``snapshot``. Its ordering lives in
libp3's native heap (``p3_fq_*``); the GPU path never goes through it.
"""

from __future__ import annotations

import ctypes
import threading

from . import _lib
from .plan import SliceKey, priority_sort_key


class DeadlockError(RuntimeError):
    """A blocking wait exceeded its deadline (queues.py:12-13)."""


def frame_order_key(frame) -> tuple[int, int, int]:
    """The total order of queued frames (queues.py:16-17): (priority, layer, slice)."""
    return priority_sort_key(frame.priority, SliceKey(frame.layer_index, frame.slice_index))


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
    """Blocking producer/consumer queue of host frames (queues.py:20-75): in priority mode a
    poll returns the minimum of ``frame_order_key`` among the queued frames (arrival breaks
    ties), in FIFO mode the earliest arrival; a batch put is atomic; after ``close`` polls
    drain what is left, then return None."""

    def __init__(self, priority_mode: bool = True) -> None:
        self.priority_mode = priority_mode
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.p3_fq_create(1 if priority_mode else 0, ctypes.byref(h)), what="p3_fq_create")
        self._h = h
        self._frames: dict[int, object] = {}
        self._next = 0
        self._closed = False
        self._cond = threading.Condition()

    def put(self, frame) -> None:
        self.put_batch([frame])

    def put_batch(self, frames) -> None:
        frames = list(frames)
        n = len(frames)
        keys = (ctypes.c_uint64 * (3 * n))()
        handles = (ctypes.c_uint64 * n)()
        if self.priority_mode:
            for i, f in enumerate(frames):
                keys[3 * i : 3 * i + 3] = frame_order_key(f)
        with self._cond:
            if self._closed:
                raise RuntimeError("queue is closed")
            for i, f in enumerate(frames):
                handles[i] = self._next + i
                self._frames[self._next + i] = f
            self._next += n
            _lib.check(self._lib.p3_fq_put_batch(self._h, keys, handles, n), what="p3_fq_put_batch")
            self._cond.notify_all()

    def poll(self, timeout: float | None = None):
        """Next frame; blocks while empty; None once closed and drained; DeadlockError when
        nothing arrives within ``timeout`` seconds."""
        out = ctypes.c_uint64()
        with self._cond:
            while not self._frames and not self._closed:
                if not self._cond.wait(timeout):
                    raise DeadlockError(f"queue poll stalled for {timeout}s ({len(self._frames)} queued)")
            if not self._frames:
                return None
            _lib.check(self._lib.p3_fq_poll(self._h, ctypes.byref(out)), what="p3_fq_poll")
            return self._frames.pop(int(out.value))

    def close(self) -> None:
        with self._cond:
            self._closed = True
            self._cond.notify_all()

    def snapshot(self) -> list:
        """Queued frames in dequeue order."""
        with self._cond:
            n = ctypes.c_uint64()
            _lib.check(self._lib.p3_fq_snapshot(self._h, None, 0, ctypes.byref(n)), what="p3_fq_snapshot")
            buf = (ctypes.c_uint64 * max(1, n.value))()
            _lib.check(self._lib.p3_fq_snapshot(self._h, buf, n.value, ctypes.byref(n)), what="p3_fq_snapshot")
            return [self._frames[int(buf[i])] for i in range(n.value)]

    def __len__(self) -> int:
        with self._cond:
            return len(self._frames)

    def __del__(self):  # pragma: no cover - best effort
        try:
            if getattr(self, "_h", None):
                self._lib.p3_fq_destroy(self._h)
                self._h = None
        except Exception:
            pass
