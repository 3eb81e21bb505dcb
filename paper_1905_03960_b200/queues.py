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
