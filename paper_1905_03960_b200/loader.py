"""Host -> device input staging for training with P3DataParallel.

``DevicePrefetcher`` copies batch i+1 from pinned host memory on a dedicated copy stream
while batch i is being computed, the way a production data loader feeds a B200: the
host-to-device traffic of every step overlaps the previous step's compute instead of
stalling the compute stream. The device side is a fixed ring of ``depth`` preallocated
batch buffers (no allocation per step — a caching-allocator miss in the step loop
synchronises the device); a buffer is refilled only after the compute stream has finished
the step that read it (event-ordered).
"""

from __future__ import annotations

import torch


class DevicePrefetcher:
    def __init__(self, host_batches, device: str = "cuda", depth: int = 2) -> None:
        if depth < 2:
            raise ValueError("depth must be >= 2 (one buffer in compute, one being filled)")
        self._it = iter(host_batches)
        self.device = device
        self.depth = depth
        self.copy_stream = torch.cuda.Stream()
        self._bufs = None
        self._free = [None] * depth  # compute-stream event after the last read of each buffer
        self._slot = 0
        self._next = None
        self._cur_slot = None
        self.h2d_bytes = 0

    def _stage(self) -> None:
        try:
            batch = next(self._it)
        except StopIteration:
            self._next = None
            return
        if self._bufs is None:
            self._bufs = [tuple(torch.empty_like(t, device=self.device) for t in batch) for _ in range(self.depth)]
        slot = self._slot
        self._slot = (slot + 1) % self.depth
        bufs = self._bufs[slot]
        with torch.cuda.stream(self.copy_stream):
            if self._free[slot] is not None:
                self.copy_stream.wait_event(self._free[slot])
            for d, h in zip(bufs, batch):
                d.copy_(h, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self.copy_stream)
        self._next = (bufs, ready, slot)
        self.h2d_bytes += sum(t.numel() * t.element_size() for t in batch)

    def __iter__(self):
        return self

    def __next__(self):
        if self._cur_slot is not None:  # the previous step's reads are all enqueued by now
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._free[self._cur_slot] = ev
        if self._next is None:
            self._stage()
            if self._next is None:
                raise StopIteration
        cur, ready, slot = self._next
        torch.cuda.current_stream().wait_event(ready)
        self._cur_slot = slot
        self._stage()  # the next copy overlaps this step's compute
        return cur
