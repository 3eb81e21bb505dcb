"""Host -> device input staging for training with P3DataParallel.

``DevicePrefetcher`` copies batch i+1 from pinned host memory on a dedicated copy stream
while batch i is being computed (double-buffered device tensors, event-ordered), the way a
production data loader feeds a B200: the host-to-device traffic of every step overlaps the
previous step's compute instead of stalling the compute stream.
"""

from __future__ import annotations

import torch


class DevicePrefetcher:
    def __init__(self, host_batches, device: str = "cuda") -> None:
        self._it = iter(host_batches)
        self.device = device
        self.copy_stream = torch.cuda.Stream()
        self._next = None
        self._ready = None
        self.h2d_bytes = 0

    def _stage(self) -> None:
        try:
            batch = next(self._it)
        except StopIteration:
            self._next = None
            return
        with torch.cuda.stream(self.copy_stream):
            self._next = tuple(t.to(self.device, non_blocking=True) for t in batch)
            self._ready = torch.cuda.Event()
            self._ready.record(self.copy_stream)
        self.h2d_bytes += sum(t.numel() * t.element_size() for t in batch)

    def __iter__(self):
        return self

    def __next__(self):
        if self._next is None:
            self._stage()
            if self._next is None:
                raise StopIteration
        cur, ev = self._next, self._ready
        torch.cuda.current_stream().wait_event(ev)
        for t in cur:
            t.record_stream(torch.cuda.current_stream())
        self._stage()  # the next copy overlaps this step's compute
        return cur
