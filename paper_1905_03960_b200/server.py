"""Parameter-server shard state: aggregate pushed gradients and apply SGD.

Host mirror of ``p3sync.server.ShardState`` / ``bcast_frames`` (reference
``pkg/src/p3sync/server.py:22-88``). ``on_push`` keeps the reference's protocol checks;
``aggregate_and_update`` runs the K4 device kernel (``p3_shard_update``), which sums in
ascending rank order from +0.0, divides by N and applies ``p - lr*g`` with separately
rounded multiply and subtract — bit-identical to the reference's numpy fp32 arithmetic.
Inside the live runtime the same routine runs per slice in the comm kernel's server role.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .plan import Slice, SliceKey
from .proto import Frame, MsgType, ProtocolError, pack_f32


def shard_update_device(params, grads: list, lr: float, momentum: float = 0.0, momentum_buf=None, stream=None) -> None:
    """In-place K4 on CUDA tensors: params -= lr * mean(grads) (rank order)."""
    n = params.numel()
    ptrs = (ctypes.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
    _lib.check(
        _lib.load().p3_shard_update(
            params.data_ptr(), ptrs, len(grads), n, ctypes.c_float(lr), ctypes.c_float(momentum),
            momentum_buf.data_ptr() if momentum_buf is not None else None, _lib.stream_handle(stream),
        ),
        what="p3_shard_update",
    )


@dataclass
class ShardState:
    """Authoritative state for one slice key (server.py:22-68)."""

    key: SliceKey
    params: np.ndarray
    num_workers: int
    lr: float
    iteration: int = 0
    pending: dict = field(default_factory=dict)

    def on_push(self, worker_rank: int, iteration: int, grad) -> bool:
        if iteration != self.iteration:
            raise ProtocolError(f"key {self.key}: push for iteration {iteration}, shard at {self.iteration}")
        if not 0 <= worker_rank < self.num_workers:
            raise ProtocolError(f"key {self.key}: push from unknown rank {worker_rank}")
        if worker_rank in self.pending:
            raise ProtocolError(f"key {self.key}: duplicate push from rank {worker_rank} at iteration {iteration}")
        if len(grad) != len(self.params):
            raise ProtocolError(f"key {self.key}: gradient length {len(grad)} != {len(self.params)}")
        self.pending[worker_rank] = grad
        return len(self.pending) == self.num_workers

    def aggregate_and_update(self):
        if len(self.pending) != self.num_workers:
            raise ProtocolError(f"key {self.key}: aggregate with {len(self.pending)}/{self.num_workers} pushes")
        import torch

        on_host = isinstance(self.params, np.ndarray)
        p_dev = torch.from_numpy(np.ascontiguousarray(self.params, dtype=np.float32)).cuda() if on_host else self.params
        grads = []
        for rank in sorted(self.pending):
            g = self.pending[rank]
            grads.append(torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32)).cuda() if isinstance(g, np.ndarray) else g)
        if len(p_dev):
            shard_update_device(p_dev, grads, self.lr)
        if on_host:
            self.params[...] = p_dev.cpu().numpy()
        self.pending.clear()
        self.iteration += 1
        return self.params


def bcast_frames(sl: Slice, iteration: int, params, worker_ranks: list[int]) -> list[Frame]:
    """One BCAST descriptor per worker, priority copied from the slice (server.py:71-88)."""
    payload = pack_f32(params.cpu().numpy() if hasattr(params, "cpu") else params)
    return [
        Frame(MsgType.BCAST, sl.priority, iteration, rank, sl.key.layer_index, sl.key.slice_index, sl.offset, payload)
        for rank in worker_ranks
    ]
