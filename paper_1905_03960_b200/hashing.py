"""Deterministic hashing: splitmix64, synthetic gradients (GradGen), FNV-1a digests.

Host mirror of ``p3sync.hashing`` (reference ``pkg/src/p3sync/hashing.py``). The
gradient generator runs on the GPU (K1 ``k_gradgen`` in csrc/p3_kernels.cu) and is
bit-exact with the reference formula (hashing.py:45-63); splitmix64 and FNV-1a run in
libp3's host code (csrc/p3_host.cpp).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

MASK64 = 0xFFFFFFFFFFFFFFFF
FNV_OFFSET = 0xCBF29CE484222325


def splitmix64_stream(seed: int, index: int) -> int:
    """index-th output of the splitmix64 sequence started at ``seed`` (hashing.py:32-35)."""
    return int(_lib.load().p3_splitmix64_stream(seed & MASK64, index & MASK64))


def splitmix64_mix(x: int) -> int:
    """splitmix64 output mixer (hashing.py:24-29): stream(x - gamma, 0) == mix(x)."""
    return splitmix64_stream((x - 0x9E3779B97F4A7C15) & MASK64, 0)


def gradient_block_device(seed: int, iteration: int, layer_index: int, start: int, count: int, out=None, stream=None):
    """K1 on the current CUDA device: returns (or fills) a float32 CUDA tensor."""
    import torch

    if out is None:
        out = torch.empty(count, dtype=torch.float32, device="cuda")
    if count:
        _lib.check(
            _lib.load().p3_gradient_block(
                seed & MASK64, iteration & MASK64, layer_index & MASK64, start, count,
                out.data_ptr(), _lib.stream_handle(stream),
            ),
            what="p3_gradient_block",
        )
    return out


def gradient_block(seed: int, iteration: int, layer_index: int, start: int, count: int) -> np.ndarray:
    """gradient_block (hashing.py:55-63), computed by the device kernel."""
    return gradient_block_device(seed, iteration, layer_index, start, count).cpu().numpy()


def gradient_value(seed: int, iteration: int, layer_index: int, element_index: int) -> np.float32:
    return np.float32(gradient_block(seed, iteration, layer_index, element_index, 1)[0])


@dataclass(frozen=True)
class GradGen:
    """Stand-in for backprop output (hashing.py:66-76)."""

    seed: int

    def value(self, iteration: int, layer_index: int, element_index: int) -> np.float32:
        return gradient_value(self.seed, iteration, layer_index, element_index)

    def block(self, iteration: int, layer_index: int, start: int, count: int) -> np.ndarray:
        return gradient_block(self.seed, iteration, layer_index, start, count)


def fnv1a64(data, h: int = FNV_OFFSET) -> int:
    """64-bit FNV-1a with chaining (hashing.py:79-83), in libp3 host code."""
    buf = bytes(data) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data).tobytes()
    cbuf = ctypes.create_string_buffer(buf, len(buf)) if buf else None
    return int(_lib.load().p3_fnv1a64(cbuf, len(buf), h & MASK64))
