"""The unit of synchronisation, without a byte codec.

``Frame`` / ``MsgType`` / ``ProtocolError`` keep the reference's names and fields
(``pkg/src/p3sync/proto.py:26-54``). Inside one NVSwitch domain nothing is serialised:
a PUSH is a set of NVLink stores into the owner's receive slot and a BCAST a set of
stores into every replica, so the 39-byte header codec (proto.py:61-141) is out of scope.
The header fields survive as the device trace record (``p3_trace_rec_t``).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class MsgType(enum.IntEnum):
    PUSH = 0
    BCAST = 1
    PULL = 2
    NOTIFY = 3
    HELLO = 4
    FIN = 5


class ProtocolError(Exception):
    """Rule-violating traffic (proto.py:35-36)."""


@dataclass(frozen=True)
class Frame:
    msg_type: MsgType
    priority: int = 0
    iteration: int = 0
    worker_rank: int = 0
    layer_index: int = 0
    slice_index: int = 0
    offset: int = 0
    payload: bytes = b""

    def payload_f32(self) -> np.ndarray:
        return np.frombuffer(self.payload, dtype="<f4")


def pack_f32(values) -> bytes:
    return np.ascontiguousarray(values, dtype="<f4").tobytes()
