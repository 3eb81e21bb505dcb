"""The unit of synchronisation and its wire form for traffic that leaves the box.

``Frame`` / ``MsgType`` / ``ProtocolError`` keep the reference's names and fields
(``pkg/src/p3sync/proto.py:26-54``). Inside one NVSwitch domain nothing is serialised: a
PUSH is a set of NVLink stores into the owner's receive slot and a BCAST a set of stores
into every replica; the header fields survive as the device trace record
(``p3_trace_rec_t``).

Across nodes frames use the reference's 39-byte little-endian header
(``proto.py:18-21``): ``encode_frame`` / ``try_decode`` / ``FrameDecoder`` are the host
codec (libp3 ``p3_frame_encode`` / ``p3_frame_decode``), and ``pack_frames`` /
``unpack_frames`` build and parse whole batches of frames in device memory
(``p3_frames_pack`` / ``p3_frames_unpack``), so a NIC can send slices straight from the
gradient and parameter arenas.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib

MAGIC = b"P3W1"
HEADER_LEN = _lib.P3_FRAME_HEADER_BYTES  # 39 = 4+1+4+8+2+4+4+8+4
DEFAULT_MAX_PAYLOAD = 16 * 1024 * 1024


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


def _frame_t(frame: Frame, payload_len: int | None = None) -> _lib.FrameT:
    f = _lib.FrameT()
    f.msg_type = int(frame.msg_type)
    f.priority = frame.priority
    f.iteration = frame.iteration
    f.worker_rank = frame.worker_rank
    f.layer = frame.layer_index
    f.slice = frame.slice_index
    f.offset = frame.offset
    f.payload_len = len(frame.payload) if payload_len is None else payload_len
    return f


def _frame_of(f: _lib.FrameT, payload: bytes) -> Frame:
    return Frame(MsgType(f.msg_type), f.priority, f.iteration, f.worker_rank, f.layer, f.slice, f.offset, payload)


def encode_frame(frame: Frame) -> bytes:
    """encode_frame (proto.py:61-79) through ``p3_frame_encode``."""
    lib = _lib.load()
    f = _frame_t(frame)
    n = ctypes.c_uint64()
    _lib.check(lib.p3_frame_encode(ctypes.byref(f), None, None, 0, ctypes.byref(n)), what="encode_frame")
    out = ctypes.create_string_buffer(n.value)
    pay = ctypes.create_string_buffer(frame.payload, len(frame.payload)) if frame.payload else None
    _lib.check(lib.p3_frame_encode(ctypes.byref(f), pay, out, n.value, ctypes.byref(n)), what="encode_frame")
    return out.raw


def try_decode(buf, max_payload: int = DEFAULT_MAX_PAYLOAD) -> tuple[Frame | None, int]:
    """try_decode (proto.py:82-120): (frame, bytes consumed) or (None, bytes still needed);
    ProtocolError on bad magic, unknown msg_type, oversized or misplaced payload."""
    data = bytes(buf)
    lib = _lib.load()
    f = _lib.FrameT()
    n = ctypes.c_uint64()
    rc = lib.p3_frame_decode(data, len(data), max_payload, ctypes.byref(f), ctypes.byref(n))
    if rc == _lib.P3_EMORE:
        return None, n.value
    _lib.check(rc, what="try_decode")
    return _frame_of(f, data[HEADER_LEN : HEADER_LEN + f.payload_len]), n.value


@dataclass
class FrameDecoder:
    """Incremental decoder (proto.py:123-141): feed arbitrary byte chunks, get whole frames."""

    max_payload: int = DEFAULT_MAX_PAYLOAD
    _buf: bytearray = field(default_factory=bytearray)

    def feed(self, data: bytes) -> list[Frame]:
        self._buf.extend(data)
        frames = []
        while True:
            frame, n = try_decode(self._buf, self.max_payload)
            if frame is None:
                break
            del self._buf[:n]
            frames.append(frame)
        return frames

    @property
    def pending_bytes(self) -> int:
        return len(self._buf)


# ---------------------------------------------------------------- device batches


def frame_sizes(frames: list[Frame], payload_lens: list[int] | None = None) -> list[int]:
    return [HEADER_LEN + (len(f.payload) if payload_lens is None else payload_lens[i]) for i, f in enumerate(frames)]


def pack_frames(headers: list[Frame], payloads: list, stream=None):
    """Build len(headers) wire frames back to back in one uint8 device tensor.

    ``payloads[i]`` is a float32 CUDA tensor (a slice view of a gradient or parameter arena)
    or None for control frames; the header's payload field is ignored in favour of it. The
    headers are validated on the host with the same rules as ``encode_frame``. Returns
    (buffer, byte offsets)."""
    import torch

    lib = _lib.load()
    n = len(headers)
    rows = (_lib.FrameT * max(n, 1))()
    lens = []
    for i, (h, p) in enumerate(zip(headers, payloads)):
        plen = 0 if p is None else int(p.numel()) * 4
        if p is not None and (p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous()):
            raise ValueError("payloads must be contiguous float32 CUDA tensors")
        rows[i] = _frame_t(h, plen)
        size = ctypes.c_uint64()
        _lib.check(lib.p3_frame_encode(ctypes.byref(rows[i]), None, None, 0, ctypes.byref(size)), what="pack_frames")
        lens.append(plen)
    offs, o = [], 0
    for plen in lens:
        offs.append(o)
        o += HEADER_LEN + plen
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(max(o, 1), dtype=torch.uint8, device=dev)
    meta = torch.frombuffer(bytearray(bytes(rows)), dtype=torch.uint8).to(dev)
    srcs = torch.tensor([0 if p is None else p.data_ptr() for p in payloads] or [0], dtype=torch.int64, device=dev)
    offt = torch.tensor(offs or [0], dtype=torch.int64, device=dev)
    _lib.check(lib.p3_frames_pack(meta.data_ptr(), srcs.data_ptr(), offt.data_ptr(), n, out.data_ptr(),
                                  _lib.stream_handle(stream)), what="p3_frames_pack")
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    return out[:o], offs


def unpack_frames(buf, offsets: list[int], dests: list | None = None, max_payload: int = DEFAULT_MAX_PAYLOAD,
                  stream=None) -> list[Frame]:
    """Parse the frames at ``offsets`` of a uint8 device tensor; copy each payload into
    ``dests[i]`` (a float32 CUDA tensor, or None). Raises ProtocolError naming the first bad
    frame. Returned frames carry an empty payload (it lives in ``dests``)."""
    import torch

    lib = _lib.load()
    n = len(offsets)
    dev = buf.device
    offt = torch.tensor(offsets or [0], dtype=torch.int64, device=dev)
    dsts = torch.tensor([0 if d is None else d.data_ptr() for d in (dests or [None] * n)] or [0], dtype=torch.int64,
                        device=dev)
    rows = torch.zeros(max(n, 1) * ctypes.sizeof(_lib.FrameT), dtype=torch.uint8, device=dev)
    err = torch.zeros(4, dtype=torch.int32, device=dev)
    _lib.check(lib.p3_frames_unpack(buf.data_ptr(), offt.data_ptr(), n, max_payload, dsts.data_ptr(), rows.data_ptr(),
                                    err.data_ptr(), _lib.stream_handle(stream)), what="p3_frames_unpack")
    e = err.cpu().tolist()
    if e[0]:
        why = {1: "bad magic", 2: "unknown msg_type", 3: "payload_len exceeds max", 4: "nonzero payload on a control frame"}
        raise ProtocolError(f"frame {e[1]}: {why.get(e[2], 'invalid header')}")
    host = bytes(rows.cpu().numpy().tobytes())
    out = []
    for i in range(n):
        f = _lib.FrameT.from_buffer_copy(host, i * ctypes.sizeof(_lib.FrameT))
        out.append(_frame_of(f, b""))
    return out
