"""Wire frames: the host codec against the reference's encodings
(tests/golden: frames encoded by p3sync.proto, and its verdicts on malformed buffers),
the properties of the reference's proto tests (tests/test_proto.py: header layout,
truncation, rejection, round trip, arbitrary stream splits), and the device pack /
unpack kernels against the host codec."""

import struct

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1905_03960_b200.proto import (
    DEFAULT_MAX_PAYLOAD,
    HEADER_LEN,
    MAGIC,
    Frame,
    FrameDecoder,
    MsgType,
    ProtocolError,
    encode_frame,
    pack_f32,
    try_decode,
)


def _frame(d):
    return Frame(MsgType(d["msg_type"]), d["priority"], d["iteration"], d["worker_rank"], d["layer_index"],
                 d["slice_index"], d["offset"], bytes.fromhex(d["payload"]))


def test_golden_encodings(golden):
    for d in golden["frames"]["frames"]:
        f = _frame(d)
        wire = encode_frame(f)
        assert wire.hex() == d["wire"]
        back, used = try_decode(wire)
        assert back == f and used == len(wire)


def test_golden_decode_verdicts(golden):
    for case in golden["frames"]["decode_cases"]:
        buf = bytes.fromhex(case["buf"])
        if "error" in case:
            with pytest.raises(ProtocolError) as e:
                try_decode(buf)
            assert case["error"] in str(e.value), case["name"]
        else:
            fr, n = try_decode(buf)
            assert (fr is not None) == case["ok"] and n == case["n"], case["name"]


def test_layout():
    assert HEADER_LEN == 39
    f = Frame(MsgType.BCAST, priority=0xA1A2A3A4, iteration=0x0102030405060708, worker_rank=0xBEEF,
              layer_index=0x11223344, slice_index=0x55667788, offset=0x99AABBCCDDEEFF00,
              payload=pack_f32(np.array([2.5], np.float32)))
    w = encode_frame(f)
    assert w[:4] == MAGIC and w[4] == 1 and len(w) == HEADER_LEN + 4
    assert struct.unpack_from("<IQHIIQI", w, 5) == (0xA1A2A3A4, 0x0102030405060708, 0xBEEF, 0x11223344, 0x55667788,
                                                   0x99AABBCCDDEEFF00, 4)
    assert len(encode_frame(Frame(MsgType.FIN, worker_rank=2))) == HEADER_LEN


def test_truncation_reports_bytes_needed():
    w = encode_frame(Frame(MsgType.PUSH, payload=pack_f32(np.arange(3, dtype=np.float32))))
    for cut in (0, 1, 20, HEADER_LEN - 1):
        assert try_decode(w[:cut]) == (None, HEADER_LEN - cut)
    for cut in (1, 5, 12):
        assert try_decode(w[:-cut]) == (None, cut)


def test_encode_rejects():
    with pytest.raises(ProtocolError):
        encode_frame(Frame(MsgType.NOTIFY, payload=b"\0\0\0\0"))
    with pytest.raises(ProtocolError):
        encode_frame(Frame(MsgType.PUSH, payload=b"\0\0\0"))  # not a float32 array


def test_max_payload_is_the_callers():
    w = encode_frame(Frame(MsgType.PUSH, payload=pack_f32(np.zeros(8, np.float32))))
    with pytest.raises(ProtocolError, match="exceeds"):
        try_decode(w, max_payload=16)
    assert try_decode(w, max_payload=32)[1] == len(w)
    assert DEFAULT_MAX_PAYLOAD == 16 * 1024 * 1024


_u = st.integers
_any_frame = st.one_of(
    st.builds(Frame, msg_type=st.sampled_from([MsgType.PUSH, MsgType.BCAST]), priority=_u(0, 2**32 - 1),
              iteration=_u(0, 2**64 - 1), worker_rank=_u(0, 2**16 - 1), layer_index=_u(0, 2**32 - 1),
              slice_index=_u(0, 2**32 - 1), offset=_u(0, 2**64 - 1),
              payload=st.lists(st.floats(width=32, allow_nan=False), max_size=12).map(
                  lambda v: pack_f32(np.array(v, np.float32)))),
    st.builds(Frame, msg_type=st.sampled_from([MsgType.PULL, MsgType.NOTIFY, MsgType.HELLO, MsgType.FIN]),
              priority=_u(0, 2**32 - 1), iteration=_u(0, 2**64 - 1), worker_rank=_u(0, 2**16 - 1),
              layer_index=_u(0, 2**32 - 1), slice_index=_u(0, 2**32 - 1), offset=_u(0, 2**64 - 1)),
)


@settings(max_examples=200, deadline=None)
@given(_any_frame)
def test_round_trip(f):
    w = encode_frame(f)
    assert try_decode(w) == (f, len(w))


@settings(max_examples=60, deadline=None)
@given(st.lists(_any_frame, max_size=5), st.data())
def test_any_split_of_a_stream(frames, data):
    blob = b"".join(encode_frame(f) for f in frames)
    dec, got, pos = FrameDecoder(), [], 0
    while pos < len(blob):
        step = data.draw(st.integers(1, len(blob) - pos))
        got += dec.feed(blob[pos : pos + step])
        pos += step
    assert got == frames and dec.pending_bytes == 0


# ------------------------------------------------------------------ device pack / unpack


@pytest.mark.gpu
def test_device_pack_matches_host_codec(cuda):
    import torch

    from paper_1905_03960_b200.proto import pack_frames

    rng = np.random.default_rng(7)
    arena = torch.from_numpy(rng.standard_normal(300_000).astype(np.float32)).cuda()
    heads, pays, host = [], [], []
    pos = 0
    for i in range(64):
        mt = MsgType(int(rng.integers(0, 6)))
        n = int(rng.integers(0, 60_000)) if mt in (MsgType.PUSH, MsgType.BCAST) else 0
        if i % 7 == 0 and n:
            n = int(rng.integers(1, 9))  # tiny payloads: only head / tail bytes
        p = arena[pos : pos + n] if n else None
        pos = (pos + n + int(rng.integers(0, 5))) % 200_000
        h = Frame(mt, int(rng.integers(0, 2**32)), int(rng.integers(0, 2**63)), int(rng.integers(0, 2**16)),
                  int(rng.integers(0, 2**32)), i, int(rng.integers(0, 2**63)))
        heads.append(h)
        pays.append(p)
        host.append(encode_frame(Frame(h.msg_type, h.priority, h.iteration, h.worker_rank, h.layer_index,
                                       h.slice_index, h.offset, b"" if p is None else p.cpu().numpy().tobytes())))
    buf, offs = pack_frames(heads, pays)
    assert bytes(buf.cpu().numpy().tobytes()) == b"".join(host)
    assert offs[1] == len(host[0])


@pytest.mark.gpu
def test_device_unpack_round_trip_and_errors(cuda):
    import torch

    from paper_1905_03960_b200.proto import pack_frames, unpack_frames

    rng = np.random.default_rng(11)
    arena = torch.from_numpy(rng.standard_normal(200_000).astype(np.float32)).cuda()
    sizes = [50_000, 3, 0, 17, 49_999, 1, 12_345]
    heads, pays, o = [], [], 0
    for i, n in enumerate(sizes):
        heads.append(Frame(MsgType.BCAST if n else MsgType.PULL, priority=i, iteration=9, worker_rank=1,
                           layer_index=i, slice_index=2 * i, offset=o))
        pays.append(arena[o : o + n] if n else None)
        o += n + 1
    buf, offs = pack_frames(heads, pays)
    dests = [torch.full((n,), float("nan"), device="cuda") if n else None for n in sizes]
    got = unpack_frames(buf, offs, dests)
    for h, g, p, d in zip(heads, got, pays, dests):
        assert (g.msg_type, g.priority, g.layer_index, g.slice_index, g.offset) == (
            h.msg_type, h.priority, h.layer_index, h.slice_index, h.offset)
        if p is not None:
            assert torch.equal(d, p)
    bad = buf.clone()
    bad[offs[4] + 1] = ord("X")  # magic of frame 4
    with pytest.raises(ProtocolError, match="frame 4: bad magic"):
        unpack_frames(bad, offs, dests)
    bad = buf.clone()
    bad[offs[2] + 35] = 4  # PULL with a payload length
    with pytest.raises(ProtocolError, match="frame 2: nonzero payload"):
        unpack_frames(bad, offs, None)
