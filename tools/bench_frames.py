"""Device wire-frame throughput: pack every P3 slice of a model's gradient into PUSH frames
(p3_frames_pack) and unpack them into a parameter-shaped arena (p3_frames_unpack);
HBM GB/s = (payload read + frame write) / kernel time, CUDA events, L2 flushed.
python tools/bench_frames.py resnet50"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1905_03960_b200.model import LayerSpec, ModelProfile
from paper_1905_03960_b200.plan import make_p3_plan
from paper_1905_03960_b200.proto import HEADER_LEN, Frame, MsgType, pack_frames, unpack_frames
from paper_1905_03960_b200.torch_models import real_counts


def main():
    m = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    counts = real_counts(m)
    plan = make_p3_plan(ModelProfile(m, 0, tuple(LayerSpec(i, "l", c, 0, 0) for i, c in enumerate(counts))), 1)
    P = sum(counts)
    grad = torch.randn(P, device="cuda")
    base = [0]
    for c in counts:
        base.append(base[-1] + c)
    heads = [Frame(MsgType.PUSH, s.priority, 3, 0, s.key.layer_index, s.key.slice_index, s.offset) for s in plan.slices]
    pays = [grad[base[s.key.layer_index] + s.offset : base[s.key.layer_index] + s.offset + s.length] for s in plan.slices]
    buf, offs = pack_frames(heads, pays)
    out = torch.empty_like(grad)
    dests = [out[base[s.key.layer_index] + s.offset : base[s.key.layer_index] + s.offset + s.length] for s in plan.slices]
    unpack_frames(buf, offs, dests)
    assert torch.equal(out, grad)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    from paper_1905_03960_b200 import _lib
    import ctypes

    lib = _lib.load()
    n = len(heads)
    rows = (_lib.FrameT * n)()
    for i, (h, p) in enumerate(zip(heads, pays)):
        rows[i].msg_type, rows[i].priority, rows[i].iteration = int(h.msg_type), h.priority, h.iteration
        rows[i].layer, rows[i].slice, rows[i].offset, rows[i].payload_len = h.layer_index, h.slice_index, h.offset, 4 * p.numel()
    meta = torch.frombuffer(bytearray(bytes(rows)), dtype=torch.uint8).cuda()
    srcs = torch.tensor([p.data_ptr() for p in pays], dtype=torch.int64, device="cuda")
    dsts = torch.tensor([d.data_ptr() for d in dests], dtype=torch.int64, device="cuda")
    offt = torch.tensor(offs, dtype=torch.int64, device="cuda")
    err = torch.zeros(4, dtype=torch.int32, device="cuda")
    fo = torch.zeros(n * ctypes.sizeof(_lib.FrameT), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    for name in ("pack", "unpack"):
        ts = []
        for k in range(8):
            flush.fill_(k)
            torch.cuda._sleep(100_000)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            if name == "pack":
                lib.p3_frames_pack(meta.data_ptr(), srcs.data_ptr(), offt.data_ptr(), n, buf.data_ptr(), st.cuda_stream)
            else:
                lib.p3_frames_unpack(buf.data_ptr(), offt.data_ptr(), n, 1 << 24, dsts.data_ptr(), fo.data_ptr(),
                                     err.data_ptr(), st.cuda_stream)
            e.record()
            torch.cuda.synchronize()
            if k >= 2:
                ts.append(s.elapsed_time(e))
        ms = sum(ts) / len(ts)
        bytes_moved = 4 * P + (4 * P + HEADER_LEN * n)  # read payloads + write frames (or the reverse)
        res[name] = {"ms": round(ms, 4), "GBps": round(bytes_moved / (ms * 1e-3) / 1e9, 1)}
    assert torch.equal(out, grad) and int(err[0]) == 0
    print(json.dumps({"model": m, "frames": n, "payload_MB": round(4 * P / 1e6, 1), **res}))


main()
