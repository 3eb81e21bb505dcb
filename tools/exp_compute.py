"""ResNet-50 bs256 bf16-autocast forward+backward time under memory-format / cuDNN settings
(the model compute both training arms share; no sync). python tools/exp_compute.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_03960_b200.torch_models import build_model, loss_fn


def run(fmt, bench, steps=10):
    torch.backends.cudnn.benchmark = bench
    torch.manual_seed(0)
    m = build_model("resnet50").cuda()
    x = torch.randn(256, 3, 224, 224, device="cuda").to(torch.bfloat16)
    if fmt == "cl":
        m = m.to(memory_format=torch.channels_last)
        x = x.contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (256,), device="cuda")
    for _ in range(5):
        loss_fn("resnet50", m, x, y).backward()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(steps):
        loss_fn("resnet50", m, x, y).backward()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for fmt in ("cl", "nchw"):
    for bench in (False, True):
        print("COMPUTE", json.dumps({"format": fmt, "cudnn_benchmark": bench, "ms": round(run(fmt, bench), 2)}), flush=True)
