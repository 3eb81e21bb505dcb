import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200.ddp import P3DataParallel, LayerwiseDataParallel
from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import build_model, synthetic_batch, loss_fn
name = "resnet50"; B = 256
x, y = synthetic_batch(name, B)

def timeit(ddp, steps=10, warm=5):
    for _ in range(warm):
        loss_fn(name, ddp, x, y).backward()
    ddp.synchronize(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(steps):
        loss_fn(name, ddp, x, y).backward()
    ddp.synchronize(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / steps

def model():
    torch.manual_seed(0)
    return build_model(name).cuda().to(memory_format=torch.channels_last)

class Plain:
    def __init__(self, m): self.m = m
    def __call__(self, *a): return self.m(*a)
    def synchronize(self):
        with torch.no_grad():
            for p in self.m.parameters():
                if p.grad is not None: p.sub_(p.grad.mul(0.01)); p.grad = None

variant = sys.argv[1]
if variant == "plain":
    print(variant, timeit(Plain(model())))
elif variant == "layerwise":
    print(variant, timeit(LayerwiseDataParallel(model(), lr=0.01)))
else:
    kw = {}
    if variant.startswith("p3ctas"):
        kw["comm_ctas"] = int(variant[6:])
    d = P3DataParallel(model(), lr=0.01, **kw)
    if variant == "p3_nogate":
        d._gate = lambda l: None
    if variant == "p3_nodrain":
        orig = SyncContext.layer_ready
        d.ctx.layer_ready = lambda li, l, k, grad=None, stream=None: orig(d.ctx, li, l, k, grad, stream)
        # publish before opening: no drain launch (iteration opened lazily at end)
        d.ctx.iteration_begin_orig = d.ctx.iteration_begin
        opened = {}
        def ib(k, stream=None): opened['k'] = (k, stream)
        def ie(k):
            d.ctx.iteration_begin_orig(*opened['k']); SyncContext.iteration_end(d.ctx, k)
        d.ctx.iteration_begin = ib; d.ctx.iteration_end = ie
    print(variant, timeit(d))
