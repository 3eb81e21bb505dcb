import faulthandler, os, sys, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200.ddp import P3DataParallel
from paper_1905_03960_b200.torch_models import build_model, synthetic_batch, loss_fn
name = sys.argv[1]; batch = int(sys.argv[2])
torch.manual_seed(0)
m = build_model(name).cuda()
if name != "seq2seq": m = m.to(memory_format=torch.channels_last)
ddp = P3DataParallel(m, lr=0.01, comm_ctas=16, timeout_s=30)
x, y = synthetic_batch(name, batch)
for it in range(6):
    t = time.time()
    loss = loss_fn(name, ddp, x, y); print("fwd", it, flush=True)
    loss.backward(); print("bwd", it, flush=True)
    print(it, loss.item(), time.time() - t, flush=True)
ddp.synchronize()
print("snap", {k: (v[:5] if isinstance(v, list) else v) for k, v in ddp.ctx.debug_snapshot(0).items()})
print("done", flush=True)
