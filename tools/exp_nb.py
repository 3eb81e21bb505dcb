import sys, ctypes
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200.runtime import SyncContext
ctx = SyncContext([1000, 2000], 1, [0], emulate_grads=True)
ctx.layer_ready(0, 0, 0, None)
torch.cuda.synchronize()
print("layer_ready ok", ctx.debug_snapshot(0)["ready"])
