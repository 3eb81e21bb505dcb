import sys, time, os
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200 import _lib
from paper_1905_03960_b200.model import builtin_profile
from paper_1905_03960_b200.runtime import SyncContext
lib = _lib.load()
prof = builtin_profile("resnet50-like")
scen = sys.argv[1]

def sleep_us(us, s):
    if scen.endswith("torchsleep"):
        with torch.cuda.stream(s):
            torch.cuda._sleep(int(us * 1900))
    elif not scen.startswith("nosleep"):
        lib.p3_emulate_compute(us, _lib.stream_handle(s))

ctx = SyncContext(prof.param_counts(), 1, [0], timeout_s=4.0, emulate_grads=True)
comm = torch.cuda.Stream()
rs = torch.cuda.Stream()
t0 = time.time()
# k_sleep alone
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(rs); lib.p3_emulate_compute(1000, _lib.stream_handle(rs)); e1.record(rs); rs.synchronize()
print(scen, "k_sleep(1000us) took", e0.elapsed_time(e1), "ms", flush=True)
def rank_work():
    for l in prof.layers:
        sleep_us(l.fwd_time, rs)
    for l in reversed(prof.layers):
        sleep_us(l.bwd_time, rs)
        ctx.gradgen_layer(0, prof.seed, 0, l.index, rs)
        ctx.layer_ready(0, l.index, 0, None, rs)
if "late" in scen:
    rank_work(); ctx.iteration_begin(0, comm)
else:
    ctx.iteration_begin(0, comm); rank_work()
try:
    ctx.sync_all(1, 5.0)
    print(scen, "OK", time.time() - t0, flush=True)
except Exception as e:
    print(scen, "FAIL", e, time.time() - t0, flush=True)
