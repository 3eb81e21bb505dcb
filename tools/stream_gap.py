"""N=1 FINISH (k_update_stream) timed as bench.py times it (256 MB L2-flush write, a sleep so the
host enqueues ahead, events around iteration_end), plus an empty kernel between the same events:
run plain for the event times, under `ncu --cache-control none` for the kernel's own duration.
python tools/stream_gap.py [MODEL]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import real_counts

counts = real_counts(sys.argv[1] if len(sys.argv) > 1 else "resnet50")
ctx = SyncContext(counts, 1, [0], comm_ctas=148, timeout_s=20.0, emulate_grads=True)
st = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for l in range(len(counts)):
    ctx.gradgen_layer(0, 7, 0, l, st)
st.synchronize()
ev, empty = [], []
for k in range(8):
    with torch.cuda.stream(st):
        flush.fill_(k)
    for l in range(len(counts)):
        ctx.layer_ready(0, l, k, None, st)
    st.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        torch.cuda._sleep(200_000)
    ctx.iteration_begin(k, st)
    s.record(st)
    ctx.iteration_end(k)
    e.record(st)
    ctx.sync_all(k + 1, 20.0)
    st.synchronize()
    # an almost empty kernel between the same kind of events
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        torch.cuda._sleep(200_000)
        s2.record(st)
        torch.cuda._sleep(1)
        e2.record(st)
    st.synchronize()
    if k >= 2:
        ev.append(s.elapsed_time(e))
        empty.append(s2.elapsed_time(e2))
print("GAP", {"finish_ms": [round(x, 4) for x in ev], "empty_kernel_ms": [round(x, 4) for x in empty]}, flush=True)
ctx.close()
