"""Sync-only FINISH launch of the general comm kernel (k_comm<false>) with N ranks emulated in
one process on one GPU (every rank's arena local; HBM instead of NVLink): a single-GPU
stand-in for ncu, which cannot replay a cross-rank kernel.
python tools/emul_sync.py MODEL WORLD [CTAS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import real_counts

counts = real_counts(sys.argv[1])
world = int(sys.argv[2])
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 148
ctx = SyncContext(counts, world, list(range(world)), comm_ctas=ctas, timeout_s=20.0, emulate_grads=True)
st = torch.cuda.Stream()
for li in range(world):
    for l in range(len(counts)):
        ctx.gradgen_layer(li, 7 + li, 0, l, st)
st.synchronize()
for k in range(4):
    for li in range(world):
        for l in range(len(counts)):
            ctx.layer_ready(li, l, k, None, st)
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
    print(sys.argv[1:], k, "ms", round(s.elapsed_time(e), 4), flush=True)
ctx.close()
