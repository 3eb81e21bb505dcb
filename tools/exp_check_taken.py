import os, sys
sys.path.insert(0, "/root/repo")
import torch, torch.distributed as dist
from paper_1905_03960_b200.runtime import SyncContext, connect
from paper_1905_03960_b200.torch_models import real_counts
from paper_1905_03960_b200.plan import make_p3_plan
from paper_1905_03960_b200.model import ModelProfile, LayerSpec
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
counts = real_counts("resnet50")
ctx = SyncContext(counts, world, [rank], comm_ctas=148, comm_threads=512, timeout_s=30.0, emulate_grads=True)
connect(ctx)
plan = make_p3_plan(ModelProfile("x", 0, tuple(LayerSpec(i, "l", c, 0, 0) for i, c in enumerate(counts))), world)
own = [0] * len(counts)
for s in plan.slices:
    if s.server == rank: own[s.key.layer_index] += 1
st = torch.cuda.Stream()
for l in range(len(counts)): ctx.gradgen_layer(0, 7 + rank, 0, l, st)
st.synchronize()
for k in range(3):
    for l in range(len(counts)): ctx.layer_ready(0, l, k, None, st)
    st.synchronize(); dist.barrier()
    ctx.iteration_begin(k, st); ctx.iteration_end(k); ctx.sync_all(k + 1, 30.0); st.synchronize()
    d = ctx.debug_snapshot(0)
    bad = [(l, d["srv_taken"][l], own[l], d["hint"][l]) for l in range(len(counts)) if d["srv_taken"][l] != own[l]]
    print(f"rank {rank} k {k} reduced {d['reduced']} own_total {sum(own)} layers with srv_taken != owned: {len(bad)} e.g. {bad[:6]}", flush=True)
    dist.barrier()
dist.destroy_process_group()
