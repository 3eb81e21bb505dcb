"""torch.profiler kernel-time breakdown of P3 vs no-sync steps (torchrun, rank 0 prints)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from torch.profiler import profile, ProfilerActivity
from paper_1905_03960_b200.ddp import P3DataParallel
from paper_1905_03960_b200.torch_models import build_model, synthetic_batch, loss_fn
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1: dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
name = sys.argv[1]; B = int(sys.argv[2])
x, y = synthetic_batch(name, B, seed=1 + rank)
torch.manual_seed(0); m = build_model(name).cuda().to(memory_format=torch.channels_last)
for mode in ("nosync", "p3"):
    if mode == "p3":
        d = P3DataParallel(m, lr=0.01)
    else:
        d = m
    for _ in range(4): loss_fn(name, d, x, y).backward()
    if mode == "p3": d.synchronize()
    torch.cuda.synchronize()
    if world > 1: dist.barrier()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3): loss_fn(name, d, x, y).backward()
        if mode == "p3": d.synchronize()
        torch.cuda.synchronize()
    if rank == 0:
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        t0 = min(e.time_range.start for e in evs); t1 = max(e.time_range.end for e in evs)
        tot = {}
        for e in evs:
            k = e.name[:70]; tot[k] = tot.get(k, 0) + (e.time_range.end - e.time_range.start)
        comm = sum(v for k, v in tot.items() if "k_comm" in k)
        print(f"PROF {mode}: span {(t1-t0)/3/1000:.2f} ms/step, kernel sum {(sum(tot.values())-comm)/3/1000:.2f} ms/step (excl comm), comm {comm/3/1000:.2f} ms/step", flush=True)
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
            print(f"PROF   {mode} {v/3/1000:8.3f} ms  {k}", flush=True)
        if mode == "p3":
            # comm kernel intervals vs the step
            cs = sorted((e.time_range.start - t0, e.time_range.end - t0) for e in evs if "k_comm" in e.name)
            print("PROF comm intervals (us):", [(round(a), round(b - a)) for a, b in cs[:40]], flush=True)
if world > 1: dist.destroy_process_group()
